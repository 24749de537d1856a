"""The reference's cone-level Python API (conic_ipm.cones: update_scaling,
ScalingState.kkt_values, apply_H, combined_ds, step_length, neighborhood_ok,
is_in_cone / is_in_dual_cone, soc_residuals_batch) served by the device cone
kernels (paper_2412_19027_b200/cones.py), against the known answers of the
unmodified reference (tests/golden/kernels.json) at the tolerances of
tests/test_oracle.py."""
import numpy as np
import pytest

from golden_io import cone_from_doc, load_kernels
from paper_2412_19027_b200 import cones as C
from paper_2412_19027_b200.exceptions import StepTooSmall
from paper_2412_19027_b200.model import ConeSpec


KERNELS = load_kernels()
CASES = KERNELS["cones"]


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(CASES)))
def test_gpu_cone_api_matches_reference(gpu, idx):
    case = CASES[idx]
    cs = C.ConeSet.from_specs([cone_from_doc(c) for c in case["cones"]])
    sv, zv, mu = np.array(case["s"]), np.array(case["z"]), case["mu"]
    st = C.update_scaling(cs, sv, zv, mu)
    diag, blocks = st.kkt_values()
    np.testing.assert_array_equal(diag, case["scaling"]["diag"])
    assert len(blocks) == len(case["scaling"]["blocks"])
    for (off, blk), (roff, rb) in zip(blocks, case["scaling"]["blocks"]):
        assert off == roff
        np.testing.assert_allclose(blk, np.array(rb).reshape(blk.shape), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(C.apply_H(st, np.array(case["v"])), case["Hv"], rtol=1e-12, atol=1e-12)
    if case["combined_ds"] is not None:
        got = C.combined_ds(st, cs, sv, zv, np.array(case["dz"]), np.array(case["ds"]), case["sigma"], mu)
        np.testing.assert_allclose(got, case["combined_ds"], rtol=1e-11, atol=1e-11)
    s = case["step"]
    req = C.StepLengthRequest(z=zv, s=sv, dz=np.array(case["dz"]), ds=np.array(case["ds"]), tau=s["tau"],
                              kappa=s["kappa"], dtau=s["dtau"], dkappa=s["dkappa"])
    if s["alpha"] is None:
        with pytest.raises(StepTooSmall):
            C.step_length(req, cs)
    else:
        assert C.step_length(req, cs) == pytest.approx(s["alpha"], rel=1e-13)
    for beta, want in case["neighborhood"].items():
        assert C.neighborhood_ok(cs, sv, zv, mu, float(beta)) == want
    assert C.is_in_cone(cs, sv, strict=True) == case["in_cone"]
    assert C.is_in_dual_cone(cs, zv, strict=True) == case["in_dual"]


@pytest.mark.gpu
def test_gpu_cone_api_soc_residuals_bitwise(gpu):
    r = KERNELS["soc_residuals"]
    cs = C.ConeSet.from_specs([ConeSpec("soc", d) for d in r["dims"]])
    np.testing.assert_array_equal(C.soc_residuals_batch(cs, np.array(r["x"])), np.array(r["r"]))


def test_cone_set_from_specs_and_degree():
    cs = C.ConeSet.from_specs([ConeSpec("zero", 2), ConeSpec("nonneg", 3), ConeSpec("soc", 4),
                               ConeSpec("exp", 3), ConeSpec("pow", 3, 0.3), ConeSpec("psd", 6, side=3)])
    assert (cs.m, cs.zero_dim, cs.nonneg_dim) == (21, 2, 3)
    assert cs.socs == [(5, 4)] and cs.exps == [9] and cs.pows == [(12, 0.3)] and cs.psds == [(15, 3)]
    assert C.degree(cs) == 3 + 1 + 3 + 3 + 3
    with pytest.raises(Exception):
        C.ConeSet.from_specs([ConeSpec("soc", 3), ConeSpec("nonneg", 2)])
