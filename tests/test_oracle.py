"""CPU tests: the oracle restatement is pinned against the reference's golden fixtures."""
import numpy as np
import pytest

from golden_io import instance_names, load_instance, load_kernels, problem_from_doc
from oracle import OracleSolver
from oracle import cones as C
from paper_2412_19027_b200.model import ConeSpec
from paper_2412_19027_b200.settings import SolverSettings

NAMES = instance_names()


def settings_of(doc):
    s = doc["settings"]
    return SolverSettings(eps_feas=s["eps_feas"], precision=s["precision"], max_iter=s["max_iter"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_bitwise(name):
    """Status, iterations, objectives, iterates and the α trace all reproduce the reference."""
    doc = load_instance(name)
    trace = []
    res = OracleSolver(problem_from_doc(doc), settings_of(doc)).solve(
        observer=lambda d: trace.append((d["state"].mu, d["alpha_affine"], d["sigma"], d["alpha_combined"])))
    ref = doc["result"]
    assert res.status == ref["status"]
    assert res.iterations == ref["iterations"]
    assert res.obj_primal == ref["obj_primal"]
    assert res.obj_dual == ref["obj_dual"]
    np.testing.assert_array_equal(res.x, np.array(ref["x"]))
    np.testing.assert_array_equal(res.z, np.array(ref["z"]))
    np.testing.assert_array_equal(res.s, np.array(ref["s"]))
    if ref["certificate"] is not None:
        np.testing.assert_array_equal(res.certificate, np.array(ref["certificate"]))
    got = [list(t) for t in trace]
    want = [[t["mu"], t["alpha_affine"], t["sigma"], t["alpha_combined"]] for t in doc["trace"]]
    assert got == want


def _layout(case):
    return C.ConeLayout.from_specs([ConeSpec(c["kind"], c["dim"], c.get("alpha"), c.get("side"))
                                    for c in case["cones"]])


def test_oracle_kernels_match_reference():
    k = load_kernels()
    for case in k["cones"]:
        lay = _layout(case)
        s, z = np.array(case["s"]), np.array(case["z"])
        sc = C.update_scaling(lay, s, z, case["mu"])
        diag, blocks = sc.kkt_blocks()
        np.testing.assert_array_equal(diag, case["scaling"]["diag"])
        for (off, b), (roff, rb) in zip(blocks, case["scaling"]["blocks"]):
            assert off == roff
            np.testing.assert_allclose(b.ravel(), rb, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(C.apply_h(sc, np.array(case["v"])), case["Hv"], rtol=1e-12, atol=1e-12)
        if case["combined_ds"] is not None:
            got = C.combined_ds(sc, s, z, np.array(case["dz"]), np.array(case["ds"]), case["sigma"], case["mu"])
            np.testing.assert_allclose(got, case["combined_ds"], rtol=1e-11, atol=1e-11)
        st = case["step"]
        if st["alpha"] is not None:
            a = C.step_length(lay, z, s, np.array(case["dz"]), np.array(case["ds"]), st["tau"], st["kappa"],
                              st["dtau"], st["dkappa"])
            assert a == pytest.approx(st["alpha"], rel=1e-13)
        for beta, want in case["neighborhood"].items():
            assert C.neighborhood_ok(lay, s, z, case["mu"], float(beta)) == want
        assert C.in_cone(lay, s) == case["in_cone"]
        assert C.in_dual_cone(lay, z) == case["in_dual"]


def test_oracle_conjugate_points():
    for c in load_kernels()["conjugate"]:
        s = np.array(c["s"])
        w = C.exp_conj(s) if c["kind"] == "exp" else C.pow_conj(s, c["alpha"])
        np.testing.assert_array_equal(w, c["w"])


def test_oracle_soc_residual_order():
    r = load_kernels()["soc_residuals"]
    dims = r["dims"]
    offs = np.concatenate([[0], np.cumsum(dims)[:-1]])
    got = C.soc_residuals_fixed_order(dims, offs, np.array(r["x"]))
    np.testing.assert_array_equal(got, r["r"])
    assert got[0] == 0.0
