"""GPU tests of the cone kernels one reference function at a time, against the
known answers the UNMODIFIED reference produced (tests/golden/kernels.json,
written by tests/golden/make_golden.py):

* update_scaling + ScalingState.kkt_values  (cones/scaling.py:201-251)
* apply_H                                    (cones/scaling.py:254-274)
* combined_ds                                (cones/scaling.py:277-320)
* step_length                                (cones/steps.py:79-116)
* neighborhood_ok                            (cones/scaling.py:364-401)
* is_in_cone / is_in_dual_cone (strict)      (cones/set.py:166-207)
* soc_residuals_batch, bit-exact (SPEC AC11) (cones/steps.py:136-186)

Tolerances are those of tests/test_oracle.py: 1e-12 for the scaling blocks and
H v, 1e-11 for combined_ds, 1e-13 relative for the step length, exact for
booleans and the batched SOC residuals.  Every call goes through the C ABI
(include/cipm.h)."""
import ctypes

import numpy as np
import pytest

from golden_io import cone_from_doc, load_kernels
from paper_2412_19027_b200.csr import CsrMatrix
from paper_2412_19027_b200.model import ProblemData

pytestmark = pytest.mark.gpu

KERNELS = load_kernels()
CASES = KERNELS["cones"]


def _host_problem(cones, n=2, seed=0):
    """A small valid problem over the given cone list (values are irrelevant: the
    seams run at an iterate set through cipm_set_iterate)."""
    m = sum(c.dim for c in cones)
    rng = np.random.default_rng(seed)
    P = CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))
    A = CsrMatrix(m, n, np.arange(m + 1, dtype=np.int64), (np.arange(m) % n).astype(np.int64),
                  rng.standard_normal(m) + 2.0)
    return ProblemData(P, A, np.zeros(n), np.zeros(m), cones)


def _solver(cones):
    from paper_2412_19027_b200.solver import Solver
    s = Solver(_host_problem(cones))
    assert np.array_equal(s._perm, np.arange(s.m)), "kernel cases are family ordered"
    return s


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _set_point(s, sv, zv, tau, kappa, mu):
    s._ctx.call("cipm_set_iterate", _ptr(np.zeros(s.n)), _ptr(zv), _ptr(sv), _ptr(np.array([tau, kappa, mu])))


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_gpu_scaling_and_apply_h_match_reference(gpu, idx):
    case = CASES[idx]
    cones = [cone_from_doc(c) for c in case["cones"]]
    s = _solver(cones)
    try:
        sv, zv = np.array(case["s"]), np.array(case["z"])
        _set_point(s, sv, zv, 1.0, 1.0, case["mu"])
        s._ctx.call("cipm_update_scaling")
        lin = s.layout.zero_dim + s.layout.nonneg_dim
        blocks = s._block_list()
        total = sum(d * (d + 1) // 2 for _, d in blocks)
        diag, hv = np.zeros(lin), np.zeros(max(total, 1))
        s._ctx.call("cipm_scaling_values", _ptr(diag), _ptr(hv))
        np.testing.assert_array_equal(diag, case["scaling"]["diag"])
        k = 0
        assert len(blocks) == len(case["scaling"]["blocks"])
        for (off, d), (roff, rb) in zip(blocks, case["scaling"]["blocks"]):
            assert off == roff
            iu = np.triu_indices(d)
            want = np.array(rb).reshape(d, d)[iu]
            np.testing.assert_allclose(hv[k:k + len(want)], want, rtol=1e-12, atol=1e-12)
            k += len(want)
        out = np.zeros(s.m)
        s._ctx.call("cipm_apply_h", _ptr(np.array(case["v"])), _ptr(out))
        np.testing.assert_allclose(out, case["Hv"], rtol=1e-12, atol=1e-12)
        if case["combined_ds"] is not None:
            got = np.zeros(s.m)
            s._ctx.call("cipm_combined_ds", _ptr(np.array(case["dz"])), _ptr(np.array(case["ds"])),
                        case["sigma"], case["mu"], _ptr(got))
            np.testing.assert_allclose(got, case["combined_ds"], rtol=1e-11, atol=1e-11)
    finally:
        s.close()


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_gpu_step_neighborhood_membership_match_reference(gpu, idx):
    from paper_2412_19027_b200.exceptions import StepTooSmall
    case = CASES[idx]
    cones = [cone_from_doc(c) for c in case["cones"]]
    s = _solver(cones)
    try:
        sv, zv = np.array(case["s"]), np.array(case["z"])
        st = case["step"]
        _set_point(s, sv, zv, st["tau"], st["kappa"], case["mu"])
        s._ctx.call("cipm_set_direction", 0, None, _ptr(np.array(case["dz"])), _ptr(np.array(case["ds"])),
                    _ptr(np.array([st["dtau"], st["dkappa"]])))
        alpha = ctypes.c_double(0.0)
        if st["alpha"] is None:
            with pytest.raises(StepTooSmall):
                s._ctx.call("cipm_step_length", 0, ctypes.byref(alpha))
        else:
            s._ctx.call("cipm_step_length", 0, ctypes.byref(alpha))
            assert alpha.value == pytest.approx(st["alpha"], rel=1e-13)
        ok = ctypes.c_int(-1)
        for beta, want in case["neighborhood"].items():
            _set_point(s, sv, zv, 1.0, 1.0, case["mu"])
            s._ctx.call("cipm_neighborhood_ok", case["mu"], float(beta), ctypes.byref(ok))
            assert bool(ok.value) == want, (beta, ok.value, want)
        inc, ind = ctypes.c_int(-1), ctypes.c_int(-1)
        s._ctx.call("cipm_membership", _ptr(sv), _ptr(zv), ctypes.byref(inc), ctypes.byref(ind))
        assert bool(inc.value) == case["in_cone"]
        assert bool(ind.value) == case["in_dual"]
        # a point outside the cone: flip the sign of the first nonneg / SOC head / PSD diagonal entry
        lay = s.layout
        heads = ([lay.zero_dim] if lay.nonneg_dim else []) + list(lay.soc_off) + list(lay.psd_off)
        if heads:
            bad = sv.copy()
            bad[heads[0]] = -abs(bad[heads[0]]) - 1.0
            s._ctx.call("cipm_membership", _ptr(bad), _ptr(zv), ctypes.byref(inc), ctypes.byref(ind))
            assert inc.value == 0 and ind.value == int(case["in_dual"])
    finally:
        s.close()


def test_gpu_soc_residuals_bitwise(gpu):
    """SPEC AC11: per-SOC t^2 - |u|^2 in the reference's fixed summation order
    (chunks of 8 left to right, then pairwise rounds with the odd partial
    carried) — equal bit for bit to soc_residuals_batch."""
    from paper_2412_19027_b200.model import ConeSpec
    r = KERNELS["soc_residuals"]
    cones = [ConeSpec("soc", d) for d in r["dims"]]
    s = _solver(cones)
    try:
        out = np.zeros(len(cones))
        s._ctx.call("cipm_soc_residuals", _ptr(np.array(r["x"])), _ptr(out))
        np.testing.assert_array_equal(out, np.array(r["r"]))
        assert out[0] == 0.0            # (5, 3, 4) -> 0 exactly
    finally:
        s.close()
