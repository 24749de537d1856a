"""Device-backed KKTSystem / assemble (paper_2412_19027_b200/kkt.py) with the
reference's interface (kkt/system.py:64-321): H from ScalingState.kkt_values()
at the reference's own cone points (tests/golden/kernels.json), numeric_factor,
solve_refined and matvec against the dense K = [P A'; A -H] solved by numpy."""
import numpy as np
import pytest

from golden_io import cone_from_doc, load_kernels
from paper_2412_19027_b200 import cones as C
from paper_2412_19027_b200.csr import CsrMatrix
from paper_2412_19027_b200.kkt import KKTSystem, assemble
from paper_2412_19027_b200.settings import FULL, MIXED, RefinementSettings

KERNELS = load_kernels()
CASES = KERNELS["cones"]


def _csr(dense):
    rows, cols = np.nonzero(dense)
    rp = np.zeros(dense.shape[0] + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    return CsrMatrix(dense.shape[0], dense.shape[1], np.cumsum(rp), cols.astype(np.int64), dense[rows, cols])


def _system(case, precision, seed=0):
    cs = C.ConeSet.from_specs([cone_from_doc(c) for c in case["cones"]])
    n, m = 3, cs.m
    rng = np.random.default_rng(seed)
    Pd = rng.standard_normal((n, n))
    Pd = Pd @ Pd.T + np.eye(n)
    Ad = rng.standard_normal((m, n))
    st = C.update_scaling(cs, np.array(case["s"]), np.array(case["z"]), case["mu"])
    diag, blocks = st.kkt_values()
    H = np.zeros((m, m))
    H[np.arange(len(diag)), np.arange(len(diag))] = diag
    for off, b in blocks:
        H[off:off + b.shape[0], off:off + b.shape[0]] = b
    K = np.block([[Pd, Ad.T], [Ad, -H]])
    kkt = assemble(_csr(Pd), _csr(Ad), cs, precision=precision)
    kkt.set_scaling(diag, blocks)
    return kkt, K, rng


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [FULL, MIXED])
@pytest.mark.parametrize("idx", range(len(CASES)))
def test_gpu_kkt_system_solves_and_multiplies(gpu, idx, precision):
    kkt, K, rng = _system(CASES[idx], precision, seed=idx)
    try:
        x = rng.standard_normal(kkt.dim)
        np.testing.assert_allclose(kkt.matvec(x), K @ x, rtol=1e-12, atol=1e-12)
        kkt.numeric_factor()
        assert kkt.num_numeric >= 1 and kkt.num_symbolic == 1
        b = rng.standard_normal(kkt.dim)
        r = kkt.solve_refined(b)
        # the reported residual is that of the returned (best) iterate, against the
        # unregularised K (system.py:279-314)
        assert r.residual == pytest.approx(np.max(np.abs(b - K @ r.x)), rel=1e-6, abs=1e-13)
        assert 1 <= r.steps <= 10
        if precision == FULL or r.residual <= 1e-12 + 1e-12 * np.max(np.abs(b)):
            want = np.linalg.solve(K, b)
            scale = max(1.0, np.max(np.abs(want)))
            np.testing.assert_allclose(r.x, want, rtol=0, atol=1e-8 * scale)
        else:                          # FP32 factor of an ill-conditioned K: the best iterate
            assert r.residual < np.max(np.abs(b))
        # a one-step budget: a valid result, at most one step
        r1 = kkt.solve_refined(b, RefinementSettings(t_max=1))
        assert r1.steps == 1
    finally:
        kkt.close()


@pytest.mark.gpu
def test_gpu_kkt_system_requires_scaling_and_factor(gpu):
    from paper_2412_19027_b200.exceptions import ConicError
    case = CASES[0]
    cs = C.ConeSet.from_specs([cone_from_doc(c) for c in case["cones"]])
    Pd, Ad = np.eye(2), np.ones((cs.m, 2))
    kkt = KKTSystem(_csr(Pd), _csr(Ad), cs)
    try:
        with pytest.raises(ConicError):
            kkt.numeric_factor()
        st = C.update_scaling(cs, np.array(case["s"]), np.array(case["z"]), case["mu"])
        kkt.set_scaling(*st.kkt_values())
        with pytest.raises(ConicError):
            kkt.solve_refined(np.ones(kkt.dim))
    finally:
        kkt.close()
