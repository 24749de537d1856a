"""GPU tests of the factorisation tiers (warp / CTA / dense tail) on problems that
exercise them, against the oracle, plus run-to-run reproducibility."""
import numpy as np
import pytest

from oracle import OracleSolver
from paper_2412_19027_b200 import generators as G
from paper_2412_19027_b200.settings import SolverSettings

pytestmark = pytest.mark.gpu


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


@pytest.mark.parametrize("n,m,prec", [(200, 400, "full"), (400, 800, "full"), (200, 400, "mixed")])
def test_dense_tail_lp_matches_oracle(gpu, n, m, prec):
    """gen_lp at these sizes has a 180-360-column root supernode: the multi-CTA
    dense tail (DMMA Schur tiles, wavefront tail solves) carries the factor."""
    from paper_2412_19027_b200.solver import Solver
    prob = G.gen_lp(n, m, seed=1)
    cfg = SolverSettings(eps_feas=1e-8, precision=prec)
    s = Solver(prob, cfg)
    assert s.symbolic.info()["max_width"] >= 64
    r1 = s.solve()
    r2 = s.solve()
    s.close()
    ref = OracleSolver(prob, cfg).solve()
    assert r1.status == ref.status == "optimal"
    assert abs(r1.iterations - ref.iterations) <= 1
    assert rel(r1.obj_primal, ref.obj_primal) <= 1e-6
    assert rel(r1.obj_dual, ref.obj_dual) <= 1e-6
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(r1.x, r2.x)


def test_kkt_solve_residual_all_tiers(gpu):
    """Refined KKT solves at an interior iterate reach the refinement target on a
    problem with warp-, CTA- and tail-tier supernodes."""
    import ctypes

    from paper_2412_19027_b200.native import pdbl
    from paper_2412_19027_b200.solver import Solver
    prob = G.gen_lp(400, 800, seed=2)
    s = Solver(prob, SolverSettings(eps_feas=1e-8, max_iter=3))
    s.solve()
    ctx = s._ctx
    ctx.call("cipm_update_scaling")
    ctx.call("cipm_factor")
    dim = s.n + s.m
    rhs = np.random.default_rng(0).standard_normal(dim)
    x = np.zeros(dim)
    steps, res = ctypes.c_int(0), ctypes.c_double(0)
    for _ in range(3):
        ctx.call("cipm_kkt_solve", pdbl(rhs), pdbl(x), ctypes.byref(steps), ctypes.byref(res))
        assert res.value <= 1e-9 * max(1.0, np.max(np.abs(rhs))), (res.value, steps.value)
    s.close()


@pytest.mark.parametrize("name", ["lp_150x300", "socp_40", "psd_6x4", "exppow_20_8", "lasso_10x40"])
def test_device_equilibration_bitwise(gpu, name):
    """setup.cu reorders and Ruiz-equilibrates on the device with the reference's
    arithmetic: D_r, D_c and c equal the host routine (problem.py:222-284) bit for bit."""
    import ctypes

    from golden_io import load_instance, problem_from_doc
    from paper_2412_19027_b200 import model
    from paper_2412_19027_b200.native import pdbl
    from paper_2412_19027_b200.solver import Solver
    prob = problem_from_doc(load_instance(name))
    s = Solver(prob, SolverSettings(eps_feas=1e-8))
    d_row, d_col, c = np.empty(s.m), np.empty(s.n), ctypes.c_double(0)
    s._ctx.call("cipm_ctx_get_equilibration", pdbl(d_row), pdbl(d_col), ctypes.byref(c))
    s.close()
    r, _ = model.reorder_cones(prob)
    _, e = model.equilibrate(r)
    np.testing.assert_array_equal(d_row, e.d_row)
    np.testing.assert_array_equal(d_col, e.d_col)
    assert c.value == e.c_obj


@pytest.mark.parametrize("side,ncones", [(6, 40), (17, 3), (24, 2), (32, 1)])
def test_gpu_psd_sides_match_oracle(gpu, side, ncones):
    """Warp-per-cone PSD kernels for every side the reference accepts (<= 32,
    problem.py:36): same status, iterations within 1 and objectives within 1e-6 of
    the oracle restatement of the reference."""
    from paper_2412_19027_b200.solver import Solver
    prob = G.gen_psd(ncones=ncones, side=side, seed=3)
    cfg = SolverSettings(eps_feas=1e-8)
    s = Solver(prob, cfg)
    r = s.solve()
    s.close()
    ref = OracleSolver(prob, cfg).solve()
    assert r.status == ref.status
    assert abs(r.iterations - ref.iterations) <= 1
    assert rel(r.obj_primal, ref.obj_primal) <= 1e-6
    assert rel(r.obj_dual, ref.obj_dual) <= 1e-6


@pytest.mark.parametrize("side", [2, 3, 6, 8])
def test_gpu_psd_register_kernels_match_lane_groups(gpu, side, monkeypatch):
    """Equal sides <= 8 run the thread-per-cone register kernels (psd_reg.cuh);
    CIPM_PSD_WARP=1 forces the lane-group kernels (psd_warp.cuh).  Same status and
    iterations, objectives to 1e-9 and iterates to 1e-6 (the Jacobi orders differ, so the
    rounding does), and both within 1e-6 of the oracle."""
    from paper_2412_19027_b200.solver import Solver
    prob = G.gen_psd(ncones=24, side=side, seed=5)
    cfg = SolverSettings(eps_feas=1e-8)
    s = Solver(prob, cfg)
    r = s.solve()
    s.close()
    monkeypatch.setenv("CIPM_PSD_WARP", "1")
    s = Solver(prob, cfg)
    w = s.solve()
    s.close()
    assert r.status == w.status
    assert r.iterations == w.iterations
    assert rel(r.obj_primal, w.obj_primal) <= 1e-9
    np.testing.assert_allclose(r.x, w.x, rtol=1e-6, atol=1e-7)   # both at the 1e-8 solve tolerance
    ref = OracleSolver(prob, cfg).solve()
    assert r.status == ref.status
    assert rel(r.obj_primal, ref.obj_primal) <= 1e-6
