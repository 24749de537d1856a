"""Batched same-pattern instances (C5b): host equilibration (CPU) and the
one-CTA-per-instance device IPM against the oracle (GPU)."""
import numpy as np
import pytest

from oracle import OracleSolver
from paper_2412_19027_b200 import generators as G
from paper_2412_19027_b200 import model
from paper_2412_19027_b200.batch import equilibrate_batch
from paper_2412_19027_b200.settings import SolverSettings


def _mpc(k):
    return [G.gen_mpc(seed=s) for s in range(k)]


def test_equilibrate_batch_bitwise_matches_per_instance():
    probs = _mpc(6)
    reo = [model.reorder_cones(p)[0] for p in probs]
    P, A = reo[0].P, reo[0].A
    pv = np.stack([r.P.values for r in reo])
    av = np.stack([r.A.values for r in reo])
    q = np.stack([r.q for r in reo])
    b = np.stack([r.b for r in reo])
    pv_s, av_s, q_s, b_s, d_row, d_col, c_obj = equilibrate_batch(P, A, pv, av, q, b)
    for k, r in enumerate(reo):
        s, e = model.equilibrate(r)
        np.testing.assert_array_equal(pv_s[k], s.P.values)
        np.testing.assert_array_equal(av_s[k], s.A.values)
        np.testing.assert_array_equal(q_s[k], s.q)
        np.testing.assert_array_equal(b_s[k], s.b)
        np.testing.assert_array_equal(d_row[k], e.d_row)
        np.testing.assert_array_equal(d_col[k], e.d_col)
        assert c_obj[k] == e.c_obj


def test_mpc_instances_share_one_pattern():
    probs = _mpc(4)
    for p in probs[1:]:
        np.testing.assert_array_equal(p.A.rowptr, probs[0].A.rowptr)
        np.testing.assert_array_equal(p.A.colidx, probs[0].A.colidx)
    assert probs[0].n == 118 and probs[0].m == 324


def _check(res, ref):
    assert res.status == ref.status, (res.status, ref.status)
    assert abs(res.iterations - ref.iterations) <= 1, (res.iterations, ref.iterations)
    if ref.status in ("optimal", "almost_optimal"):
        tol = 1e-6 * max(1.0, abs(ref.obj_primal))
        assert abs(res.obj_primal - ref.obj_primal) <= tol
        assert abs(res.obj_dual - ref.obj_dual) <= 1e-6 * max(1.0, abs(ref.obj_dual))
        np.testing.assert_allclose(res.x, ref.x, atol=1e-5 * max(1.0, np.max(np.abs(ref.x))))


@pytest.mark.gpu
def test_gpu_batch_mpc_matches_oracle(gpu):
    from paper_2412_19027_b200.batch import BatchSolver
    probs = _mpc(24)
    cfg = SolverSettings(eps_feas=1e-8)
    bs = BatchSolver(probs, cfg)
    out = bs.solve()
    bs.close()
    for p, r in zip(probs, out):
        _check(r, OracleSolver(p, cfg).solve())


@pytest.mark.gpu
def test_gpu_batch_lp_family_and_update(gpu):
    from paper_2412_19027_b200.batch import BatchSolver
    base = G.gen_lp(40, 80, seed=3)
    rng = np.random.default_rng(0)
    probs = []
    for k in range(8):
        p = base.copy()
        p.q = base.q * (1.0 + 0.1 * rng.standard_normal(base.n))
        probs.append(p)
    cfg = SolverSettings(eps_feas=1e-8)
    bs = BatchSolver(probs, cfg)
    out = bs.solve()
    for p, r in zip(probs, out):
        _check(r, OracleSolver(p, cfg).solve())
    # parametric: new q for every instance, same device pattern
    q2 = np.stack([p.q * 1.05 for p in probs])
    bs.update_data(q=q2)
    out2 = bs.solve()
    bs.close()
    for k, r in enumerate(out2):
        p = probs[k].copy()
        p.q = q2[k]
        _check(r, OracleSolver(p, cfg).solve())


@pytest.mark.gpu
def test_gpu_batch_infeasible_instances(gpu):
    from golden_io import load_instance, problem_from_doc
    from paper_2412_19027_b200.batch import BatchSolver
    for name in ("primal_infeasible_lp", "dual_infeasible_lp"):
        doc = load_instance(name)
        p = problem_from_doc(doc)
        s = doc["settings"]
        cfg = SolverSettings(eps_feas=s["eps_feas"], max_iter=s["max_iter"])
        bs = BatchSolver([p, p.copy()], cfg)
        out = bs.solve()
        bs.close()
        for r in out:
            assert r.status == doc["result"]["status"]
            assert abs(r.iterations - doc["result"]["iterations"]) <= 1
            if doc["result"]["certificate"] is not None:
                np.testing.assert_allclose(r.certificate, doc["result"]["certificate"], atol=1e-6)


@pytest.mark.gpu
def test_gpu_batch_partial_updates_match_fresh(gpu):
    """update_data(b=) alone, then q and b together, then after a host-equilibrated
    upload: each equals a fresh BatchSolver on the same data bit for bit."""
    from paper_2412_19027_b200.batch import BatchSolver
    base = G.gen_mpc(seed=5)
    probs = [G.gen_mpc(seed=5 + k) for k in range(6)]
    cfg = SolverSettings(eps_feas=1e-8)
    rng = np.random.default_rng(1)
    bs = BatchSolver(probs, cfg)
    bs.solve()

    def fresh(qs, bsv):
        ps = []
        for k, p in enumerate(probs):
            c = p.copy()
            c.q, c.b = qs[k].copy(), bsv[k].copy()
            ps.append(c)
        f = BatchSolver(ps, cfg)
        out = f.solve()
        f.close()
        return out

    def same(a, b):
        for ra, rb in zip(a, b):
            assert ra.status == rb.status and ra.iterations == rb.iterations
            np.testing.assert_array_equal(ra.x, rb.x)
            np.testing.assert_array_equal(ra.z, rb.z)

    q0 = np.stack([p.q for p in probs])
    b1 = np.stack([p.b for p in probs]) * (1.0 + 0.05 * rng.standard_normal((len(probs), base.m)))
    bs.update_data(b=b1)
    same(bs.solve(), fresh(q0, b1))
    q2 = q0 * 1.1
    b2 = b1 * 0.9
    bs.update_data(q=q2, b=b2)
    same(bs.solve(), fresh(q2, b2))
    bs._upload_host_equilibrated()
    q3 = q2 * 0.95
    bs.update_data(q=q3)                 # must re-send raw P / A / b, not reuse the scaled arrays
    out3 = bs.solve()
    bs.close()
    ref3 = fresh(q3, b2)
    for ra, rb in zip(out3, ref3):
        assert ra.status == rb.status
        assert abs(ra.obj_primal - rb.obj_primal) <= 1e-9 * max(1.0, abs(rb.obj_primal))


def test_batch_update_rejects_non_finite():
    """BatchSolver.update_data re-validates like the reference's update_data (problem.py:149-174)."""
    from paper_2412_19027_b200.batch import BatchSolver
    from paper_2412_19027_b200.exceptions import NonFiniteData
    bs = BatchSolver.__new__(BatchSolver)
    bs.count, bs.n, bs.m = 2, 3, 4
    q = np.ones((2, 3))
    q[1, 2] = np.nan
    with pytest.raises(NonFiniteData):
        bs.update_data(q=q)
    b = np.ones((2, 4))
    b[0, 0] = np.inf
    with pytest.raises(NonFiniteData):
        bs.update_data(b=b)


@pytest.mark.gpu
def test_gpu_batch_c5b_all_2048_match_reference(gpu):
    """The whole C5b batch (2048 MPC QPs, seeds 0..2047) against the unmodified
    reference's per-instance results (tests/golden/mpc2048.json, written by
    tests/golden/make_mpc.py): same status, iterations within 1, objectives
    within 1e-6 relative, for every instance."""
    import json
    import os
    from paper_2412_19027_b200.batch import BatchSolver
    doc = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mpc2048.json")))
    probs = G.build_instances("c5b_mpc", 0, len(doc["status"]))
    bs = BatchSolver(probs, SolverSettings(eps_feas=doc["eps_feas"]))
    out = bs.solve()
    bs.close()
    bad = []
    for k, r in enumerate(out):
        ok = (r.status == doc["status"][k] and abs(r.iterations - doc["iterations"][k]) <= 1
              and abs(r.obj_primal - doc["obj_primal"][k]) <= 1e-6 * max(1.0, abs(doc["obj_primal"][k]))
              and abs(r.obj_dual - doc["obj_dual"][k]) <= 1e-6 * max(1.0, abs(doc["obj_dual"][k])))
        if not ok:
            bad.append((k, r.status, r.iterations, r.obj_primal, doc["status"][k], doc["iterations"][k]))
    assert not bad, bad[:10]
    assert sum(r.iterations for r in out) == pytest.approx(sum(doc["iterations"]), abs=len(out) // 100)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 8])
def test_gpu_batch_shards_equal_the_whole_batch(gpu, world):
    """The multi-GPU bench shards the instances contiguously (bench.shard) with no
    collective on the solve path: every shard solved on its own returns, bit for
    bit, what the whole batch returns for those instances (one CTA per instance,
    nothing shared between instances)."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2412_19027_b200.batch import BatchSolver
    total = 256
    cfg = SolverSettings(eps_feas=1e-8)
    probs = G.build_instances("c5b_mpc", 0, total)
    bs = BatchSolver(probs, cfg)
    whole = bs.solve()
    bs.close()
    for rank in range(world):
        lo, hi = bench.shard(total, world, rank)
        part = BatchSolver(G.build_instances("c5b_mpc", lo, hi), cfg)
        got = part.solve()
        part.close()
        for k, r in enumerate(got):
            w = whole[lo + k]
            assert r.status == w.status and r.iterations == w.iterations
            np.testing.assert_array_equal(r.x, w.x)
            np.testing.assert_array_equal(r.z, w.z)
            assert r.obj_primal == w.obj_primal


@pytest.mark.gpu
def test_gpu_solve_many_heterogeneous_equals_per_instance(gpu):
    """solve_many groups instances by pattern: the MPC QPs and the LP family run
    batched, the SOCP / exp-pow / PSD instances through the single-problem path;
    every result equals the per-instance Solver result (status, iterations,
    objectives to 1e-9)."""
    from paper_2412_19027_b200.batch import solve_many
    from paper_2412_19027_b200.solver import Solver
    probs = (G.build_instances("c5b_mpc", 0, 6) + [G.gen_socp(ncones=20, seed=s) for s in range(2)] + [G.gen_lp(n=20, m=40, seed=3)]
             + G.build_instances("c5b_mpc", 6, 9) + [G.gen_psd(ncones=3, side=3, seed=1)])
    cfg = SolverSettings(eps_feas=1e-8)
    got = solve_many(probs, cfg)
    assert len(got) == len(probs)
    for p, r in zip(probs, got):
        s = Solver(p, cfg)
        w = s.solve()
        s.close()
        assert r.status == w.status
        assert abs(r.iterations - w.iterations) <= 1
        assert abs(r.obj_primal - w.obj_primal) <= 1e-9 * max(1.0, abs(w.obj_primal))


def test_batch_results_sequence_cpu():
    """BatchResults: a lazy sequence of reference SolveResults over the host arrays of
    one batched D2H (len, indexing, slices, iteration, cached objects, whole-batch
    columns, certificates as the reference normalises them, ipm.py:401-407)."""
    from paper_2412_19027_b200.batch import BatchResults
    from paper_2412_19027_b200.settings import Status
    c, n, m = 4, 3, 5
    rng = np.random.default_rng(0)
    codes = np.array([0, 1, 2, 3], dtype=np.int32)          # optimal, primal / dual infeasible, almost
    res = rng.standard_normal((c, 9))
    res[:, 8] = [7, 11, 13, 9]
    x, z, s = rng.standard_normal((c, n)), rng.standard_normal((c, m)), rng.standard_normal((c, m))
    q, b = rng.standard_normal((c, n)), rng.standard_normal((c, m))
    out = BatchResults(codes, res, x, z, s, q, b, 0.5, 0.25)
    assert len(out) == c
    assert out.status == [Status.OPTIMAL, Status.PRIMAL_INFEASIBLE, Status.DUAL_INFEASIBLE, Status.ALMOST_OPTIMAL]
    np.testing.assert_array_equal(out.iterations, [7, 11, 13, 9])
    np.testing.assert_array_equal(out.obj_primal, res[:, 0])
    r0 = out[0]
    assert r0 is out[0] and out[-4] is r0                   # built once, cached
    assert r0.iterations == 7 and r0.obj_primal == res[0, 0] and r0.certificate is None
    assert r0.gap == abs(res[0, 0] - res[0, 1]) and r0.setup_seconds == 0.5 and r0.solve_seconds == 0.25
    np.testing.assert_array_equal(out[1].certificate, z[1] / abs(float(b[1] @ z[1])))
    np.testing.assert_array_equal(out[2].certificate, x[2] / abs(float(q[2] @ x[2])))
    assert [r.iterations for r in out] == [7, 11, 13, 9]
    assert [r.iterations for r in out[1:3]] == [11, 13]
    with pytest.raises(IndexError):
        out[4]


def test_max_abs_is_the_finiteness_test():
    a = np.random.default_rng(1).standard_normal(1000)
    assert model.max_abs(a) == np.max(np.abs(a))
    assert model.max_abs(np.zeros(0)) == 0.0
    for bad in (np.nan, np.inf, -np.inf):
        for pos in (0, 500, 999):
            v = a.copy()
            v[pos] = bad
            assert not np.isfinite(model.max_abs(v))
