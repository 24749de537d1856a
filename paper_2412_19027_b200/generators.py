"""Seeded synthetic instances of the BASELINE.json configurations.

The reference ships generators only for portfolio / Huber / entropy /
multistage (``pkg/src/conic_ipm/generators.py``); the north-star configs
need LP, lasso, SOCP, exp+pow, PSD and MPC families, frozen here from the
recipes in SURVEY.md §8(d).  Every generator is a pure function of its size
arguments and ``seed`` (numpy ``default_rng``), so the CPU oracle and the
GPU path see bit-identical inputs.

    C1  gen_lp(2000, 4000)                     random feasible sparse LP
    C2  gen_lasso(50_000, 200_000)             banded lasso QP (mixed precision)
    C3  gen_socp(100_000)                      SOCP, SOC dims U{3..10}
    C4  gen_exppow(50_000, 20_000)             entropy (exp) + geometric mean (pow)
    C5a gen_psd(10_000, 6)                     PSD cones of side 6
    C5b gen_mpc(seed) for seed in 0..2047      MPC QPs sharing one pattern
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .csr import CsrMatrix
from .model import (ProblemData, exp_cone, nonneg_cone, pow_cone, psd_cone,
                    soc_cone, zero_cone)


def _csr(mat) -> CsrMatrix:
    return CsrMatrix.from_scipy(sp.csr_matrix(mat))


def _banded(rng, m: int, n: int, per_row: int, half_width: int, scale: float = 1.0):
    """m×n matrix, per_row N(0,1) entries per row at floor(i n/m) + U{-w..w} mod n."""
    centre = (np.arange(m, dtype=np.int64) * n) // m
    offs = rng.integers(-half_width, half_width + 1, size=(m, per_row))
    cols = (centre[:, None] + offs) % n
    vals = scale * rng.standard_normal((m, per_row))
    rows = np.repeat(np.arange(m, dtype=np.int64), per_row)
    mat = sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(m, n))
    mat.sum_duplicates()
    mat.eliminate_zeros()
    return mat


def _soc_interior(rng, dims) -> np.ndarray:
    parts = []
    for d in dims:
        u = rng.standard_normal(d - 1)
        parts.append(np.concatenate([[np.linalg.norm(u) + 1.0], u]))
    return np.concatenate(parts) if parts else np.zeros(0)


# ---------------------------------------------------------------------------
# C1: random feasible sparse LP
# ---------------------------------------------------------------------------

def gen_lp(n: int = 2000, m: int = 4000, per_row: float = 8.0, seed: int = 0) -> ProblemData:
    """min q'x s.t. Ax + s = b, s ∈ {0}^{m/4} × R_+^{3m/4}; primal+dual feasible."""
    rng = np.random.default_rng(seed)
    mz = m // 4
    a = sp.random(m, n, density=per_row / n, format="csr", random_state=rng,
                  data_rvs=rng.standard_normal)
    x0 = rng.random(n)
    s0 = np.concatenate([np.zeros(mz), rng.random(m - mz)])
    y = np.concatenate([rng.standard_normal(mz), rng.random(m - mz)])
    b = a @ x0 + s0
    q = -(a.T @ y)
    return ProblemData(CsrMatrix.zeros(n, n), _csr(a), q, b,
                       [zero_cone(mz), nonneg_cone(m - mz)])


# ---------------------------------------------------------------------------
# C2: lasso  min y'y + λ 1't  s.t.  y = Ax - b, -t <= x <= t
# ---------------------------------------------------------------------------

def gen_lasso(nf: int = 50_000, mr: int = 200_000, seed: int = 0) -> ProblemData:
    rng = np.random.default_rng(seed)
    a = _banded(rng, mr, nf, 4, 8)
    xs = rng.standard_normal(nf) * (rng.random(nf) < 0.1)
    b = a @ xs + 0.1 * rng.standard_normal(mr)
    lam = 0.2 * float(np.max(np.abs(a.T @ b)))
    n = nf + mr + nf
    eye_f = sp.identity(nf, format="csr")
    eye_r = sp.identity(mr, format="csr")
    zr_f = sp.csr_matrix((mr, nf))
    zf_r = sp.csr_matrix((nf, mr))
    rows_zero = sp.hstack([a, -eye_r, zr_f])           # Ax - y + s = b, s = 0
    rows_up = sp.hstack([eye_f, zf_r, -eye_f])         # x - t <= 0
    rows_dn = sp.hstack([-eye_f, zf_r, -eye_f])        # -x - t <= 0
    a_c = sp.vstack([rows_zero, rows_up, rows_dn]).tocsr()
    b_c = np.concatenate([b, np.zeros(2 * nf)])
    q = np.concatenate([np.zeros(nf + mr), lam * np.ones(nf)])
    pdiag = np.concatenate([np.zeros(nf), 2.0 * np.ones(mr), np.zeros(nf)])
    P = sp.diags(pdiag).tocsr()
    P.eliminate_zeros()
    return ProblemData(_csr(P), _csr(a_c), q, b_c, [zero_cone(mr), nonneg_cone(2 * nf)])


# ---------------------------------------------------------------------------
# C3: SOCP with many small second-order cones
# ---------------------------------------------------------------------------

def gen_socp(ncones: int = 100_000, seed: int = 0, dmin: int = 3, dmax: int = 10) -> ProblemData:
    rng = np.random.default_rng(seed)
    dims = rng.integers(dmin, dmax + 1, size=ncones)
    m = int(dims.sum())
    n = 2 * ncones
    a = _banded(rng, m, n, 3, 8)
    s0 = _soc_interior(rng, dims)
    y = _soc_interior(rng, dims)
    x0 = rng.standard_normal(n)
    b = a @ x0 + s0
    q = -(a.T @ y)
    P = 0.1 * sp.identity(n, format="csr")
    return ProblemData(_csr(P), _csr(a), q, b, [soc_cone(int(d)) for d in dims])


# ---------------------------------------------------------------------------
# C4: block-simplex entropy maximisation (exp) + geometric means (pow)
# ---------------------------------------------------------------------------

def gen_exppow(n_exp: int = 50_000, n_pow: int = 20_000, seed: int = 0,
               block: int = 100) -> ProblemData:
    """max Σ t_i + Σ w_j over (x, t, u, v, w).

    exp cones (t_i, x_i, 1); block simplex rows Σ_{i∈b} x_i = 1/#blocks;
    banded A_e x <= A_e x̂ (4 nnz/row, scaled by √n_e); pow cones
    (u_j, v_j, w_j) ∈ K_pow(α_j) with a banded nonnegative coupling
    |C|[u;v] + u + v <= 1.
    """
    rng = np.random.default_rng(seed)
    ne, npw = n_exp, n_pow
    nblk = max(1, ne // block)
    blk_of = np.minimum(np.arange(ne) // block, nblk - 1)
    me = int(np.floor(0.5 * ne + 0.5))
    ae = _banded(rng, me, ne, 4, 8, scale=np.sqrt(ne))
    v = rng.random(ne)
    vsum = np.bincount(blk_of, weights=v, minlength=nblk)
    xhat = v / (nblk * vsum[blk_of])
    be = ae @ xhat
    alphas = rng.uniform(0.2, 0.8, size=npw)
    coup = _banded(rng, npw, 2 * npw, 2, 4) if npw else sp.csr_matrix((0, 0))
    coup = abs(coup) * 0.1

    n = 2 * ne + 3 * npw
    ix, it = 0, ne
    iu, iv, iw = 2 * ne, 2 * ne + npw, 2 * ne + 2 * npw
    rows = []
    rhs = []
    # zero: block simplex
    zr = sp.csr_matrix((np.ones(ne), (blk_of, ix + np.arange(ne))), shape=(nblk, n))
    rows.append(zr)
    rhs.append(np.full(nblk, 1.0 / nblk))
    # nonneg: A_e x <= b_e
    rows.append(sp.hstack([ae, sp.csr_matrix((me, n - ne))]).tocsr())
    rhs.append(be)
    # nonneg: coupling on (u, v)
    if npw:
        cu = coup + sp.hstack([sp.identity(npw), sp.identity(npw)])
        rows.append(sp.hstack([sp.csr_matrix((npw, 2 * ne)), cu, sp.csr_matrix((npw, npw))]).tocsr())
        rhs.append(np.ones(npw))
    # exp cones: s = (t_i, x_i, 1)
    r = np.arange(3 * ne)
    ecols = np.empty(3 * ne, dtype=np.int64)
    evals = np.zeros(3 * ne)
    ecols[0::3] = it + np.arange(ne)
    ecols[1::3] = ix + np.arange(ne)
    ecols[2::3] = 0
    evals[0::3] = -1.0
    evals[1::3] = -1.0
    ex = sp.csr_matrix((evals, (r, ecols)), shape=(3 * ne, n))
    ex.eliminate_zeros()
    rows.append(ex)
    erhs = np.zeros(3 * ne)
    erhs[2::3] = 1.0
    rhs.append(erhs)
    # pow cones: s = (u_j, v_j, w_j)
    if npw:
        r = np.arange(3 * npw)
        pc = np.empty(3 * npw, dtype=np.int64)
        pc[0::3] = iu + np.arange(npw)
        pc[1::3] = iv + np.arange(npw)
        pc[2::3] = iw + np.arange(npw)
        rows.append(sp.csr_matrix((-np.ones(3 * npw), (r, pc)), shape=(3 * npw, n)))
        rhs.append(np.zeros(3 * npw))
    a_c = sp.vstack(rows).tocsr()
    b_c = np.concatenate(rhs)
    q = np.zeros(n)
    q[it:it + ne] = -1.0
    q[iw:iw + npw] = -1.0
    cones = [zero_cone(nblk), nonneg_cone(me + npw)]
    cones += [exp_cone() for _ in range(ne)]
    cones += [pow_cone(float(a)) for a in alphas]
    return ProblemData(CsrMatrix.zeros(n, n), _csr(a_c), q, b_c, cones)


# ---------------------------------------------------------------------------
# C5a: many equal-size PSD cones
# ---------------------------------------------------------------------------

def _svec(x: np.ndarray) -> np.ndarray:
    side = x.shape[0]
    il, jl = np.tril_indices(side)
    order = np.lexsort((il, jl))          # column-major lower triangle
    il, jl = il[order], jl[order]
    v = x[il, jl].copy()
    v[il != jl] *= np.sqrt(2.0)
    return v


def gen_psd(ncones: int = 10_000, side: int = 6, seed: int = 0) -> ProblemData:
    rng = np.random.default_rng(seed)
    d = side * (side + 1) // 2
    m = ncones * d
    n = m // 3
    a = _banded(rng, m, n, 3, 8)

    def interior():
        parts = []
        for _ in range(ncones):
            g = rng.standard_normal((side, side))
            parts.append(_svec(g @ g.T / side + np.eye(side)))
        return np.concatenate(parts)

    s0 = interior()
    y = interior()
    x0 = rng.standard_normal(n)
    b = a @ x0 + s0
    q = -(a.T @ y)
    return ProblemData(CsrMatrix.zeros(n, n), _csr(a), q, b, [psd_cone(side) for _ in range(ncones)])


# ---------------------------------------------------------------------------
# C5b: MPC QP (one instance per seed; all instances share one pattern)
# ---------------------------------------------------------------------------

def gen_mpc(seed: int = 0, nx: int = 8, nu: int = 3, horizon: int = 10,
            xmax: float = 5.0, umax: float = 1.0) -> ProblemData:
    """min Σ ½x_k'x_k + ½·0.1 u_k'u_k  s.t. x_{k+1} = A x_k + B u_k, x_0 fixed, boxes."""
    rng = np.random.default_rng(seed)
    ad = np.eye(nx) + 0.1 * rng.standard_normal((nx, nx))
    rho = float(np.max(np.abs(np.linalg.eigvals(ad))))
    ad = ad * (0.95 / rho) if rho >= 0.95 else ad
    bd = rng.standard_normal((nx, nu))
    x0 = rng.standard_normal(nx)
    # keep the u = 0 trajectory inside the box so every instance is feasible
    traj, xk = [], x0.copy()
    for _ in range(horizon + 1):
        traj.append(np.max(np.abs(xk)))
        xk = ad @ xk
    peak = max(traj)
    if peak > 0.8 * xmax:
        x0 = x0 * (0.8 * xmax / peak)

    N = horizon
    nxv = (N + 1) * nx
    n = nxv + N * nu

    def xs(k):
        return k * nx

    def us(k):
        return nxv + k * nu

    dyn = sp.lil_matrix((nx + N * nx, n))
    rhs_z = np.zeros(nx + N * nx)
    dyn[0:nx, xs(0):xs(0) + nx] = np.eye(nx)        # x_0 = x0
    rhs_z[0:nx] = x0
    for k in range(N):
        r0 = nx + k * nx
        dyn[r0:r0 + nx, xs(k + 1):xs(k + 1) + nx] = np.eye(nx)
        dyn[r0:r0 + nx, xs(k):xs(k) + nx] = -ad
        dyn[r0:r0 + nx, us(k):us(k) + nu] = -bd
    box = sp.vstack([sp.identity(n), -sp.identity(n)])
    lim = np.concatenate([np.full(nxv, xmax), np.full(N * nu, umax)])
    a_c = sp.vstack([dyn.tocsr(), box]).tocsr()
    b_c = np.concatenate([rhs_z, lim, lim])
    pdiag = np.concatenate([np.ones(nxv), 0.1 * np.ones(N * nu)])
    P = sp.diags(pdiag).tocsr()
    return ProblemData(_csr(P), _csr(a_c), np.zeros(n), b_c,
                       [zero_cone(nx + N * nx), nonneg_cone(2 * n)])


CONFIGS = {
    "c1_lp": dict(gen="lp", kwargs=dict(n=2000, m=4000), precision="full"),
    "c2_lasso": dict(gen="lasso", kwargs=dict(nf=50_000, mr=200_000), precision="mixed"),
    "c3_socp": dict(gen="socp", kwargs=dict(ncones=100_000), precision="full"),
    "c4_exppow": dict(gen="exppow", kwargs=dict(n_exp=50_000, n_pow=20_000), precision="full"),
    "c5a_psd": dict(gen="psd", kwargs=dict(ncones=10_000, side=6), precision="full"),
    # C5b: 8 x 256 = 2048 independent MPC QPs (seeds 0..2047), one shared pattern
    "c5b_mpc": dict(gen="mpc", kwargs=dict(), precision="full", instances=2048),
}


def build_instances(config: str, lo: int, hi: int):
    """Instances lo .. hi-1 of a batched config (seed = instance index)."""
    spec = CONFIGS[config]
    return [GENERATORS[spec["gen"]](seed=k, **spec["kwargs"]) for k in range(lo, hi)]

GENERATORS = {"lp": gen_lp, "lasso": gen_lasso, "socp": gen_socp, "exppow": gen_exppow,
              "psd": gen_psd, "mpc": gen_mpc}


def build(config: str, seed: int = 0, **overrides) -> ProblemData:
    spec = CONFIGS[config]
    kw = dict(spec["kwargs"])
    kw.update(overrides)
    return GENERATORS[spec["gen"]](seed=seed, **kw)
