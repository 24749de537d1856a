"""The reference's benchmark problem families (portfolio, huber, entropy,
multistage), restated so the `gen` / `bench` CLI subcommands build the same
instances the reference's `conic-ipm gen` / `conic-ipm bench` do (same seeds,
same draw order, same matrices: tests/test_io_cli.py pins them against hashes of
the reference's own output, tests/golden/families.json).

Reference: pkg/src/conic_ipm/generators.py:37-330 (GenSpec :49-75, portfolio
:78-111, huber :114-147, entropy :150-190, multistage :198-330).  The random
stream is numpy's Philox keyed by the seed (:37-38); sizes round half up
(:41-42).  Assembly here goes through COO triplets instead of the reference's
block stacking; the CSR is canonicalised the same way (sorted, duplicates summed).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .csr import CsrMatrix
from .exceptions import ConicError
from .model import ConeSpec, ProblemData

MULTISTAGE_COST = 1e-3
MULTISTAGE_GAMMA = 1.0
MULTISTAGE_INFLOW = 1.0
MULTISTAGE_BOX = 0.1

FAMILIES = ("portfolio", "huber", "entropy", "multistage")


class InfeasibleBoxBudget(ConicError):
    """The multistage budget cannot fit inside the allocation box (generators.py:33-34)."""


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=np.uint64(seed)))


def _round_half_up(x: float) -> int:
    return int(np.floor(x + 0.5))


class _Triplets:
    """Row-block builder: append (row, col, value) blocks and right-hand sides."""

    def __init__(self, ncols: int):
        self.ncols = ncols
        self.rows, self.cols, self.vals, self.rhs = [], [], [], []
        self.nrows = 0

    def add(self, r, c, v, nrows: int, rhs):
        self.rows.append(np.asarray(r, dtype=np.int64) + self.nrows)
        self.cols.append(np.asarray(c, dtype=np.int64))
        self.vals.append(np.asarray(v, dtype=np.float64))
        self.rhs.append(np.broadcast_to(np.asarray(rhs, dtype=np.float64), (nrows,)).copy())
        self.nrows += nrows

    def dense_block(self, mat, col0: int, rhs):
        mat = np.atleast_2d(np.asarray(mat, dtype=np.float64))
        r, c = np.nonzero(mat)
        self.add(r, c + col0, mat[r, c], mat.shape[0], rhs)

    def csr(self) -> tuple[CsrMatrix, np.ndarray]:
        r = np.concatenate(self.rows) if self.rows else np.zeros(0, dtype=np.int64)
        c = np.concatenate(self.cols) if self.cols else np.zeros(0, dtype=np.int64)
        v = np.concatenate(self.vals) if self.vals else np.zeros(0)
        mat = sp.coo_matrix((v, (r, c)), shape=(self.nrows, self.ncols))
        return CsrMatrix.from_scipy(mat), np.concatenate(self.rhs) if self.rhs else np.zeros(0)


def _diag_p(d: np.ndarray) -> CsrMatrix:
    return CsrMatrix.from_scipy(sp.diags(np.asarray(d, dtype=np.float64)))


def gen_portfolio(n: int, gamma: float = 1.0, seed: int = 0, mu=None, factor=None, dvec=None) -> ProblemData:
    """Factor-model portfolio QP over the simplex (generators.py:78-111): variables
    (x in R^n, y in R^p), min x'Dx + y'y - mu'x (scaled by gamma) s.t. 1'x = 1,
    F'x = y, x >= 0."""
    if n < 2:
        raise ValueError("portfolio requires n >= 2")
    rng = _rng(seed)
    p = max(1, _round_half_up(0.1 * n))
    f = rng.standard_normal((n, p))
    d = (1.0 - rng.random(n)) + 1e-3
    mu_v = 0.1 * rng.standard_normal(n)
    f = f if factor is None else np.asarray(factor, dtype=np.float64)
    d = d if dvec is None else np.asarray(dvec, dtype=np.float64)
    mu_v = mu_v if mu is None else np.asarray(mu, dtype=np.float64)
    p = f.shape[1]
    nv = n + p
    T = _Triplets(nv)
    T.add(np.zeros(n), np.arange(n), np.ones(n), 1, 1.0)                    # budget
    T.dense_block(np.hstack([f.T, -np.eye(p)]), 0, 0.0)                      # factor rows
    T.add(np.arange(n), np.arange(n), -np.ones(n), n, 0.0)                   # x >= 0
    A, b = T.csr()
    P = _diag_p(np.concatenate([2.0 * gamma * d, 2.0 * gamma * np.ones(p)]))
    q = np.concatenate([-mu_v, np.zeros(p)])
    return ProblemData(P, A, q, b, [ConeSpec("zero", 1 + p), ConeSpec("nonneg", n)])


def gen_huber(n: int, seed: int = 0, noise: float = 0.1, outlier_frac: float = 0.1) -> ProblemData:
    """Huber fitting QP, threshold 1, m = round(1.5 n) residuals (generators.py:114-147):
    variables (x, u, v), min u'u + 2 1'v s.t. |A x - b| <= u + v, v >= 0."""
    if n < 1:
        raise ValueError("huber requires n >= 1")
    rng = _rng(seed)
    m = _round_half_up(1.5 * n)
    a = rng.standard_normal((m, n))
    x_true = rng.standard_normal(n) / np.sqrt(n)
    eps = rng.standard_normal(m)
    sel = rng.random(m)
    mag = 2.0 * rng.random(m) - 1.0
    bv = a @ x_true + noise * eps
    bv = bv + np.where(sel < outlier_frac, 10.0 * mag, 0.0)
    nv = n + 2 * m
    I = np.arange(m)
    T = _Triplets(nv)
    for sign, rhs in ((1.0, bv), (-1.0, -bv)):
        r, c = np.nonzero(a)
        rr = np.concatenate([r, I, I])
        cc = np.concatenate([c, n + I, n + m + I])
        vv = np.concatenate([sign * a[r, c], -np.ones(m), -np.ones(m)])
        T.add(rr, cc, vv, m, rhs)
    T.add(I, n + m + I, -np.ones(m), m, 0.0)
    A, b = T.csr()
    P = _diag_p(np.concatenate([np.zeros(n), 2.0 * np.ones(m), np.zeros(m)]))
    q = np.concatenate([np.zeros(n + m), 2.0 * np.ones(m)])
    return ProblemData(P, A, q, b, [ConeSpec("nonneg", 3 * m)])


def gen_entropy(n: int, seed: int = 0, include_ineq: bool = True) -> ProblemData:
    """Entropy maximisation over the simplex (generators.py:150-190): variables
    (x, t), max sum t s.t. 1'x = 1, A x <= b, (t_i, x_i, 1) in K_exp."""
    if n < 2:
        raise ValueError("entropy requires n >= 2")
    rng = _rng(seed)
    m = _round_half_up(0.5 * n)
    a = np.sqrt(n) * rng.standard_normal((m, n))
    v = rng.random(n)
    b_ineq = a @ (v / np.sum(v))
    T = _Triplets(2 * n)
    T.add(np.zeros(n), np.arange(n), np.ones(n), 1, 1.0)
    cones = [ConeSpec("zero", 1)]
    if include_ineq:
        T.dense_block(a, 0, b_ineq)
        cones.append(ConeSpec("nonneg", m))
    i = np.arange(n)
    T.add(np.concatenate([3 * i, 3 * i + 1]), np.concatenate([n + i, i]), -np.ones(2 * n), 3 * n,
          np.tile([0.0, 0.0, 1.0], n))
    cones += [ConeSpec("exp", 3) for _ in range(n)]
    A, b = T.csr()
    P = CsrMatrix.from_scipy(sp.csr_matrix((2 * n, 2 * n)))
    q = np.concatenate([np.zeros(n), -np.ones(n)])
    return ProblemData(P, A, q, b, cones)


def gen_multistage_portfolio(n: int, k: int, periods: int, seed: int = 0) -> ProblemData:
    """Multistage portfolio SOCP (generators.py:198-330).  Per period t the
    variables are x_t (n), y_t (k), z_t (n), r_t; rows: budgets and y_t = F_t x_t
    (zero cone), trade volumes z_t >= |x_t - x_{t-1}| and boxes x, y in [0, 0.1]
    (nonneg), and the risk cone (r_t, U y_t, D x_t) per period."""
    if not (n >= k >= 1) or periods < 1:
        raise ValueError("multistage requires n >= k >= 1 and periods >= 1")
    rng = _rng(seed)
    x0 = rng.random(n)
    x0 = x0 / np.sum(x0)
    budget = MULTISTAGE_INFLOW + float(np.sum(x0))
    if MULTISTAGE_BOX * n < budget - 1e-9:
        raise InfeasibleBoxBudget(f"box capacity {MULTISTAGE_BOX * n:.3f} cannot hold budget {budget:.3f}")
    d_sqrt = 0.1 + rng.random(n)
    g = rng.standard_normal((k, k))
    u_fac = np.linalg.cholesky(g @ g.T / k + 1e-3 * np.eye(k)).T
    fs, mus = [], []
    for _ in range(periods):
        f_t = np.abs(rng.standard_normal((k, n)))
        fs.append(0.5 * f_t / f_t.sum(axis=1, keepdims=True))
        mus.append(rng.standard_normal(n))
    per = 2 * n + k + 1
    nv = periods * per
    X, Y, Z, R = (lambda t: t * per), (lambda t: t * per + n), (lambda t: t * per + n + k), \
        (lambda t: t * per + 2 * n + k)
    ii, kk = np.arange(n), np.arange(k)
    T = _Triplets(nv)
    # zero rows: one budget per period, then the k factor rows per period
    for t in range(periods):
        if t == 0:
            T.add(np.zeros(n), X(0) + ii, np.ones(n), 1, budget)
        else:
            T.add(np.zeros(2 * n), np.concatenate([X(t - 1) + ii, X(t) + ii]),
                  np.concatenate([-np.ones(n), np.ones(n)]), 1, 0.0)
    for t in range(periods):
        blk = np.zeros((k, nv))
        blk[:, X(t):X(t) + n] = fs[t]
        blk[:, Y(t):Y(t) + k] = -np.eye(k)
        T.dense_block(blk, 0, 0.0)
    zero_rows = periods * (1 + k)
    # nonneg rows: trade volumes (up, down) per period, then the boxes
    for t in range(periods):
        for sx in (1.0, -1.0):
            cols = [X(t) + ii, Z(t) + ii]
            vals = [sx * np.ones(n), -np.ones(n)]
            if t > 0:
                cols.append(X(t - 1) + ii)
                vals.append(-sx * np.ones(n))
            T.add(np.tile(ii, len(cols)), np.concatenate(cols), np.concatenate(vals), n,
                  sx * x0 if t == 0 else 0.0)
    for t in range(periods):
        T.add(ii, X(t) + ii, -np.ones(n), n, 0.0)
        T.add(ii, X(t) + ii, np.ones(n), n, MULTISTAGE_BOX)
        T.add(kk, Y(t) + kk, -np.ones(k), k, 0.0)
        T.add(kk, Y(t) + kk, np.ones(k), k, MULTISTAGE_BOX)
    nonneg_rows = periods * (2 * n) + periods * (2 * n + 2 * k)
    # risk cones
    for t in range(periods):
        blk = np.zeros((n + k + 1, nv))
        blk[0, R(t)] = -1.0
        blk[1:k + 1, Y(t):Y(t) + k] = -u_fac
        blk[k + 1:, X(t):X(t) + n] = -np.diag(d_sqrt)
        T.dense_block(blk, 0, 0.0)
    A, b = T.csr()
    q = np.zeros(nv)
    for t in range(periods):
        q[X(t):X(t) + n] = -mus[t]
        q[Z(t):Z(t) + n] = MULTISTAGE_COST
        q[R(t)] = MULTISTAGE_GAMMA
    P = CsrMatrix.from_scipy(sp.csr_matrix((nv, nv)))
    cones = [ConeSpec("zero", zero_rows), ConeSpec("nonneg", nonneg_rows)]
    cones += [ConeSpec("soc", n + k + 1) for _ in range(periods)]
    return ProblemData(P, A, q, b, cones)


@dataclass(frozen=True)
class GenSpec:
    """One benchmark instance request (generators.py:49-75)."""

    family: str
    n: int
    seed: int
    k: int = 0
    periods: int = 0
    gamma: float = 1.0

    def build(self) -> ProblemData:
        if self.family == "portfolio":
            return gen_portfolio(self.n, self.gamma, self.seed)
        if self.family == "huber":
            return gen_huber(self.n, self.seed)
        if self.family == "entropy":
            return gen_entropy(self.n, self.seed)
        if self.family == "multistage":
            return gen_multistage_portfolio(self.n, self.k, self.periods, self.seed)
        raise ValueError(f"unknown family {self.family!r}")

    @property
    def name(self) -> str:
        if self.family == "multistage":
            return f"multistage_n{self.n}_k{self.k}_T{self.periods}_s{self.seed}"
        return f"{self.family}_n{self.n}_s{self.seed}"
