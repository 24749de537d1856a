"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product path).

CPU restatement of the reference KKT system (kkt/system.py:64-321): the
upper-triangle pattern of K = [P A'; A -H] with slots for every scaling
entry, the one-time symbolic analysis (minimum degree, permuted upper CSC,
gather map, signs, etree, column counts), the regularised numeric LDL' and
iterative refinement against the unregularised full-precision K.  The
sequential kernels run in ``ldl_oracle.c`` (restating kkt/ldl.py and
kkt/ordering.py); the pattern build is vectorised numpy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2412_19027_b200.exceptions import ConicError, FactorizationFailure
from paper_2412_19027_b200.settings import (FULL, RefinementSettings, default_dynamic_reg,
                                            default_static_reg)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_ldl.so")
_lib = None


def build_oracle_lib(force: bool = False) -> str:
    src = os.path.join(HERE, "ldl_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_oracle_lib()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_min_degree.argtypes = [i64, P, P, P]
        L.oracle_min_degree.restype = ctypes.c_int
        L.oracle_ldl_symbolic.argtypes = [i64, P, P, P, P, P]
        for nm, ft in (("oracle_ldl_numeric_f64", ctypes.c_double), ("oracle_ldl_numeric_f32", ctypes.c_float)):
            f = getattr(L, nm)
            f.argtypes = [i64] + [P] * 13 + [ft, ft]
            f.restype = i64
        L.oracle_ldl_solve_f64.argtypes = [i64, P, P, P, P, P]
        L.oracle_ldl_solve_f32.argtypes = [i64, P, P, P, P, P]
        L.oracle_symm_matvec.argtypes = [i64, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class RefineOutcome:
    x: np.ndarray
    steps: int
    stalled: bool
    residual: float


class OracleKKT:
    """KKT matrix with reusable symbolic factorisation (reference KKTSystem)."""

    def __init__(self, P, A, lay, precision=FULL, delta_s=None, delta_d=None):
        self.n, self.m = P.nrows, A.nrows
        self.dim = self.n + self.m
        self.precision = precision
        self.delta_s = default_static_reg(precision) if delta_s is None else delta_s
        self.delta_d = default_dynamic_reg(precision) if delta_d is None else delta_d
        self.num_symbolic = 0
        self.num_numeric = 0
        self._fresh = False
        self._build_pattern(P, A, lay)
        self.set_matrices(P, A)
        self._symbolic_done = False

    # pattern: upper triangle of [P A'; A -H] with H slots (system.py:87-148)
    def _build_pattern(self, P, A, lay):
        n, m, dim = self.n, self.m, self.dim
        p_rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(P.rowptr))
        p_upper = P.colidx >= p_rows
        a_rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(A.rowptr))
        lin = lay.zero_dim + lay.nonneg_dim
        r_parts = [np.arange(n), p_rows[p_upper], A.colidx, n + np.arange(lin)]
        c_parts = [np.arange(n), P.colidx[p_upper], n + a_rows, n + np.arange(lin)]
        self._blocks = list(lay.blocks())
        for off, d in self._blocks:
            iu, ju = np.triu_indices(d)
            r_parts.append(n + off + iu)
            c_parts.append(n + off + ju)
        rr = np.concatenate(r_parts).astype(np.int64)
        cc = np.concatenate(c_parts).astype(np.int64)
        key = np.unique(rr * dim + cc)
        rows = key // dim
        self.colidx = key % dim
        self.rowptr = np.zeros(dim + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=dim), out=self.rowptr[1:])
        self.values = np.zeros(len(key))

        def slot(r, c):
            return np.searchsorted(key, r * dim + c)

        self._p_src = np.nonzero(p_upper)[0]
        self._p_dst = slot(p_rows[p_upper], P.colidx[p_upper])
        self._a_map = slot(A.colidx, n + a_rows)
        self._hdiag = slot(n + np.arange(lin), n + np.arange(lin))
        self._hblock = []
        for off, d in self._blocks:
            iu, ju = np.triu_indices(d)
            self._hblock.append((slot(n + off + iu, n + off + ju), iu, ju))
        self._p_pattern = (P.rowptr.copy(), P.colidx.copy())
        self._a_pattern = (A.rowptr.copy(), A.colidx.copy())

    def set_matrices(self, P=None, A=None):
        if P is not None:
            self.values[self._p_dst] = P.values[self._p_src]
        if A is not None:
            self.values[self._a_map] = A.values
        self._fresh = False

    def set_scaling(self, diag, blocks):
        self.values[self._hdiag] = -diag
        for (slots, iu, ju), (_, blk) in zip(self._hblock, blocks):
            self.values[slots] = -blk[iu, ju]
        self._fresh = False

    # symbolic analysis (system.py:188-240)
    def symbolic_factor(self, perm=None):
        """``perm`` (test hook) replaces the minimum-degree order, e.g. to probe
        ordering sensitivity as in SURVEY.md §8(c)."""
        if self._symbolic_done:
            return
        L = lib()
        dim = self.dim
        if perm is None:
            perm = np.empty(dim, dtype=np.int64)
            if L.oracle_min_degree(dim, _p(self.rowptr), _p(self.colidx), _p(perm)) != 0:
                raise MemoryError("oracle min-degree allocation failed")
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        iperm = np.empty(dim, dtype=np.int64)
        iperm[perm] = np.arange(dim, dtype=np.int64)
        self.perm, self.iperm = perm, iperm
        rows = np.repeat(np.arange(dim, dtype=np.int64), np.diff(self.rowptr))
        pi, pj = iperm[rows], iperm[self.colidx]
        r = np.minimum(pi, pj)
        c = np.maximum(pi, pj)
        order = np.lexsort((r, c))
        self._ci = np.ascontiguousarray(r[order])
        self._gather = np.ascontiguousarray(order.astype(np.int64))
        self._cp = np.zeros(dim + 1, dtype=np.int64)
        np.cumsum(np.bincount(c, minlength=dim), out=self._cp[1:])
        diag_pos = np.nonzero(r[order] == c[order])[0]
        self._static_pos = np.empty(dim, dtype=np.int64)
        self._static_pos[c[order][diag_pos]] = diag_pos
        self._signs = np.where(perm < self.n, 1, -1).astype(np.int8)
        self._parent = np.empty(dim, dtype=np.int64)
        lnz = np.empty(dim, dtype=np.int64)
        self._flag = np.empty(dim, dtype=np.int64)
        L.oracle_ldl_symbolic(dim, _p(self._cp), _p(self._ci), _p(self._parent), _p(lnz), _p(self._flag))
        self._lp = np.zeros(dim + 1, dtype=np.int64)
        np.cumsum(lnz, out=self._lp[1:])
        self._li = np.empty(int(self._lp[-1]), dtype=np.int64)
        self._lnz_count = np.empty(dim, dtype=np.int64)
        self._pattern = np.empty(dim, dtype=np.int64)
        dt = self.dtype
        self._lx = np.empty(int(self._lp[-1]), dtype=dt)
        self._d = np.empty(dim, dtype=dt)
        self._y = np.zeros(dim, dtype=dt)
        self.num_symbolic += 1
        self._symbolic_done = True

    @property
    def dtype(self):
        return np.float64 if self.precision == FULL else np.float32

    @property
    def nnz_l(self) -> int:
        return int(self._lp[-1])

    def numeric_factor(self):
        if not self._symbolic_done:
            self.symbolic_factor()
        dt = self.dtype
        src = self.values if self.precision == FULL else self.values.astype(np.float32)
        cx = src[self._gather].astype(dt, copy=True)
        cx[self._static_pos] += (self._signs * dt(self.delta_s)).astype(dt)
        L = lib()
        fn = L.oracle_ldl_numeric_f64 if dt == np.float64 else L.oracle_ldl_numeric_f32
        st = fn(self.dim, _p(self._cp), _p(self._ci), _p(cx), _p(self._lp), _p(self._parent),
                _p(self._lnz_count), _p(self._li), _p(self._lx), _p(self._d), _p(self._y),
                _p(self._pattern), _p(self._flag), _p(self._signs), dt(self.delta_s), dt(self.delta_d))
        if st < 0:
            raise FactorizationFailure("zero pivot after regularization")
        self.last_bumped_pivots = int(st)
        self.num_numeric += 1
        self._fresh = True

    def factor_solve(self, rhs):
        dt = self.dtype
        xp = np.ascontiguousarray(rhs[self.perm].astype(dt, copy=True))
        fn = lib().oracle_ldl_solve_f64 if dt == np.float64 else lib().oracle_ldl_solve_f32
        fn(self.dim, _p(self._lp), _p(self._li), _p(self._lx), _p(self._d), _p(xp))
        out = np.empty(self.dim)
        out[self.perm] = xp.astype(np.float64)
        return out

    def matvec(self, x):
        out = np.empty(self.dim)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        lib().oracle_symm_matvec(self.dim, _p(self.rowptr), _p(self.colidx), _p(self.values),
                                 _p(xx), _p(out))
        return out

    def solve_refined(self, b, st: RefinementSettings | None = None) -> RefineOutcome:
        """Iterative refinement (system.py:279-314)."""
        if not self._fresh:
            raise ConicError("numeric factorization is stale; call numeric_factor first")
        st = st or RefinementSettings()
        target = st.t_abs + st.t_rel * (float(np.max(np.abs(b))) if len(b) else 0.0)
        x = np.zeros(self.dim)
        r = b.copy()
        best_x, best = x.copy(), np.inf
        prev = np.inf
        ups = 0
        for step in range(1, st.t_max + 1):
            x = x + self.factor_solve(r)
            r = b - self.matvec(x)
            rn = float(np.max(np.abs(r))) if len(r) else 0.0
            if rn < best:
                best_x, best = x.copy(), rn
            if rn <= target:
                return RefineOutcome(x, step, False, rn)
            if rn > prev:
                ups += 1
                if ups >= 2:
                    return RefineOutcome(best_x, step, True, best)
            else:
                ups = 0
            prev = rn
        return RefineOutcome(best_x, st.t_max, False, best)
