"""Batched independent instances on one GPU (C5b).

``BatchSolver(problems, settings).solve()`` solves many problems that share
one sparsity pattern (e.g. the MPC QPs of the paper's §4.6, or one parametric
family) and returns one reference-compatible ``SolveResult`` per instance —
the same results the reference produces when it runs ``Solver(p).solve()``
for each instance (its ``bench --jobs`` mode, bench.py:98-113).

Host side (once per batch): validation, cone reordering and a Ruiz
equilibration vectorised across instances (bitwise the per-instance
``model.equilibrate``), then ONE launch of the device kernel in which each CTA
runs one instance's whole Algorithm-1 loop (csrc/batch.cu).  Multi-GPU:
one process per GPU, each with its own contiguous shard of instances and no
collective on the solve path (bench.py --config c5b_mpc under torchrun).

Scope: zero + nonnegative cones (LP/QP), full precision.
"""
from __future__ import annotations

import ctypes
import time
from collections.abc import Sequence

import numpy as np

from .exceptions import ConicError, NonFiniteData, PatternMismatch, raise_for_status
from .model import NONNEG, SCALE_MAX, SCALE_MIN, ZERO, ProblemData, max_abs, reorder_cones, validate
from .native import Layout, Settings, c_void_p, lib, make_desc, pdbl, pi64, pinned_copy, pinned_empty, require_device
from .settings import FULL, SolveResult, SolverSettings, Status, default_dynamic_reg, default_static_reg

RUIZ_ITERS = 10
_STATUS = {0: Status.OPTIMAL, 1: Status.PRIMAL_INFEASIBLE, 2: Status.DUAL_INFEASIBLE, 3: Status.ALMOST_OPTIMAL,
           4: Status.MAX_ITERATIONS, 6: Status.INSUFFICIENT_PROGRESS, 7: Status.NUMERICAL_ERROR}


def _rows(rowptr):
    return np.repeat(np.arange(len(rowptr) - 1, dtype=np.int64), np.diff(rowptr))


def equilibrate_batch(P, A, pv, av, q, b, iters=RUIZ_ITERS):
    """Ruiz equilibration of B instances at once (problem.py:222-284 restated on
    (B, nnz) arrays; zero + nonneg cones so there is no block-uniform step).
    Elementwise identical to ``model.equilibrate`` per instance."""
    B, n, m = q.shape[0], P.nrows, A.nrows
    p_rows, p_cols = _rows(P.rowptr), P.colidx
    a_rows, a_cols = _rows(A.rowptr), A.colidx
    pv, av, qc, bc = pv.copy(), av.copy(), q.copy(), b.copy()
    d_col = np.ones((B, n))
    d_row = np.ones((B, m))
    inst_p = np.arange(B)[:, None]
    for _ in range(iters):
        cnorm = np.zeros((B, n))
        if pv.shape[1]:
            np.maximum.at(cnorm, (np.broadcast_to(inst_p, pv.shape), np.broadcast_to(p_cols, pv.shape)), np.abs(pv))
        if av.shape[1]:
            np.maximum.at(cnorm, (np.broadcast_to(inst_p, av.shape), np.broadcast_to(a_cols, av.shape)), np.abs(av))
        rnorm = np.zeros((B, m))
        if av.shape[1]:
            np.maximum.at(rnorm, (np.broadcast_to(inst_p, av.shape), np.broadcast_to(a_rows, av.shape)), np.abs(av))
        cstep = np.where(cnorm > 0, 1.0 / np.sqrt(np.where(cnorm > 0, cnorm, 1.0)), 1.0)
        rstep = np.where(rnorm > 0, 1.0 / np.sqrt(np.where(rnorm > 0, rnorm, 1.0)), 1.0)
        new_dcol = np.clip(d_col * cstep, SCALE_MIN, SCALE_MAX)
        new_drow = np.clip(d_row * rstep, SCALE_MIN, SCALE_MAX)
        cstep = new_dcol / d_col
        rstep = new_drow / d_row
        d_col, d_row = new_dcol, new_drow
        pv = (cstep[:, p_rows] * pv) * cstep[:, p_cols]
        av = (rstep[:, a_rows] * av) * cstep[:, a_cols]
        qc *= cstep
        bc *= rstep
    qmax = np.max(np.abs(qc), axis=1) if n else np.zeros(B)
    c_obj = np.where(qmax == 0.0, 1.0, np.clip(1.0 / np.where(qmax == 0.0, 1.0, qmax), SCALE_MIN, SCALE_MAX))
    pv = pv * c_obj[:, None]
    qc = qc * c_obj[:, None]
    return pv, av, qc, bc, d_row, d_col, c_obj


class BatchResults(Sequence):
    """The per-instance results of one batched solve: a sequence of reference
    ``SolveResult`` objects backed by the host arrays of one device-to-host copy.
    Each ``SolveResult`` is built when it is first accessed; whole-batch columns
    (``status``, ``iterations``, ``obj_primal``, ``obj_dual``, ``x``, ``z``, ``s``)
    are available as arrays without building them."""

    def __init__(self, status_codes, res, x, z, s, q, b, setup_seconds, solve_seconds):
        self._codes, self._res, self.x, self.z, self.s = status_codes, res, x, z, s
        self._q, self._b = q, b
        self._setup, self._secs = setup_seconds, solve_seconds
        self._cache: dict = {}

    def __len__(self) -> int:
        return len(self._codes)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        r = self._cache.get(k)
        if r is None:
            r = self._cache[k] = self._build(k)
        return r

    @property
    def status(self) -> list:
        return [_STATUS[v] for v in self._codes.tolist()]

    @property
    def iterations(self) -> np.ndarray:
        return self._res[:, 8].astype(np.int64)

    @property
    def obj_primal(self) -> np.ndarray:
        return self._res[:, 0]

    @property
    def obj_dual(self) -> np.ndarray:
        return self._res[:, 1]

    def _build(self, k: int) -> SolveResult:
        st = _STATUS[int(self._codes[k])]
        g_p, g_d, rp, rd, tau, kappa, mu, mu0, iters = self._res[k].tolist()
        # the device returned unscaled, user-row-order iterates (divided by tau unless a certificate)
        x_o, z_o, s_o = self.x[k], self.z[k], self.s[k]
        cert = None
        if st == Status.PRIMAL_INFEASIBLE:
            cert = z_o / abs(float(self._b[k] @ z_o))
        elif st == Status.DUAL_INFEASIBLE:
            cert = x_o / abs(float(self._q[k] @ x_o))
        return SolveResult(status=st, x=x_o, z=z_o, s=s_o, certificate=cert, obj_primal=g_p, obj_dual=g_d,
                           iterations=int(iters), setup_seconds=self._setup, solve_seconds=self._secs,
                           norm_rp=rp, norm_rd=rd, gap=abs(g_p - g_d), tau=tau, kappa=kappa, mu_initial=mu0,
                           mu_final=mu)


class BatchSolver:
    """Many same-pattern instances, one device launch (one CTA per instance)."""

    def __init__(self, problems, settings: SolverSettings | None = None, device: int = 0):
        if not problems:
            raise ConicError("empty batch")
        self.settings = st = settings or SolverSettings()
        if st.precision != FULL:
            raise ConicError("batched instances run the full-precision factorisation")
        torch = require_device()
        torch.cuda.set_device(device)
        t0 = time.perf_counter()
        first = problems[0]
        for p in problems:
            validate(p)
            if not (np.array_equal(p.P.rowptr, first.P.rowptr) and np.array_equal(p.P.colidx, first.P.colidx)
                    and np.array_equal(p.A.rowptr, first.A.rowptr) and np.array_equal(p.A.colidx, first.A.colidx)
                    and list(p.cones) == list(first.cones)):
                raise PatternMismatch("batched instances must share one sparsity pattern and cone list")
        if any(c.kind not in (ZERO, NONNEG) for c in first.cones):
            raise ConicError("batched instances support zero + nonnegative cones only")
        self.problems = [p.copy() for p in problems]
        self.count = len(problems)
        # current q / b of every instance (user row order); update_data replaces them
        self._q_cur = np.stack([p.q for p in self.problems])
        self._b_cur = np.stack([p.b for p in self.problems])
        ref0, self._perm = reorder_cones(first)
        self._pattern = ref0
        self.layout = Layout(ref0.cones)
        self.n, self.m = ref0.n, ref0.m
        cs = Settings()
        cs.precision = 0
        cs.delta_s = default_static_reg(FULL) if st.delta_s is None else st.delta_s
        cs.delta_d = default_dynamic_reg(FULL) if st.delta_d is None else st.delta_d
        cs.beta, cs.backtrack, cs.step_scale = st.beta, st.backtrack, st.step_scale
        cs.refine_abs, cs.refine_rel, cs.refine_max = (st.refinement.t_abs, st.refinement.t_rel,
                                                       st.refinement.t_max)
        cs.device = device
        cs.stream = None
        self._desc, self._keep = make_desc(ref0.P, ref0.A, self.layout)
        h = c_void_p()
        rc = lib().cipm_batch_create(ctypes.byref(self._desc), self.count, ctypes.byref(cs), st.eps_feas,
                                     st.eps_inf, st.max_iter, ctypes.byref(h))
        raise_for_status(rc, "batch creation")
        self.handle = h
        self._upload()
        c, n, m = self.count, self.n, self.m             # warm torch's pinned host cache (see Solver)
        _warm = [pinned_empty(sh) for _ in range(3) for sh in ((c, n), (c, m), (c, n), (c, m), (c, m))]
        del _warm
        self.setup_seconds = time.perf_counter() - t0
        self.last_kernel_ms = 0.0

    def _upload(self):
        """Raw user-order arrays to the device; each instance's CTA reorders and
        Ruiz-equilibrates its own data (batch.cu, the reference's arithmetic)."""
        if not getattr(self, "_reorder_set", False):
            perm = np.ascontiguousarray(self._perm, dtype=np.int64)
            a_src = np.ascontiguousarray(_take_rows_src(self.problems[0].A, self._perm), dtype=np.int64)
            raise_for_status(lib().cipm_batch_set_reorder(self.handle, pi64(perm), pi64(a_src)), "batch reorder")
            self._reorder_set = True
        V = np.concatenate([np.stack([p.P.values for p in self.problems]),
                            np.stack([p.A.values for p in self.problems])], axis=1)
        self._host = [np.ascontiguousarray(a) for a in (V, self._q_cur, self._b_cur)]
        rc = lib().cipm_batch_set_raw_values(self.handle, *[pdbl(a) for a in self._host],
                                             1 if self.settings.do_equilibrate else 0)
        raise_for_status(rc, "batch upload")
        self._raw_on_device = True

    def _upload_host_equilibrated(self):
        """Alternative path: host reorder + vectorised Ruiz (equilibrate_batch), scaled upload."""
        perm = self._perm
        P, A = self._pattern.P, self._pattern.A
        a_src = _take_rows_src(self.problems[0].A, perm)
        pv = np.stack([p.P.values for p in self.problems])
        av = np.stack([p.A.values[a_src] for p in self.problems])
        q = self._q_cur
        b = self._b_cur[:, perm]
        norm_q = np.max(np.abs(q), axis=1) if self.n else np.zeros(self.count)
        norm_b = np.max(np.abs(b), axis=1) if self.m else np.zeros(self.count)
        pv_s, av_s, q_s, b_s, d_row, d_col, c_obj = equilibrate_batch(P, A, pv, av, q, b)
        self._host = [np.ascontiguousarray(a) for a in
                      (np.concatenate([pv_s, av_s], axis=1), q_s, b_s, d_row, d_col, c_obj, norm_q, norm_b)]
        rc = lib().cipm_batch_set_values(self.handle, *[pdbl(a) for a in self._host])
        raise_for_status(rc, "batch upload")
        self._raw_on_device = False

    def update_data(self, q=None, b=None):
        """Parametric re-solve of every instance (same patterns): q, b as (count, n) / (count, m).
        Only the given arrays are sent; the device keeps the raw P / A values."""
        qs = np.asarray(q, dtype=np.float64) if q is not None else None
        bs = np.asarray(b, dtype=np.float64) if b is not None else None
        if qs is not None and qs.shape != (self.count, self.n):
            raise ValueError(f"q must be ({self.count}, {self.n})")
        if bs is not None and bs.shape != (self.count, self.m):
            raise ValueError(f"b must be ({self.count}, {self.m})")
        # the reference's update_data re-validates (problem.py:149-174): non-finite data raises
        if qs is not None and not np.isfinite(max_abs(qs)):
            raise NonFiniteData("q")
        if bs is not None and not np.isfinite(max_abs(bs)):
            raise NonFiniteData("b")
        # own page-locked copies: the H2D is one DMA, and they back the results' certificates
        if qs is not None:
            self._q_cur = pinned_copy(qs)
        if bs is not None:
            self._b_cur = pinned_copy(bs)
        if not getattr(self, "_raw_on_device", True):
            self._upload()                  # after a host-equilibrated upload: re-send the raw arrays
            return
        rc = lib().cipm_batch_set_raw_values(self.handle, None, pdbl(qs) if qs is not None else None,
                                             pdbl(bs) if bs is not None else None,
                                             1 if self.settings.do_equilibrate else 0)
        raise_for_status(rc, "batch upload")

    def info(self) -> dict:
        out = np.zeros(9, dtype=np.int64)
        raise_for_status(lib().cipm_batch_info(self.handle, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return dict(zip(("count", "n", "m", "nnz_l", "smem_bytes", "in_smem", "cta_factor", "root_width", "groups"),
                        (int(v) for v in out)))

    def run(self) -> float:
        """Device solve of every instance; returns the CUDA-event time (ms)."""
        ms = ctypes.c_double(0.0)
        raise_for_status(lib().cipm_batch_solve(self.handle, ctypes.byref(ms)), "batch solve")
        self.last_kernel_ms = ms.value
        return ms.value

    def results(self, secs: float | None = None):
        c, n, m = self.count, self.n, self.m
        status = np.zeros(c, dtype=np.int32)
        res = np.zeros((c, 9))
        x, z, s = pinned_empty((c, n)), pinned_empty((c, m)), pinned_empty((c, m))   # D2H by DMA
        raise_for_status(lib().cipm_batch_results(self.handle, status.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                                  pdbl(res), pdbl(x), pdbl(z), pdbl(s)), "batch results")
        secs = self.last_kernel_ms / 1e3 if secs is None else secs
        return BatchResults(status, res, x, z, s, self._q_cur, self._b_cur, self.setup_seconds, secs)

    def solve(self):
        t0 = time.perf_counter()
        self.run()
        return self.results(time.perf_counter() - t0)

    def close(self):
        if getattr(self, "handle", None):
            lib().cipm_batch_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _take_rows_src(A, rows):
    rows = np.asarray(rows, dtype=np.int64)
    counts = A.rowptr[rows + 1] - A.rowptr[rows]
    rp = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    if not rp[-1]:
        return np.zeros(0, dtype=np.int64)
    return np.repeat(A.rowptr[rows] - rp[:-1], counts) + np.arange(rp[-1], dtype=np.int64)


def _user_rows(v, perm):
    out = np.empty_like(v)
    out[perm] = v
    return out


def _pattern_key(p: ProblemData):
    """Instances with equal keys share one sparsity pattern and cone list."""
    return (p.n, p.m, p.P.rowptr.tobytes(), p.P.colidx.tobytes(), p.A.rowptr.tobytes(), p.A.colidx.tobytes(),
            tuple((c.kind, c.dim, c.alpha, c.side) for c in p.cones))


def solve_many(problems, settings: SolverSettings | None = None, device: int = 0):
    """Solve a heterogeneous list of problems on one GPU: instances are grouped by
    sparsity pattern and cone list; each group of zero / nonneg (LP / QP) instances
    in full precision runs as one ``BatchSolver`` launch (a CTA per instance), every
    other instance (SOC / exp / pow / PSD cones, mixed precision, singletons) through
    the single-problem device path.  Returns the ``SolveResult`` list in input
    order — what ``Solver(p).solve()`` returns for each instance."""
    from .solver import Solver
    st = settings or SolverSettings()
    groups: dict = {}
    for k, p in enumerate(problems):
        groups.setdefault(_pattern_key(p), []).append(k)
    out = [None] * len(problems)
    for idx in groups.values():
        first = problems[idx[0]]
        batchable = (len(idx) > 1 and st.precision == FULL
                     and all(c.kind in (ZERO, NONNEG) for c in first.cones))
        if batchable:
            bs = BatchSolver([problems[k] for k in idx], st, device=device)
            try:
                for k, r in zip(idx, bs.solve()):
                    out[k] = r
            finally:
                bs.close()
            continue
        for k in idx:
            s = Solver(problems[k], st)
            try:
                out[k] = s.solve()
            finally:
                s.close()
    return out
