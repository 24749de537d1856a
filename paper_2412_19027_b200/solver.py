"""B200 drop-in for the reference ``conic_ipm.ipm`` (Solver / solve).

The host keeps the reference's control flow (``pkg/src/conic_ipm/ipm.py``):
setup (validate → reorder → equilibrate → KKT symbolic analysis, ipm.py:150-171),
then the Algorithm-1 loop (ipm.py:411-496) with identical termination,
infeasibility, stall, best-iterate and recovery rules.  Every per-iteration
vector operation runs on the GPU through the C ABI (``include/cipm.h``); the
host only sees the scalar block (one read per iteration plus the reads the
refinement / backtracking decisions need).

There is no CPU fallback: constructing a Solver without the native library or
without a CUDA device raises.
"""
from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np

from .exceptions import ConicError, DeviceError, PatternMismatch
from .model import (Equilibration, ProblemData, csr_row_gather_src, max_abs, reorder_cones, validate,
                    validate_values)
from .native import (P_I64, SC, DeviceContext, Layout, Settings, SymbolicAnalysis, pdbl, pi64, pinned_copy,
                     pinned_empty, require_device)
from .settings import (ALMOST_OPTIMAL_FACTOR, FULL, MIXED, STALL_IMPROVEMENT, STALL_WINDOW, SolveResult,
                       SolverSettings, Status, default_dynamic_reg, default_static_reg)


@dataclass
class Residuals:
    """Unscaled residuals, objectives and norms (reference ipm.py:98-114).  The loop
    only needs the norms (fused device reductions); r_p / r_d are filled by
    Solver.compute_residuals, which fetches the residual vectors."""

    g_p: float
    g_d: float
    norm_rp: float
    norm_rd: float
    norm_xbar: float
    norm_sbar: float
    norm_zbar: float
    r_p: np.ndarray | None = None
    r_d: np.ndarray | None = None

    @property
    def gap(self) -> float:
        return abs(self.g_p - self.g_d)


@dataclass
class IterateState:
    x: np.ndarray
    z: np.ndarray
    s: np.ndarray
    tau: float
    kappa: float
    mu: float

    @property
    def xi(self) -> np.ndarray:
        return self.x / self.tau

    def copy(self) -> "IterateState":
        return IterateState(self.x.copy(), self.z.copy(), self.s.copy(), self.tau, self.kappa, self.mu)


class DeviceScaling:
    """Observer view of the scaling state (reference ScalingState subset: kkt_values / dense)."""

    def __init__(self, solver: "Solver"):
        self._solver = solver
        lay = solver.layout
        lin = lay.zero_dim + lay.nonneg_dim
        ctx = solver._ctx
        nn_h = solver._vector("nn_h")
        self.diag = np.zeros(lin)
        self.diag[lay.zero_dim:] = nn_h
        hv = solver._vector("hv")
        self.blocks = []
        k = 0
        for off, d in solver._block_list():
            iu, ju = np.triu_indices(d)
            blk = np.zeros((d, d))
            cnt = d * (d + 1) // 2
            blk[iu, ju] = hv[k:k + cnt]
            blk[ju, iu] = hv[k:k + cnt]
            k += cnt
            self.blocks.append((off, blk))
        del ctx

    def kkt_values(self):
        return self.diag, self.blocks

    def dense(self) -> np.ndarray:
        m = self._solver.layout.m
        h = np.zeros((m, m))
        h[np.arange(len(self.diag)), np.arange(len(self.diag))] = self.diag
        for off, blk in self.blocks:
            d = blk.shape[0]
            h[off:off + d, off:off + d] = blk
        return h


class DeviceKKT:
    """Counters of the device KKT system (reference KKTSystem, kkt/system.py:78-79,
    239, 261-262).  num_symbolic counts host symbolic analyses of this Solver (one:
    update_data reuses it); num_numeric and last_bumped_pivots come from the device."""

    def __init__(self, solver: "Solver"):
        self._solver = solver
        self.num_symbolic = 0
        self.precision = solver.settings.precision

    def _counters(self):
        out = np.zeros(2, dtype=np.int64)
        self._solver._ctx.call("cipm_kkt_counters", pi64(out))
        return out

    @property
    def num_numeric(self) -> int:
        return int(self._counters()[0])

    @property
    def last_bumped_pivots(self) -> int:
        return int(self._counters()[1])

    @property
    def dim(self) -> int:
        return self._solver.n + self._solver.m


class Solver:
    """One problem instance: setup once on the host + GPU, solve and re-solve."""

    def __init__(self, problem: ProblemData, settings: SolverSettings | None = None, device: int = 0,
                 ordering: int = 3, nd_leaf: int = 0):
        self.settings = settings or SolverSettings()
        torch = require_device()
        self.device = device
        t0 = time.perf_counter()
        validate(problem)
        self._original = problem.copy()
        reordered, perm = reorder_cones(problem)
        self._perm = perm
        self._reordered = reordered          # pattern of the reordered problem (values: user order on the device)
        self.layout = Layout(reordered.cones)
        self.nu = self.layout.degree
        self.n, self.m = reordered.n, reordered.m
        # ordering (not a reference setting): 3 = auto, see native.SymbolicAnalysis
        self.symbolic = SymbolicAnalysis(reordered.P, reordered.A, self.layout, ordering=ordering, nd_leaf=nd_leaf)
        self.kkt = DeviceKKT(self)
        self.kkt.num_symbolic += 1          # the only symbolic analysis of this Solver (system.py:239)
        st = self.settings
        prec = st.precision
        cs = Settings()
        cs.precision = 0 if prec == FULL else 1
        cs.delta_s = default_static_reg(prec) if st.delta_s is None else st.delta_s
        cs.delta_d = default_dynamic_reg(prec) if st.delta_d is None else st.delta_d
        if prec == MIXED:
            # the reference casts δ to float32 before use (system.py:253-258)
            cs.delta_s = float(np.float32(cs.delta_s))
            cs.delta_d = float(np.float32(cs.delta_d))
        cs.beta, cs.backtrack, cs.step_scale = st.beta, st.backtrack, st.step_scale
        cs.refine_abs, cs.refine_rel, cs.refine_max = (st.refinement.t_abs, st.refinement.t_rel,
                                                       st.refinement.t_max)
        cs.device = device
        cs.stream = None
        torch.cuda.set_device(device)
        self._ctx = DeviceContext(self.symbolic, cs)
        # reorder maps once: reordered row i <- user row perm[i]; reordered A nonzero k <- user nonzero
        self._row_perm = np.ascontiguousarray(perm, dtype=np.int64)
        self._a_src = np.ascontiguousarray(csr_row_gather_src(problem.A, perm), dtype=np.int64)
        self._ctx.call("cipm_ctx_set_reorder", pi64(self._row_perm) or P_I64(), pi64(self._a_src) or P_I64())
        self._upload_values()
        # page-locked blocks for the parametric updates (q, b) and the results (x, z, s)
        # in torch's host cache (three generations alive at once: the current data and
        # results, the next ones, slack), so no solve pays for pinning them
        _warm = [pinned_empty(k) for _ in range(3) for k in (self.n, self.m, self.n, self.m, self.m)]
        del _warm
        self.setup_seconds = time.perf_counter() - t0
        self._sc = np.zeros(64)
        self.last_refine_steps = []

    # -- data plumbing --------------------------------------------------------

    def _upload_values(self, changed=(True, True, True, True)):
        """Raw user-order values to the device; cone reordering and Ruiz equilibration
        run there (setup.cu, bitwise the reference's problem.py:177-284 arithmetic).
        Arrays flagged unchanged (P, A, q, b) are not re-sent: the device keeps the
        previous raw values."""
        prob = self._original
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (prob.P.values, prob.A.values, prob.q, prob.b)]
        k = [pdbl(a) if ch else None for a, ch in zip(self._keep, changed)]
        self._ctx.call("cipm_ctx_set_problem", k[0], k[1], k[2], k[3],
                       1 if self.settings.do_equilibrate else 0)
        # only the scalar c is needed per iteration; D_r / D_c are fetched when a
        # result is recovered (_scaling), not on every parametric update
        c_obj = ctypes.c_double(1.0)
        self._ctx.call("cipm_ctx_get_equilibration", None, None, ctypes.byref(c_obj))
        self._equil = Equilibration(None, None, float(c_obj.value))
        # termination norms use the reordered unscaled data (ipm.py:184-185); max is order-free
        self._norm_q = max_abs(prob.q)
        self._norm_b = max_abs(prob.b)

    def update_data(self, P=None, A=None, q=None, b=None) -> None:
        """Parametric re-solve (reference ipm.py:187-221): same patterns, fresh
        equilibration, value-only upload; the symbolic analysis is reused.  Only
        the changed arrays are re-validated (the patterns are checked equal)."""
        prob = self._original
        if P is not None:
            if not (np.array_equal(P.rowptr, prob.P.rowptr) and np.array_equal(P.colidx, prob.P.colidx)):
                raise PatternMismatch("P pattern differs from the setup pattern")
        if A is not None:
            if not (np.array_equal(A.rowptr, prob.A.rowptr) and np.array_equal(A.colidx, prob.A.colidx)):
                raise PatternMismatch("A pattern differs from the setup pattern")
        if q is not None and len(q) != prob.n:
            raise PatternMismatch("q length changed")
        if b is not None and len(b) != prob.m:
            raise PatternMismatch("b length changed")
        new = ProblemData(P.copy() if P is not None else prob.P, A.copy() if A is not None else prob.A,
                          pinned_copy(q) if q is not None else prob.q,
                          pinned_copy(b) if b is not None else prob.b, prob.cones)
        validate_values(new, P is not None, A is not None, q is not None, b is not None)
        self._original = new
        self._upload_values((P is not None, A is not None, q is not None, b is not None))

    def _block_list(self):
        lay = self.layout
        out = [(int(o), int(d)) for o, d in zip(lay.soc_off, lay.soc_dim)]
        out += [(int(o), 3) for o in lay.exp_off]
        out += [(int(o), 3) for o in lay.pow_off]
        out += [(int(o), int(s) * (int(s) + 1) // 2) for o, s in zip(lay.psd_off, lay.psd_side)]
        return out

    def _vector(self, name: str) -> np.ndarray:
        from .native import lib
        cnt = ctypes.c_int64(0)
        lib().cipm_get_vector(self._ctx.handle, name.encode(), None, ctypes.byref(cnt))
        out = np.zeros(cnt.value)
        self._ctx.call("cipm_get_vector", name.encode(), pdbl(out), ctypes.byref(cnt))
        return out

    def _to_user_rows(self, v):
        out = np.empty_like(v)
        out[self._perm] = v
        return out

    def _state(self, which: int = 0) -> IterateState:
        x, z, s = np.zeros(self.n), np.zeros(self.m), np.zeros(self.m)
        tkm = np.zeros(3)
        self._ctx.call("cipm_get_iterate", which, pdbl(x), pdbl(z), pdbl(s), pdbl(tkm))
        return IterateState(x, z, s, float(tkm[0]), float(tkm[1]), float(tkm[2]))

    # -- residuals ------------------------------------------------------------

    def _residuals(self, sc) -> Residuals:
        """Eq.(7) quantities from the fused device reductions (scaled-space identities)."""
        tau, c = sc[SC["TAU"]], self._equil.c_obj
        xpx, qx, bz = sc[SC["XPX"]], sc[SC["QX"]], sc[SC["BZ"]]
        hq = 0.5 * xpx / (c * tau * tau)
        return Residuals(g_p=hq + qx / (c * tau), g_d=-hq - bz / (c * tau),
                         norm_rp=sc[SC["NRM_GZ"]] / tau, norm_rd=sc[SC["NRM_GX"]] / (c * tau),
                         norm_xbar=sc[SC["NRM_XU"]] / tau, norm_sbar=sc[SC["NRM_SU"]] / tau,
                         norm_zbar=sc[SC["NRM_ZU"]] / (c * tau))

    @property
    def num_symbolic(self) -> int:
        return self.kkt.num_symbolic

    def compute_residuals(self, state: IterateState | None = None) -> Residuals:
        """Residuals and objectives of the normalised iterate on the unscaled,
        reordered data (reference ipm.py:233-251), with the r_p / r_d vectors (rows
        in the reordered order, as the reference's).  state=None evaluates the
        device iterate; a given (scaled) state is uploaded into the device iterate
        first.  Not on the hot path: the loop uses the fused norms only."""
        ctx = self._ctx
        if state is not None:
            ctx.call("cipm_set_iterate", pdbl(state.x), pdbl(state.z), pdbl(state.s),
                     pdbl(np.array([state.tau, state.kappa, state.mu])))
        sc = np.zeros(64)
        ctx.call("cipm_residuals", pdbl(sc))
        res = self._residuals(sc)
        if self._equil.d_row is None:
            d_row, d_col, c_obj = np.empty(self.m), np.empty(self.n), ctypes.c_double(1.0)
            ctx.call("cipm_ctx_get_equilibration", pdbl(d_row), pdbl(d_col), ctypes.byref(c_obj))
            self._equil = Equilibration(d_row, d_col, float(c_obj.value))
        tau, c = float(sc[SC["TAU"]]), self._equil.c_obj
        # g_z = s + A x - b tau and g_x = -(P x + A'z + q tau) in the scaled space:
        # r_p = -g_z / (D_r tau), r_d = -g_x / (D_c c tau)
        res.r_p = -self._vector("gz") / (self._equil.d_row * tau)
        res.r_d = -self._vector("gx") / (self._equil.d_col * c * tau)
        return res

    def _ratios(self, r: Residuals):
        return (r.norm_rp / max(1.0, self._norm_b + r.norm_xbar + r.norm_sbar),
                r.norm_rd / max(1.0, self._norm_q + r.norm_xbar + r.norm_zbar),
                r.gap / max(1.0, min(abs(r.g_p), abs(r.g_d))))

    def _converged(self, r: Residuals, eps: float) -> bool:
        a, b, c = self._ratios(r)
        return a < eps and b < eps and c < eps

    def _infeasible(self, sc):
        """Eq.(9) tests on the unscaled, un-normalised iterate (ipm.py:263-280)."""
        eps = self.settings.eps_inf
        c = self._equil.c_obj
        bz = sc[SC["BZ"]] / c
        qx = sc[SC["QX"]] / c
        nx, nz, ns = sc[SC["NRM_XU"]], sc[SC["NRM_ZU"]] / c, sc[SC["NRM_SU"]]
        atz = sc[SC["NRM_ATZ"]] / c if self.n else 0.0
        if atz < -eps * max(1.0, nx + nz) * bz and bz < -eps:
            return Status.PRIMAL_INFEASIBLE
        px = sc[SC["NRM_PX"]] / c if self.n else 0.0
        axs = sc[SC["NRM_AXS"]]
        if px < -eps * max(1.0, nx) * bz and axs < -eps * max(1.0, nx + ns) * qx and qx < -eps:
            return Status.DUAL_INFEASIBLE
        return None

    # -- recovery -------------------------------------------------------------

    def _recover(self, which, res: Residuals, status, iterations, secs, tkm=None) -> SolveResult:
        """Result assembly (reference ipm.py:383-407).  Unscaling, the division by τ and
        the scatter back to the user's row order run on the device (cipm_get_solution);
        only x, z and s cross PCIe."""
        cert_mode = status in (Status.PRIMAL_INFEASIBLE, Status.DUAL_INFEASIBLE)
        x_o, z_o, s_o = pinned_empty(self.n), pinned_empty(self.m), pinned_empty(self.m)
        t = np.zeros(3)
        self._ctx.call("cipm_get_solution", which, 1 if cert_mode else 0, pdbl(x_o), pdbl(z_o), pdbl(s_o), pdbl(t))
        tau, kappa, mu = (float(v) for v in (tkm if tkm is not None else t))
        cert = None
        if status == Status.PRIMAL_INFEASIBLE:
            cert = z_o / abs(float(self._original.b @ z_o))
        elif status == Status.DUAL_INFEASIBLE:
            cert = x_o / abs(float(self._original.q @ x_o))
        return SolveResult(status=status, x=x_o, z=z_o, s=s_o, certificate=cert, obj_primal=res.g_p,
                           obj_dual=res.g_d, iterations=iterations, setup_seconds=self.setup_seconds,
                           solve_seconds=secs, norm_rp=res.norm_rp, norm_rd=res.norm_rd, gap=res.gap,
                           tau=tau, kappa=kappa, mu_initial=self._mu_initial, mu_final=mu)

    # -- main loop ------------------------------------------------------------

    _STATUS_CODES = {1: Status.OPTIMAL, 2: Status.PRIMAL_INFEASIBLE, 3: Status.DUAL_INFEASIBLE,
                     4: Status.MAX_ITERATIONS, 5: Status.INSUFFICIENT_PROGRESS}

    def solve(self, observer=None) -> SolveResult:
        """Algorithm 1 (reference ipm.py:411-496).  Default: the device-side loop — the
        termination / infeasibility / stall / best-iterate decisions run on the GPU and
        the host reads the scalar block once per iteration (cipm_loop_check).  With an
        observer (or CIPM_HOST_LOOP=1) the host-driven loop runs instead (debug mode:
        per-iteration documents need the directions on the host)."""
        if observer is not None or os.environ.get("CIPM_HOST_LOOP", "0") != "0":
            return self._solve_host(observer)
        t_start = time.perf_counter()
        cfg = self.settings
        ctx = self._ctx
        sc = self._sc
        ctx.call("cipm_loop_begin", self._norm_q, self._norm_b, cfg.eps_feas, cfg.eps_inf, int(cfg.max_iter))
        status = None
        res = None
        iterations = 0
        self.last_refine_steps = []
        for it in range(cfg.max_iter + 1):
            try:
                ctx.call("cipm_loop_check", it, pdbl(sc))
            except DeviceError:
                raise                    # CUDA / ABI faults are infrastructure errors, not a solver status
            except ConicError as err:    # the previous body failed (ipm.py:483-486)
                if cfg.verbose:
                    print(f"numerical error: {err}")
                status = Status.NUMERICAL_ERROR
                iterations = it - 1
                break
            if it == 0:
                self._mu_initial = float(sc[SC["MU"]])
            else:
                self.last_refine_steps.append((int(sc[SC["REF_STEPS_A"]]), int(sc[SC["REF_STEPS_C"]])))
            iterations = it
            res = self._residuals(sc)
            if cfg.verbose:
                print(f"iter {it:3d}  mu={sc[SC['MU']]:9.2e}  rp={res.norm_rp:9.2e}  "
                      f"rd={res.norm_rd:9.2e}  gap={res.gap:9.2e}  tau={sc[SC['TAU']]:8.2e}")
            code = int(sc[SC["STATUS"]])
            if code:
                status = self._STATUS_CODES[code]
                break
            if time.perf_counter() - t_start > cfg.time_limit:
                status = Status.TIME_LIMIT
                break
            try:
                ctx.call("cipm_loop_body")
            except DeviceError:
                raise
            except ConicError as err:    # an eager-mode body (profiling) failed synchronously
                if cfg.verbose:
                    print(f"numerical error: {err}")
                status = Status.NUMERICAL_ERROR
                break
        secs = time.perf_counter() - t_start
        if status in (Status.OPTIMAL, Status.PRIMAL_INFEASIBLE, Status.DUAL_INFEASIBLE):
            return self._recover(0, res, status, iterations, secs)
        if sc[SC["BEST_VALID"]] == 0.0:
            raise ConicError("solve failed before the first residual evaluation")
        best_res = Residuals(g_p=float(sc[SC["BEST_GP"]]), g_d=float(sc[SC["BEST_GD"]]),
                             norm_rp=float(sc[SC["BEST_RP"]]), norm_rd=float(sc[SC["BEST_RD"]]),
                             norm_xbar=float("nan"), norm_sbar=float("nan"), norm_zbar=float("nan"))
        e10 = ALMOST_OPTIMAL_FACTOR * cfg.eps_feas
        if max(sc[SC["BEST_R1"]], sc[SC["BEST_R2"]], sc[SC["BEST_R3"]]) < e10 and \
                sc[SC["BEST_R1"]] < e10 and sc[SC["BEST_R2"]] < e10 and sc[SC["BEST_R3"]] < e10:
            status = Status.ALMOST_OPTIMAL
        tkm = (float(sc[SC["BEST_TAU"]]), float(sc[SC["BEST_KAPPA"]]), float(sc[SC["BEST_MU"]]))
        return self._recover(1, best_res, status, iterations, secs, tkm=tkm)

    def _solve_host(self, observer=None) -> SolveResult:
        """Host-driven loop (one C call per step; used with an observer)."""
        t_start = time.perf_counter()
        cfg = self.settings
        ctx = self._ctx
        sc = self._sc
        ctx.call("cipm_init_iterate")
        ctx.call("cipm_read_scalars", pdbl(sc))
        self._mu_initial = float(sc[SC["MU"]])
        best_score = np.inf
        best_res = None
        best_tkm = None
        stall = [np.inf, np.inf, np.inf, 0]
        res = None
        status = None
        iterations = 0
        steps = ctypes.c_int(0)
        alpha = ctypes.c_double(0.0)
        self.last_refine_steps = []
        try:
            for it in range(cfg.max_iter + 1):
                ctx.call("cipm_residuals", pdbl(sc))
                tau, kappa, mu = float(sc[SC["TAU"]]), float(sc[SC["KAPPA"]]), float(sc[SC["MU"]])
                res = self._residuals(sc)
                score = max(self._ratios(res))
                if score < best_score or best_res is None:
                    if score < best_score:
                        best_score = score
                    best_res = res
                    best_tkm = (tau, kappa, mu)
                    ctx.call("cipm_save_best")
                if cfg.verbose:
                    print(f"iter {it:3d}  mu={mu:9.2e}  rp={res.norm_rp:9.2e}  "
                          f"rd={res.norm_rd:9.2e}  gap={res.gap:9.2e}  tau={tau:8.2e}")
                if self._converged(res, cfg.eps_feas):
                    status = Status.OPTIMAL
                    break
                inf_status = self._infeasible(sc)
                if inf_status is not None:
                    status = inf_status
                    break
                if it >= cfg.max_iter:
                    status = Status.MAX_ITERATIONS
                    break
                if time.perf_counter() - t_start > cfg.time_limit:
                    status = Status.TIME_LIMIT
                    break
                improved = (mu < STALL_IMPROVEMENT * stall[0] or res.norm_rp < STALL_IMPROVEMENT * stall[1]
                            or res.norm_rd < STALL_IMPROVEMENT * stall[2])
                stall[0] = min(stall[0], mu)
                stall[1] = min(stall[1], res.norm_rp)
                stall[2] = min(stall[2], res.norm_rd)
                stall[3] = 0 if improved else stall[3] + 1
                if stall[3] >= STALL_WINDOW:
                    status = Status.INSUFFICIENT_PROGRESS
                    break

                state_before = self._state(0) if observer is not None else None
                ctx.call("cipm_update_scaling")
                ctx.call("cipm_factor")
                ctx.call("cipm_solve_affine", ctypes.byref(steps))
                s_aff = steps.value
                ctx.call("cipm_step_affine")
                ctx.call("cipm_solve_combined", ctypes.byref(steps))
                s_comb = steps.value
                ctx.call("cipm_step_combined", ctypes.byref(alpha))
                self.last_refine_steps.append((s_aff, s_comb))
                if observer is not None:
                    observer(self._observer_doc(it, state_before))
                ctx.call("cipm_take_step")
                iterations = it + 1
        except DeviceError:
            raise                    # CUDA / ABI faults are infrastructure errors, not a solver status
        except (ConicError, np.linalg.LinAlgError) as err:
            if cfg.verbose:
                print(f"numerical error: {err}")
            status = Status.NUMERICAL_ERROR

        secs = time.perf_counter() - t_start
        if status in (Status.OPTIMAL, Status.PRIMAL_INFEASIBLE, Status.DUAL_INFEASIBLE):
            return self._recover(0, res, status, iterations, secs)
        if best_res is not None and self._converged(best_res, ALMOST_OPTIMAL_FACTOR * cfg.eps_feas):
            status = Status.ALMOST_OPTIMAL
        if best_res is None:
            raise ConicError("solve failed before the first residual evaluation")
        return self._recover(1, best_res, status, iterations, secs, tkm=best_tkm)

    def _observer_doc(self, it, state: IterateState) -> dict:
        sc = np.zeros(64)
        self._ctx.call("cipm_read_scalars", pdbl(sc))

        def direction(which):
            dx, dz, ds, dtk = np.zeros(self.n), np.zeros(self.m), np.zeros(self.m), np.zeros(2)
            self._ctx.call("cipm_get_direction", which, pdbl(dx), pdbl(dz), pdbl(ds), pdbl(dtk))
            return dx, dz, float(dtk[0]), ds, float(dtk[1])

        gx, gz = self._vector("gx"), self._vector("gz")
        sigma = float(sc[SC["SIGMA"]])
        f = 1.0 - sigma
        da = direction(0)
        d_aff = (gx, gz, float(sc[SC["GTAU"]]), state.s.copy(), state.kappa * state.tau)
        d_kappa_c = state.kappa * state.tau + da[4] * da[2] - sigma * state.mu
        d_comb = (f * gx, f * gz, f * float(sc[SC["GTAU"]]), self._vector("dsc"), d_kappa_c)
        return dict(iteration=it, state=state, scaling=DeviceScaling(self), d_affine=d_aff,
                    delta_affine=da, d_combined=d_comb, delta_combined=direction(1),
                    alpha_affine=float(sc[SC["ALPHA_A"]]), sigma=sigma,
                    alpha_combined=float(sc[SC["ALPHA_FINAL"]]))

    def close(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None:
            ctx.close()
            self._ctx = None
        sym = getattr(self, "symbolic", None)
        if sym is not None:
            sym.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve(problem: ProblemData, settings: SolverSettings | None = None, observer=None) -> SolveResult:
    """Validate, set up on the GPU and solve one problem instance (reference ipm.py:499-502)."""
    s = Solver(problem, settings)
    try:
        return s.solve(observer=observer)
    finally:
        s.close()
