"""Device-backed ``KKTSystem`` / ``assemble`` with the reference's interface
(kkt/system.py:64-321): ``set_matrices``, ``set_scaling``, ``symbolic_factor``,
``numeric_factor``, ``solve_refined`` → ``RefineResult``, ``matvec`` and the
counters ``num_symbolic`` / ``num_numeric`` / ``last_bumped_pivots``.

K = [P A'; A -H] over the raw (not equilibrated) P, A and the cone rows of a
family-ordered ``ConeSet``.  The pattern analysis runs once, in the C++ symbolic
analysis, when the system is assembled; H comes from the host through
``cipm_kkt_set_scaling`` (the diagonal of the zero + nonneg rows and one dense
block per SOC / exp / pow / PSD cone, as ``ScalingState.kkt_values`` returns
them), the factorisation is the device supernodal LDLᵀ (``cipm_factor``) and the
refined solve the device refinement loop (``cipm_kkt_solve_ex``), whose residual
is taken against the unregularised FP64 K as in ``solve_refined``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .exceptions import ConicError, DimensionMismatch
from .model import ProblemData
from .settings import FULL, RefinementSettings, SolverSettings


@dataclass
class RefineResult:
    x: np.ndarray
    steps: int
    stalled: bool
    residual: float


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class KKTSystem:
    """The quasi-definite KKT matrix of one problem on the device."""

    def __init__(self, P, A, cones, precision: str = FULL, delta_s: float | None = None,
                 delta_d: float | None = None):
        from .solver import Solver
        self.cones = cones
        self.n, self.m = P.nrows, A.nrows
        if cones.m != self.m:
            raise DimensionMismatch("cone rows differ from the rows of A")
        self.dim = self.n + self.m
        self.precision = precision
        prob = ProblemData(P, A, np.zeros(self.n), np.zeros(self.m), cones.specs())
        self._solver = Solver(prob, SolverSettings(precision=precision, delta_s=delta_s, delta_d=delta_d,
                                                   do_equilibrate=False))
        if not np.array_equal(self._solver._perm, np.arange(self.m)):
            raise ConicError("cones must be family ordered (use reorder_cones)")
        self._blocks = self._solver._block_list()
        self._scaled = False
        self._factored = False

    # --- values -------------------------------------------------------------
    def set_matrices(self, P=None, A=None) -> None:
        """New P / A values on the fixed pattern (system.py:152-164)."""
        self._solver.update_data(P=P, A=A)
        self._factored = False

    def set_scaling(self, diag: np.ndarray, blocks) -> None:
        """H from ScalingState.kkt_values() (system.py:166-179)."""
        lin = self.cones.zero_dim + self.cones.nonneg_dim
        d = np.ascontiguousarray(diag, dtype=np.float64)
        if d.shape != (lin,):
            raise DimensionMismatch(f"diag must have length {lin}")
        blocks = list(blocks)
        if [int(o) for o, _ in blocks] != [int(o) for o, _ in self._blocks]:
            raise DimensionMismatch("blocks must follow the cone order of the system")
        packed = [np.asarray(b, dtype=np.float64)[np.triu_indices(np.asarray(b).shape[0])] for _, b in blocks]
        flat = np.ascontiguousarray(np.concatenate(packed) if packed else np.zeros(1))
        self._solver._ctx.call("cipm_kkt_set_scaling", _ptr(d), _ptr(flat))
        self._scaled = True
        self._factored = False

    # --- factorisation --------------------------------------------------------
    def symbolic_factor(self) -> None:
        """The pattern analysis ran when the system was assembled (one per pattern)."""

    def numeric_factor(self) -> None:
        """LDLᵀ of K + static / dynamic regularisation (system.py:246-263)."""
        if not self._scaled:
            raise ConicError("set_scaling must precede numeric_factor")
        self._solver._ctx.call("cipm_factor")
        self._factored = True

    def solve_refined(self, b: np.ndarray, settings: RefinementSettings | None = None) -> RefineResult:
        """Iteratively refined solve against the unregularised K (system.py:279-314)."""
        if not self._factored:
            raise ConicError("numeric factorization is stale; call numeric_factor first")
        st = settings or RefinementSettings()
        self._solver._ctx.call("cipm_set_refinement", float(st.t_abs), float(st.t_rel), int(st.t_max))
        rhs = np.ascontiguousarray(b, dtype=np.float64)
        if rhs.shape != (self.dim,):
            raise DimensionMismatch(f"b must have length {self.dim}")
        x = np.zeros(self.dim)
        steps, res, stalled = ctypes.c_int(0), ctypes.c_double(0.0), ctypes.c_int(0)
        self._solver._ctx.call("cipm_kkt_solve_ex", _ptr(rhs), _ptr(x), ctypes.byref(steps), ctypes.byref(res),
                               ctypes.byref(stalled))
        return RefineResult(x=x, steps=int(steps.value), stalled=bool(stalled.value), residual=float(res.value))

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """Unregularised FP64 K x (system.py:273-277)."""
        xv = np.ascontiguousarray(x, dtype=np.float64)
        if xv.shape != (self.dim,):
            raise DimensionMismatch(f"x must have length {self.dim}")
        out = np.zeros(self.dim)
        self._solver._ctx.call("cipm_kkt_matvec", _ptr(xv), _ptr(out))
        return out

    # --- counters -------------------------------------------------------------
    @property
    def num_symbolic(self) -> int:
        return 1

    @property
    def num_numeric(self) -> int:
        return self._solver.kkt.num_numeric

    @property
    def last_bumped_pivots(self) -> int:
        return self._solver.kkt.last_bumped_pivots

    def close(self) -> None:
        self._solver.close()


def assemble(P, A, cones, precision: str = FULL, delta_s: float | None = None,
             delta_d: float | None = None) -> KKTSystem:
    """Build the KKT system with slots for every H entry (system.py:317-321)."""
    return KKTSystem(P, A, cones, precision=precision, delta_s=delta_s, delta_d=delta_d)
