"""Settings, statuses and result types (API-compatible with the reference).

Mirrors ``SolverSettings`` (``ipm.py:54-75``), ``Status`` (``ipm.py:40-51``),
``SolveResult`` (``ipm.py:117-139``), ``RefinementSettings``
(``kkt/system.py:45-53``) and the module constants of ``ipm.py:33-37`` /
``kkt/system.py:28-42``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FULL = "full"
MIXED = "mixed"

MIN_COMBINED_STEP = 1e-11
MIN_STEP = 1e-11
DENOM_GUARD = 1e-14
STALL_WINDOW = 5
STALL_IMPROVEMENT = 0.99
ALMOST_OPTIMAL_FACTOR = 10.0

_EPS32 = float(np.finfo(np.float32).eps)
_EPS64 = float(np.finfo(np.float64).eps)


def default_static_reg(precision: str) -> float:
    """δ_s: 1e-8 in full precision, √eps32 in mixed (reference system.py:35-37)."""
    return 1e-8 if precision == FULL else float(np.sqrt(np.finfo(np.float32).eps))


def default_dynamic_reg(precision: str) -> float:
    """δ_d: square of the active machine epsilon (reference system.py:40-42)."""
    return _EPS64 ** 2 if precision == FULL else _EPS32 ** 2


class Status:
    OPTIMAL = "optimal"
    PRIMAL_INFEASIBLE = "primal_infeasible"
    DUAL_INFEASIBLE = "dual_infeasible"
    ALMOST_OPTIMAL = "almost_optimal"
    MAX_ITERATIONS = "max_iterations"
    TIME_LIMIT = "time_limit"
    NUMERICAL_ERROR = "numerical_error"
    INSUFFICIENT_PROGRESS = "insufficient_progress"


TERMINAL_OK = (Status.OPTIMAL, Status.PRIMAL_INFEASIBLE, Status.DUAL_INFEASIBLE)


@dataclass
class RefinementSettings:
    t_abs: float = 1e-12
    t_rel: float = 1e-12
    t_max: int = 10

    def __post_init__(self):
        if self.t_abs <= 0 or self.t_rel <= 0 or self.t_max < 1:
            raise ValueError("refinement tolerances must be positive, t_max >= 1")


@dataclass
class SolverSettings:
    eps_feas: float = 1e-6
    eps_inf: float = 1e-8
    max_iter: int = 200
    time_limit: float = np.inf
    precision: str = FULL
    delta_s: float | None = None
    delta_d: float | None = None
    beta: float = 1e-6
    backtrack: float = 0.8
    step_scale: float = 0.99
    do_equilibrate: bool = True
    verbose: bool = False
    refinement: RefinementSettings = field(default_factory=RefinementSettings)

    def __post_init__(self):
        if not (0.0 < self.step_scale < 1.0):
            raise ValueError("step_scale must lie in (0, 1)")
        for name in ("eps_feas", "eps_inf", "max_iter", "time_limit", "beta", "backtrack"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be nonnegative")
        if self.precision not in (FULL, MIXED):
            raise ValueError(f"unknown precision mode {self.precision!r}")


@dataclass
class SolveResult:
    status: str
    x: np.ndarray
    z: np.ndarray
    s: np.ndarray
    certificate: np.ndarray | None
    obj_primal: float
    obj_dual: float
    iterations: int
    setup_seconds: float
    solve_seconds: float
    norm_rp: float
    norm_rd: float
    gap: float
    tau: float
    kappa: float
    mu_initial: float
    mu_final: float

    @property
    def is_terminal_ok(self) -> bool:
        return self.status in TERMINAL_OK


def centering(alpha_affine: float) -> float:
    """σ = (1 − α_a)³ (reference ipm.py:142-144)."""
    return (1.0 - alpha_affine) ** 3
