"""B200-native interior-point hot path for quadratic conic programs (arXiv 2412.19027).

Drop-in for the reference ``conic_ipm`` solver API: problems are given as

    minimize ½x'Px + q'x   subject to   Ax + s = b,  s ∈ K

with K a product of zero, nonnegative, second-order, exponential, power and
PSD cones.  Host setup (validation, cone reordering, Ruiz equilibration,
one-time symbolic analysis) stays on the CPU; every per-iteration operation of
Algorithm 1 runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/cipm.h`` (``lib/libcipm.so``).
"""
from .csr import CsrMatrix
from .exceptions import (BadConeSpec, ConicError, DegenerateDenominator, DeviceError, DimensionMismatch,
                         DomainError, FactorizationFailure, LostInterior, NonFiniteData, NonSymmetricP,
                         PatternMismatch, ScalingFailure, StepTooSmall, ValidationError)
from .model import (ConeSpec, Equilibration, ProblemData, equilibrate, exp_cone, nonneg_cone, pow_cone,
                    psd_cone, reorder_cones, scale_values, soc_cone, unscale_solution, validate, zero_cone)
from .settings import (FULL, MIXED, RefinementSettings, SolveResult, SolverSettings, Status, TERMINAL_OK,
                       centering)
from .families import (GenSpec, InfeasibleBoxBudget, gen_entropy, gen_huber, gen_multistage_portfolio,
                       gen_portfolio)
from .io import read_problem, write_problem
from .metrics import perf_profiles, shifted_geomean
# the reference's cone-level functions, computed by the device cone kernels (cones.py)
from .cones import (ConeSet, ScalingState, StepLengthRequest, apply_H, combined_ds, degree, is_in_cone,
                    is_in_dual_cone, neighborhood_ok, soc_residuals_batch, step_length, update_scaling)

__version__ = "0.1.0"


def __getattr__(name):
    # the device solver is imported lazily so the data model works without CUDA
    if name in ("Solver", "solve", "IterateState", "Residuals"):
        from . import solver as _s
        return getattr(_s, name)
    if name in ("KKTSystem", "assemble", "RefineResult"):
        from . import kkt as _k
        return getattr(_k, name)
    if name in ("BatchSolver", "solve_many"):
        from . import batch as _b
        return getattr(_b, name)
    raise AttributeError(name)
