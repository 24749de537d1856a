"""Exception hierarchy of the solver, name-compatible with the reference.

Mirrors ``conic_ipm.errors`` (reference ``pkg/src/conic_ipm/errors.py:4-53``)
so user code catching e.g. ``ScalingFailure`` keeps working.  Device kernels
report failures as negative int status codes through the C ABI
(``include/cipm.h``); :func:`raise_for_status` maps them back onto these types
so the IPM status machine (``ipm.py:483-486`` in the reference) is unchanged.
"""
from __future__ import annotations


class ConicError(Exception):
    """Root of every error this package raises."""


class ValidationError(ConicError):
    """Structural invariant of the problem data violated."""


class DimensionMismatch(ValidationError):
    """Array / matrix / cone sizes disagree."""


class NonSymmetricP(ValidationError):
    """P is not exactly symmetric."""


class BadConeSpec(ValidationError):
    """A cone descriptor is malformed (dim, alpha, side)."""


class NonFiniteData(ValidationError):
    """NaN or Inf in P, A, q or b."""


class DomainError(ConicError):
    """A point is outside the (strict) interior of its cone."""


class ScalingFailure(ConicError):
    """A scaling block could not be formed: the iterate lost the interior."""


class StepTooSmall(ConicError):
    """Step-length search collapsed below the minimum step."""


class FactorizationFailure(ConicError):
    """LDL' pivot exactly zero after regularization."""


class PatternMismatch(ConicError):
    """Updated data does not share the setup sparsity pattern."""


class DegenerateDenominator(ConicError):
    """The tau-step denominator vanished."""


class LostInterior(ConicError):
    """The accepted step left the cone interior."""


class DeviceError(ConicError):
    """A CUDA runtime call failed inside the native library."""


# Status codes returned by the C ABI (include/cipm.h, CIPM_E_*).
_CODE_TO_EXC = {
    -1: ScalingFailure,
    -2: StepTooSmall,
    -3: FactorizationFailure,
    -4: DegenerateDenominator,
    -5: LostInterior,
    -6: DomainError,
    -7: PatternMismatch,
    -8: DimensionMismatch,
    -20: DeviceError,
    -21: DeviceError,
}

_CODE_TEXT = {
    -1: "scaling block is not positive definite / iterate lost the cone interior",
    -2: "step length collapsed below the minimum step",
    -3: "zero pivot after regularization",
    -4: "tau-step denominator is numerically zero",
    -5: "accepted step left the cone interior",
    -6: "point outside the cone interior",
    -7: "pattern mismatch",
    -8: "dimension mismatch",
    -20: "CUDA runtime error",
    -21: "invalid argument to native library",
}


def raise_for_status(code: int, where: str = "") -> None:
    """Raise the ConicError subclass matching a negative C-ABI status code."""
    if code >= 0:
        return
    exc = _CODE_TO_EXC.get(code, ConicError)
    msg = _CODE_TEXT.get(code, f"native status {code}")
    raise exc(f"{where}: {msg}" if where else msg)
