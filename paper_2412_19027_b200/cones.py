"""Device-backed mirror of the reference's cone-level API (``conic_ipm.cones``):
``ConeSet``, ``degree``, ``update_scaling`` → ``ScalingState`` (``kkt_values``,
``dense``), ``apply_H``, ``combined_ds``, ``StepLengthRequest`` / ``step_length``,
``neighborhood_ok``, ``is_in_cone`` / ``is_in_dual_cone`` (strict) and
``soc_residuals_batch`` — same names, arguments and exceptions as
``cones/set.py``, ``cones/scaling.py`` and ``cones/steps.py``, every value computed
by the sm_100a cone kernels through the C ABI seams of ``include/cipm.h``
(``cipm_update_scaling``, ``cipm_scaling_values``, ``cipm_apply_h``,
``cipm_combined_ds``, ``cipm_set_direction`` + ``cipm_step_length``,
``cipm_neighborhood_ok``, ``cipm_membership``, ``cipm_soc_residuals``).

A cone set is bound to a small device context (the cone list over a 2-variable
problem; only its conic rows are used), created once per ``ConeSet`` and reused.
The row order is the family order of ``reorder_cones`` (the reference's
``ConeSet.from_specs`` requires it too).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from .csr import CsrMatrix
from .exceptions import ValidationError
from .model import ConeSpec, ProblemData

BACKTRACK = 0.8   # reference cones/steps.py default


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _vec(v, n, name):
    a = np.ascontiguousarray(v, dtype=np.float64)
    if a.shape != (n,):
        raise ValidationError(f"{name} must have length {n}")
    return a


@dataclass
class ConeSet:
    """Family-grouped index ranges over the m conic rows (reference cones/set.py:26-83)."""

    m: int
    zero_dim: int
    nonneg_dim: int
    socs: list = field(default_factory=list)    # (offset, dim)
    exps: list = field(default_factory=list)    # offset
    pows: list = field(default_factory=list)    # (offset, alpha)
    psds: list = field(default_factory=list)    # (offset, side)

    @property
    def nonneg_start(self) -> int:
        return self.zero_dim

    @property
    def degree(self) -> int:
        return (self.nonneg_dim + len(self.socs) + 3 * len(self.exps) + 3 * len(self.pows)
                + sum(side for _, side in self.psds))

    @staticmethod
    def from_specs(cones) -> "ConeSet":
        """Build from a family-ordered cone list (see reorder_cones)."""
        order = {"zero": 0, "nonneg": 1, "soc": 2, "exp": 3, "pow": 4, "psd": 5}
        stage, off = 0, 0
        cs = ConeSet(m=0, zero_dim=0, nonneg_dim=0)
        for c in cones:
            k = order[c.kind]
            if k < stage:
                raise ValidationError("cones must be family ordered (use reorder_cones)")
            stage = k
            if c.kind == "zero":
                cs.zero_dim += c.dim
            elif c.kind == "nonneg":
                cs.nonneg_dim += c.dim
            elif c.kind == "soc":
                cs.socs.append((off, c.dim))
            elif c.kind == "exp":
                cs.exps.append(off)
            elif c.kind == "pow":
                cs.pows.append((off, float(c.alpha)))
            else:
                cs.psds.append((off, int(c.side)))
            off += c.dim
        cs.m = off
        return cs

    def specs(self):
        out = []
        if self.zero_dim:
            out.append(ConeSpec("zero", self.zero_dim))
        if self.nonneg_dim:
            out.append(ConeSpec("nonneg", self.nonneg_dim))
        out += [ConeSpec("soc", d) for _, d in self.socs]
        out += [ConeSpec("exp", 3) for _ in self.exps]
        out += [ConeSpec("pow", 3, a) for _, a in self.pows]
        out += [ConeSpec("psd", s * (s + 1) // 2, side=s) for _, s in self.psds]
        return out


def degree(cones: ConeSet) -> int:
    return cones.degree


_CTX = {}


def _device(cones: ConeSet):
    """The device context bound to this cone set (a 2-variable problem over its rows)."""
    key = id(cones)
    hit = _CTX.get(key)
    if hit is not None and hit[0] is cones:
        return hit[1]
    from .solver import Solver
    specs = cones.specs()
    m, n = cones.m, 2
    P = CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))
    A = CsrMatrix(m, n, np.arange(m + 1, dtype=np.int64), (np.arange(m) % n).astype(np.int64),
                  np.linspace(1.0, 2.0, m) if m else np.zeros(0))
    s = Solver(ProblemData(P, A, np.zeros(n), np.zeros(m), specs))
    _CTX[key] = (cones, s)
    return s


def _set_point(s, sv, zv, tau=1.0, kappa=1.0, mu=1.0):
    s._ctx.call("cipm_set_iterate", _ptr(np.zeros(s.n)), _ptr(zv), _ptr(sv), _ptr(np.array([tau, kappa, mu])))


@dataclass
class ScalingState:
    """The scaling blocks at one (s, z), resident on the device (reference ScalingState)."""

    cones: ConeSet
    mu: float
    _solver: object = None
    _s: np.ndarray = None
    _z: np.ndarray = None

    def _refresh(self):
        _set_point(self._solver, self._s, self._z, mu=self.mu)
        self._solver._ctx.call("cipm_update_scaling")

    def kkt_values(self):
        """Diagonal over the zero+nonneg span and dense blocks per cone."""
        s = self._solver
        self._refresh()
        lin = self.cones.zero_dim + self.cones.nonneg_dim
        blocks = s._block_list()
        total = sum(d * (d + 1) // 2 for _, d in blocks)
        diag, hv = np.zeros(lin), np.zeros(max(total, 1))
        s._ctx.call("cipm_scaling_values", _ptr(diag), _ptr(hv))
        out, k = [], 0
        for off, d in blocks:
            iu = np.triu_indices(d)
            blk = np.zeros((d, d))
            blk[iu] = hv[k:k + len(iu[0])]
            blk = blk + np.triu(blk, 1).T
            out.append((int(off), blk))
            k += len(iu[0])
        return diag, out

    def dense(self) -> np.ndarray:
        h = np.zeros((self.cones.m, self.cones.m))
        diag, blocks = self.kkt_values()
        h[np.arange(len(diag)), np.arange(len(diag))] = diag
        for off, blk in blocks:
            d = blk.shape[0]
            h[off:off + d, off:off + d] = blk
        return h


def update_scaling(cones: ConeSet, s: np.ndarray, z: np.ndarray, mu: float) -> ScalingState:
    """Refresh every scaling block at (s, z) with complementarity mu (scaling.py:229-251);
    ScalingFailure off the cone interior."""
    sv, zv = _vec(s, cones.m, "s"), _vec(z, cones.m, "z")
    dev = _device(cones)
    st = ScalingState(cones=cones, mu=float(mu), _solver=dev, _s=sv.copy(), _z=zv.copy())
    st._refresh()
    return st


def apply_H(state: ScalingState, v: np.ndarray) -> np.ndarray:
    """Blockwise H v; the zero block maps to 0 (scaling.py:254-274)."""
    vv = _vec(v, state.cones.m, "v")
    state._refresh()
    out = np.zeros(state.cones.m)
    state._solver._ctx.call("cipm_apply_h", _ptr(vv), _ptr(out))
    return out


def combined_ds(state: ScalingState, cones: ConeSet, s: np.ndarray, z: np.ndarray,
                dz_a: np.ndarray, ds_a: np.ndarray, sigma: float, mu: float) -> np.ndarray:
    """Right-hand side d_s of the combined step (scaling.py:277-320), at the state's (s, z)."""
    m = cones.m
    sv, zv = _vec(s, m, "s"), _vec(z, m, "z")
    if not (np.array_equal(sv, state._s) and np.array_equal(zv, state._z)):
        state = update_scaling(cones, sv, zv, state.mu)
    state._refresh()
    out = np.zeros(m)
    state._solver._ctx.call("cipm_combined_ds", _ptr(_vec(dz_a, m, "dz_a")), _ptr(_vec(ds_a, m, "ds_a")),
                            float(sigma), float(mu), _ptr(out))
    return out


@dataclass
class StepLengthRequest:
    """Current iterate, direction and search controls (steps.py:21-37)."""

    z: np.ndarray
    s: np.ndarray
    dz: np.ndarray
    ds: np.ndarray
    tau: float
    kappa: float
    dtau: float
    dkappa: float
    alpha_max: float = 1.0
    backtrack: float = BACKTRACK


def step_length(req: StepLengthRequest, cones: ConeSet) -> float:
    """Largest alpha in (0, alpha_max] keeping the iterate interior (steps.py:79-116);
    StepTooSmall when the exp / pow backtracking runs out."""
    m = cones.m
    dev = _device(cones)
    _set_point(dev, _vec(req.s, m, "s"), _vec(req.z, m, "z"), float(req.tau), float(req.kappa))
    dev._ctx.call("cipm_set_direction", 0, None, _ptr(_vec(req.dz, m, "dz")), _ptr(_vec(req.ds, m, "ds")),
                  _ptr(np.array([float(req.dtau), float(req.dkappa)])))
    alpha = ctypes.c_double(0.0)
    dev._ctx.call("cipm_step_length", 0, ctypes.byref(alpha))
    return min(alpha.value, float(req.alpha_max))


def neighborhood_ok(cones: ConeSet, s: np.ndarray, z: np.ndarray, mu: float, beta: float) -> bool:
    """Central-path proximity per cone (scaling.py:364-401)."""
    m = cones.m
    dev = _device(cones)
    _set_point(dev, _vec(s, m, "s"), _vec(z, m, "z"), mu=float(mu))
    ok = ctypes.c_int(-1)
    dev._ctx.call("cipm_neighborhood_ok", float(mu), float(beta), ctypes.byref(ok))
    return bool(ok.value)


def _membership(cones: ConeSet, v: np.ndarray, strict: bool):
    if not strict:
        raise ValidationError("the device membership kernel is the strict-interior test of the IPM "
                              "(strict=True)")
    m = cones.m
    vv = _vec(v, m, "v")
    dev = _device(cones)
    inc, ind = ctypes.c_int(-1), ctypes.c_int(-1)
    dev._ctx.call("cipm_membership", _ptr(vv), _ptr(vv), ctypes.byref(inc), ctypes.byref(ind))
    return bool(inc.value), bool(ind.value)


def is_in_cone(cones: ConeSet, v: np.ndarray, strict: bool = True) -> bool:
    """Strict membership in int K (set.py:166-187)."""
    return _membership(cones, v, strict)[0]


def is_in_dual_cone(cones: ConeSet, v: np.ndarray, strict: bool = True) -> bool:
    """Strict membership in int K* (set.py:189-207)."""
    return _membership(cones, v, strict)[1]


def soc_residuals_batch(cones: ConeSet, x: np.ndarray) -> np.ndarray:
    """Per-SOC t^2 - |u|^2 in the reference's fixed summation order, bit for bit
    (steps.py:136-186, SPEC AC11)."""
    if not cones.socs:
        return np.zeros(0)
    dev = _device(cones)
    out = np.zeros(len(cones.socs))
    dev._ctx.call("cipm_soc_residuals", _ptr(_vec(x, cones.m, "x")), _ptr(out))
    return out
