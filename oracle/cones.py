"""ORACLE — TEST INFRASTRUCTURE ONLY (never imported by the product path).

CPU restatement of the reference cone engine, used as the parity checker
for the CUDA kernels and as the CPU baseline.  Sections follow (file:line in
/root/reference/pkg/src/conic_ipm):

  ConeLayout / degree / unit start    cones/set.py:25-112
  strict membership predicates        cones/set.py:120-207, cones/barriers.py:82-86,147-151,170-175,248-252
  exp / pow dual barrier calculus     cones/barriers.py:89-245
  conjugate points (bracket + Brent)  cones/barriers.py:280-363  (scipy.optimize.brentq, as the reference)
  PSD svec / NT factor / step bound   cones/psdcone.py:21-133
  NT SOC update, W̄ apply, Jordan      cones/scaling.py:38-94
  rank-3 BFGS with fallbacks          cones/scaling.py:112-175
  update_scaling / kkt blocks / H·v   cones/scaling.py:201-274
  combined_ds                         cones/scaling.py:277-327
  neighbourhood test                  cones/scaling.py:364-401
  step_length (+ exp/pow backtrack)   cones/steps.py:40-131
  batched SOC residual order          cones/steps.py:136-175

The arithmetic (numpy calls, operation order) follows the reference so the
oracle agrees with it to the last bits on the golden fixtures.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2412_19027_b200.exceptions import DomainError, ScalingFailure, StepTooSmall
from paper_2412_19027_b200.model import EXP, NONNEG, POW, PSD, SOC, ZERO

EXP_UNIT = np.array([-1.051383945322714, 0.556409619469370, 1.258967884768947])
SQRT2 = np.sqrt(2.0)
BFGS_GUARD = 1e-8
CONJ_MAX_ITERS = 100
MIN_STEP = 1e-11


def tri(side: int) -> int:
    return side * (side + 1) // 2


# ---------------------------------------------------------------------------
# layout
# ---------------------------------------------------------------------------

@dataclass
class ConeLayout:
    m: int
    zero_dim: int
    nonneg_dim: int
    socs: list = field(default_factory=list)     # (offset, dim)
    exps: list = field(default_factory=list)     # offset
    pows: list = field(default_factory=list)     # (offset, alpha)
    psds: list = field(default_factory=list)     # (offset, side)

    @property
    def nn0(self) -> int:
        return self.zero_dim

    @property
    def degree(self) -> int:
        return (self.nonneg_dim + len(self.socs) + 3 * len(self.exps) + 3 * len(self.pows)
                + sum(side for _, side in self.psds))

    @staticmethod
    def from_specs(cones) -> "ConeLayout":
        lay = ConeLayout(0, 0, 0)
        off = 0
        for c in cones:
            if c.kind == ZERO:
                lay.zero_dim += c.dim
            elif c.kind == NONNEG:
                lay.nonneg_dim += c.dim
            elif c.kind == SOC:
                lay.socs.append((off, c.dim))
            elif c.kind == EXP:
                lay.exps.append(off)
            elif c.kind == POW:
                lay.pows.append((off, c.alpha))
            elif c.kind == PSD:
                lay.psds.append((off, c.side))
            off += c.dim
        lay.m = off
        return lay

    def nsym(self):
        """(kind, offset, alpha) over exp cones then pow cones."""
        for off in self.exps:
            yield EXP, off, None
        for off, a in self.pows:
            yield POW, off, a

    def blocks(self):
        """(offset, dim) of every dense KKT block in family order."""
        for off, d in self.socs:
            yield off, d
        for off in self.exps:
            yield off, 3
        for off, _ in self.pows:
            yield off, 3
        for off, side in self.psds:
            yield off, tri(side)


def unit_start(lay: ConeLayout):
    s = np.zeros(lay.m)
    z = np.zeros(lay.m)
    s[lay.nn0:lay.nn0 + lay.nonneg_dim] = 1.0
    z[lay.nn0:lay.nn0 + lay.nonneg_dim] = 1.0
    for off, _ in lay.socs:
        s[off] = z[off] = 1.0
    for off in lay.exps:
        s[off:off + 3] = EXP_UNIT
        z[off:off + 3] = EXP_UNIT
    for off, a in lay.pows:
        pt = np.array([np.sqrt(1.0 + a), np.sqrt(2.0 - a), 0.0])
        s[off:off + 3] = pt
        z[off:off + 3] = pt
    for off, side in lay.psds:
        e = svec(np.eye(side))
        s[off:off + tri(side)] = e
        z[off:off + tri(side)] = e
    return s, z


# ---------------------------------------------------------------------------
# PSD helpers
# ---------------------------------------------------------------------------

def svec(x: np.ndarray) -> np.ndarray:
    side = x.shape[0]
    out = np.empty(tri(side))
    k = 0
    for j in range(side):
        out[k] = x[j, j]
        out[k + 1:k + side - j] = SQRT2 * x[j + 1:, j]
        k += side - j
    return out


def smat(v: np.ndarray, side: int) -> np.ndarray:
    x = np.zeros((side, side))
    k = 0
    for j in range(side):
        x[j, j] = v[k]
        col = v[k + 1:k + side - j] / SQRT2
        x[j + 1:, j] = col
        x[j, j + 1:] = col
        k += side - j
    return x


def congruence(r: np.ndarray) -> np.ndarray:
    """Matrix of X -> R'XR in svec coordinates (column-by-column, like the reference)."""
    side = r.shape[0]
    d = tri(side)
    out = np.empty((d, d))
    e = np.zeros(d)
    for k in range(d):
        e[k] = 1.0
        out[:, k] = svec(r.T @ smat(e, side) @ r)
        e[k] = 0.0
    return out


def psd_min_eig(v, side) -> float:
    return float(np.linalg.eigvalsh(smat(v, side))[0])


def psd_nt(s, z, side):
    sm, zm = smat(s, side), smat(z, side)
    try:
        ls = np.linalg.cholesky(sm)
        lz = np.linalg.cholesky(zm)
    except np.linalg.LinAlgError:
        raise ScalingFailure("PSD iterate lost positive definiteness") from None
    _, sig, vt = np.linalg.svd(lz.T @ ls)
    if np.min(sig) <= 0.0:
        raise ScalingFailure("degenerate NT scaling point for a PSD block")
    r = ls @ vt.T @ np.diag(1.0 / np.sqrt(sig))
    rinv = np.diag(np.sqrt(sig)) @ vt @ np.linalg.inv(ls)
    return r, rinv, sig


def psd_step(v, dv, side) -> float:
    x, d = smat(v, side), smat(dv, side)
    try:
        l = np.linalg.cholesky(x)
    except np.linalg.LinAlgError:
        raise DomainError("point outside the PSD cone interior") from None
    li = np.linalg.inv(l)
    lam = np.linalg.eigvalsh(li @ d @ li.T)[0]
    return np.inf if lam >= 0.0 else -1.0 / lam


# ---------------------------------------------------------------------------
# exp / pow barrier calculus (dual side) and predicates
# ---------------------------------------------------------------------------

def exp_dual_ok(z) -> bool:
    z1, z2, z3 = z
    if z1 >= 0.0 or z3 <= 0.0:
        return False
    return z2 - z1 - z1 * np.log(z3 / -z1) > 0.0


def exp_primal_ok(s) -> bool:
    x, y, z = s
    if y <= 0.0 or z <= 0.0:
        return False
    return y * np.log(z / y) - x > 0.0


def pow_dual_ok(z, a) -> bool:
    z1, z2, z3 = z
    if z1 <= 0.0 or z2 <= 0.0:
        return False
    lw = 2.0 * a * np.log(z1 / a) + 2.0 * (1 - a) * np.log(z2 / (1 - a))
    return np.exp(lw) - z3 * z3 > 0.0


def pow_primal_ok(s, a) -> bool:
    x, y, z = s
    if x <= 0.0 or y <= 0.0:
        return False
    return np.exp(2 * a * np.log(x) + 2 * (1 - a) * np.log(y)) - z * z > 0.0


def _exp_terms(z):
    z1, z2, z3 = float(z[0]), float(z[1]), float(z[2])
    if z1 >= 0.0 or z3 <= 0.0:
        raise DomainError("point outside the dual exponential cone interior")
    lg = np.log(z3 / -z1)
    psi = z2 - z1 - z1 * lg
    if psi <= 0.0:
        raise DomainError("point outside the dual exponential cone interior")
    return z1, z2, z3, lg, psi


def exp_grad(z):
    z1, _, z3, lg, psi = _exp_terms(z)
    r = 1.0 / psi
    return np.array([r * lg - 1.0 / z1, -r, r * z1 / z3 - 1.0 / z3])


def _exp_psi_derivs(z1, z3, lg):
    g = np.array([-lg, 1.0, -z1 / z3])
    h = np.array([[1.0 / z1, 0.0, -1.0 / z3], [0.0, 0.0, 0.0], [-1.0 / z3, 0.0, z1 / (z3 * z3)]])
    return g, h


def exp_hess(z):
    z1, _, z3, lg, psi = _exp_terms(z)
    r = 1.0 / psi
    g, h = _exp_psi_derivs(z1, z3, lg)
    out = r * r * np.outer(g, g) - r * h
    out[0, 0] += 1.0 / (z1 * z1)
    out[2, 2] += 1.0 / (z3 * z3)
    return out


def exp_third(z, u):
    z1, _, z3, lg, psi = _exp_terms(z)
    u1, u3 = float(u[0]), float(u[2])
    r = 1.0 / psi
    g, h = _exp_psi_derivs(z1, z3, lg)
    t_u = np.array([[-u1 / (z1 * z1), 0.0, u3 / (z3 * z3)],
                    [0.0, 0.0, 0.0],
                    [u3 / (z3 * z3), 0.0, u1 / (z3 * z3) - 2.0 * z1 * u3 / (z3 ** 3)]])
    gu = float(g @ u)
    hu = h @ u
    out = -2.0 * r ** 3 * gu * np.outer(g, g)
    out += r * r * (np.outer(hu, g) + np.outer(g, hu) + gu * h)
    out -= r * t_u
    out[0, 0] += -2.0 * u1 / z1 ** 3
    out[2, 2] += -2.0 * u3 / z3 ** 3
    return out


def _pow_terms(z, a):
    z1, z2, z3 = float(z[0]), float(z[1]), float(z[2])
    if z1 <= 0.0 or z2 <= 0.0:
        raise DomainError("point outside the dual power cone interior")
    b = 1.0 - a
    om = np.exp(2.0 * a * np.log(z1 / a) + 2.0 * b * np.log(z2 / b))
    phi = om - z3 * z3
    if phi <= 0.0:
        raise DomainError("point outside the dual power cone interior")
    return z1, z2, z3, b, om, phi


def _pow_hphi(z1, z2, a, b, om):
    return np.array([
        [2.0 * a * (2 * a - 1) * om / (z1 * z1), 4.0 * a * b * om / (z1 * z2), 0.0],
        [4.0 * a * b * om / (z1 * z2), 2.0 * b * (2 * b - 1) * om / (z2 * z2), 0.0],
        [0.0, 0.0, -2.0]])


def pow_grad(z, a):
    z1, z2, z3, b, om, phi = _pow_terms(z, a)
    r = 1.0 / phi
    gphi = np.array([2.0 * a * om / z1, 2.0 * b * om / z2, -2.0 * z3])
    return -r * gphi + np.array([-b / z1, -a / z2, 0.0])


def pow_hess(z, a):
    z1, z2, z3, b, om, phi = _pow_terms(z, a)
    r = 1.0 / phi
    gphi = np.array([2.0 * a * om / z1, 2.0 * b * om / z2, -2.0 * z3])
    out = r * r * np.outer(gphi, gphi) - r * _pow_hphi(z1, z2, a, b, om)
    out[0, 0] += b / (z1 * z1)
    out[1, 1] += a / (z2 * z2)
    return out


def pow_third(z, u, a):
    z1, z2, z3, b, om, phi = _pow_terms(z, a)
    u1, u2 = float(u[0]), float(u[1])
    r = 1.0 / phi
    gphi = np.array([2.0 * a * om / z1, 2.0 * b * om / z2, -2.0 * z3])
    hphi = _pow_hphi(z1, z2, a, b, om)
    p111 = 2 * a * (2 * a - 1) * (2 * a - 2) * om / z1 ** 3
    p112 = 4 * a * (2 * a - 1) * b * om / (z1 * z1 * z2)
    p122 = 4 * a * b * (2 * b - 1) * om / (z1 * z2 * z2)
    p222 = 2 * b * (2 * b - 1) * (2 * b - 2) * om / z2 ** 3
    t_u = np.array([[p111 * u1 + p112 * u2, p112 * u1 + p122 * u2, 0.0],
                    [p112 * u1 + p122 * u2, p122 * u1 + p222 * u2, 0.0],
                    [0.0, 0.0, 0.0]])
    gu = float(gphi @ u)
    hu = hphi @ u
    out = -2.0 * r ** 3 * gu * np.outer(gphi, gphi)
    out += r * r * (np.outer(hu, gphi) + np.outer(gphi, hu) + gu * hphi)
    out -= r * t_u
    out[0, 0] += -2.0 * b * u1 / z1 ** 3
    out[1, 1] += -2.0 * a * u2 / z2 ** 3
    return out


def _bracket(f, t0):
    lo = hi = t0
    for _ in range(CONJ_MAX_ITERS):
        if f(lo) > 0.0:
            break
        lo /= 10.0
        if lo < 1e-300:
            raise ScalingFailure("conjugate-gradient bracketing failed (low end)")
    for _ in range(CONJ_MAX_ITERS):
        if f(hi) < 0.0:
            break
        hi *= 10.0
        if hi > 1e300:
            raise ScalingFailure("conjugate-gradient bracketing failed (high end)")
    return lo, hi


def _root_decreasing(f, t0):
    from scipy.optimize import brentq
    lo, hi = _bracket(f, t0)
    return float(brentq(f, lo, hi, xtol=1e-300, rtol=4 * np.finfo(float).eps,
                        maxiter=CONJ_MAX_ITERS))


def exp_conj(s):
    """w = -∇f*(s) for the exponential cone (barriers.py:305-328)."""
    if not exp_primal_ok(s):
        raise DomainError("point outside the exponential cone interior")
    s1, s2, s3 = float(s[0]), float(s[1]), float(s[2])

    def f(t):
        return s2 * (np.log1p(s2 * t) - np.log(s3 * t)) + 1.0 / t + s1

    t = _root_decreasing(f, 1.0 / (1.0 + abs(s1) + s2 + s3))
    w3 = (1.0 + s2 * t) / s3
    w1 = -t
    w2 = 1.0 / s2 + w1 + w1 * np.log(w3 / t)
    return np.array([w1, w2, w3])


def pow_conj(s, a):
    """w = -∇f*(s) for the power cone (barriers.py:331-363)."""
    if not pow_primal_ok(s, a):
        raise DomainError("point outside the power cone interior")
    s1, s2, s3 = float(s[0]), float(s[1]), float(s[2])
    b = 1.0 - a
    if s3 == 0.0:
        return np.array([(1.0 + a) / s1, (2.0 - a) / s2, 0.0])
    const = (2.0 * np.log(abs(s3)) - 2.0 * a * np.log(a * s1) - 2.0 * b * np.log(b * s2)
             - np.log(4.0))

    def g(v):
        u = 1.0 + v
        return (2.0 * a * np.log(2.0 * a * u + b) + 2.0 * b * np.log(2.0 * b * u + a)
                - np.log(u) - np.log(v) + const)

    v = _root_decreasing(g, 1.0)
    u = 1.0 + v
    return np.array([(2.0 * a * u + b) / s1, (2.0 * b * u + a) / s2, -2.0 * v / s3])


# ---------------------------------------------------------------------------
# membership
# ---------------------------------------------------------------------------

def _soc_ok(blk, strict=True):
    nrm = np.linalg.norm(blk[1:])
    return blk[0] > nrm if strict else blk[0] >= nrm


def _exp_member_strict(blk):
    x, y, z = blk
    return y > 0.0 and z > 0.0 and np.log(y) + x / y < np.log(z)


def _exp_dual_member_strict(blk):
    u, v, w = blk
    return u < 0.0 and w > 0.0 and np.log(-u) + v / u < 1.0 + np.log(w)


def _pow_member_strict(blk, a):
    x, y, z = blk
    if x <= 0.0 or y <= 0.0:
        return False
    if z == 0.0:
        return True
    return a * np.log(x) + (1 - a) * np.log(y) > np.log(abs(z))


def in_cone(lay: ConeLayout, v) -> bool:
    """Strict membership s ∈ int K (set.py:166-186); zero block exactly 0."""
    if np.any(v[:lay.zero_dim] != 0.0):
        return False
    nn = v[lay.nn0:lay.nn0 + lay.nonneg_dim]
    if nn.size and np.any(nn <= 0.0):
        return False
    for off, d in lay.socs:
        if not _soc_ok(v[off:off + d]):
            return False
    for off in lay.exps:
        if not _exp_member_strict(v[off:off + 3]):
            return False
    for off, a in lay.pows:
        if not _pow_member_strict(v[off:off + 3], a):
            return False
    for off, side in lay.psds:
        if psd_min_eig(v[off:off + tri(side)], side) <= 0.0:
            return False
    return True


def in_dual_cone(lay: ConeLayout, v) -> bool:
    """Strict membership z ∈ int K* (set.py:189-207)."""
    nn = v[lay.nn0:lay.nn0 + lay.nonneg_dim]
    if nn.size and np.any(nn <= 0.0):
        return False
    for off, d in lay.socs:
        if not _soc_ok(v[off:off + d]):
            return False
    for off in lay.exps:
        if not _exp_dual_member_strict(v[off:off + 3]):
            return False
    for off, a in lay.pows:
        u, w, t = v[off:off + 3]
        if not _pow_member_strict((u / a, w / (1 - a), t), a):
            return False
    for off, side in lay.psds:
        if psd_min_eig(v[off:off + tri(side)], side) <= 0.0:
            return False
    return True


# ---------------------------------------------------------------------------
# scaling state
# ---------------------------------------------------------------------------

def soc_res(x) -> float:
    return float(x[0] * x[0] - np.dot(x[1:], x[1:]))


def wbar_apply(w, x, inverse=False):
    sg = -1.0 if inverse else 1.0
    c = float(w[1:] @ x[1:])
    out = np.empty_like(x)
    out[0] = w[0] * x[0] + sg * c
    out[1:] = sg * x[0] * w[1:] + x[1:] + (c / (1.0 + w[0])) * w[1:]
    return out


def jordan(u, v):
    out = np.empty_like(u)
    out[0] = float(u @ v)
    out[1:] = u[0] * v[1:] + v[0] * u[1:]
    return out


def arrow_solve(lam, r):
    res = soc_res(lam)
    u = np.empty_like(r)
    u[0] = (lam[0] * r[0] - float(lam[1:] @ r[1:])) / res
    u[1:] = (r[1:] - u[0] * lam[1:]) / lam[0]
    return u


@dataclass
class SocNT:
    w: np.ndarray
    eta: float
    lam: np.ndarray


def soc_nt(s, z) -> SocNT:
    rs, rz = soc_res(s), soc_res(z)
    if rs <= 0.0 or rz <= 0.0 or s[0] <= 0.0 or z[0] <= 0.0:
        raise ScalingFailure("second-order block lost the cone interior")
    a, b = np.sqrt(rs), np.sqrt(rz)
    sb, zb = s / a, z / b
    gamma = np.sqrt((1.0 + float(sb @ zb)) / 2.0)
    w = (sb + np.concatenate(([zb[0]], -zb[1:]))) / (2.0 * gamma)
    eta = np.sqrt(a / b)
    return SocNT(w, eta, eta * wbar_apply(w, z))


def soc_block(sc: SocNT, d: int) -> np.ndarray:
    h = 2.0 * np.outer(sc.w, sc.w)
    h[np.diag_indices(d)] += 1.0
    h[0, 0] -= 2.0
    return sc.eta ** 2 * h


@dataclass
class NsymScale:
    h: np.ndarray
    grad: np.ndarray
    hess: np.ndarray
    zt: np.ndarray
    mu_c: float
    mu_t: float


def bfgs_block(s, z, mu, grad, hess, zt):
    st = -grad
    mu_c = float(s @ z) / 3.0
    mu_t = float(st @ zt) / 3.0
    ds = s - mu_c * st
    dz = z - mu_c * zt
    dot_d = float(ds @ dz)
    nrm = float(np.linalg.norm(ds) * np.linalg.norm(dz))
    ha = mu * hess
    h1 = np.outer(s, s) / float(s @ z)
    h = None
    if dot_d > BFGS_GUARD * nrm and nrm > 0.0:
        zbar = np.column_stack([z, dz])
        haz = ha @ zbar
        m2 = zbar.T @ haz
        m2 = 0.5 * (m2 + m2.T)
        try:
            t3 = ha - haz @ np.linalg.solve(m2, haz.T)
            h = h1 + np.outer(ds, ds) / dot_d + t3
            h = 0.5 * (h + h.T)
            np.linalg.cholesky(h)
        except np.linalg.LinAlgError:
            h = None
    if h is None:
        haz = ha @ z
        h = ha - np.outer(haz, haz) / float(z @ haz) + h1
        h = 0.5 * (h + h.T)
        try:
            np.linalg.cholesky(h)
        except np.linalg.LinAlgError:
            h = 0.5 * (ha + ha.T)
            try:
                np.linalg.cholesky(h)
            except np.linalg.LinAlgError:
                raise ScalingFailure("nonsymmetric scaling block is not positive definite") from None
    return h, mu_c, mu_t


def nsym_scale(kind, a, s, z, mu) -> NsymScale:
    if kind == EXP:
        if not exp_primal_ok(s) or not exp_dual_ok(z):
            raise ScalingFailure("exponential block lost the cone interior")
        grad, hess, zt = exp_grad(z), exp_hess(z), exp_conj(s)
    else:
        if not pow_primal_ok(s, a) or not pow_dual_ok(z, a):
            raise ScalingFailure("power block lost the cone interior")
        grad, hess, zt = pow_grad(z, a), pow_hess(z, a), pow_conj(s, a)
    h, mu_c, mu_t = bfgs_block(s, z, mu, grad, hess, zt)
    return NsymScale(h, grad, hess, zt, mu_c, mu_t)


@dataclass
class ScalingSnapshot:
    lay: ConeLayout
    mu: float
    nn_h: np.ndarray
    nn_w: np.ndarray
    nn_lam: np.ndarray
    socs: list = field(default_factory=list)
    nsyms: list = field(default_factory=list)
    psds: list = field(default_factory=list)     # (r, rinv, lam)

    def kkt_blocks(self):
        diag = np.zeros(self.lay.zero_dim + self.lay.nonneg_dim)
        diag[self.lay.zero_dim:] = self.nn_h
        blocks = []
        for (off, d), sc in zip(self.lay.socs, self.socs):
            blocks.append((off, soc_block(sc, d)))
        offs = list(self.lay.exps) + [o for o, _ in self.lay.pows]
        for off, ns in zip(offs, self.nsyms):
            blocks.append((off, ns.h))
        for (off, side), (r, _, _) in zip(self.lay.psds, self.psds):
            blocks.append((off, congruence(r @ r.T)))
        return diag, blocks

    def dense(self) -> np.ndarray:
        h = np.zeros((self.lay.m, self.lay.m))
        diag, blocks = self.kkt_blocks()
        h[np.arange(len(diag)), np.arange(len(diag))] = diag
        for off, b in blocks:
            d = b.shape[0]
            h[off:off + d, off:off + d] = b
        return h


def update_scaling(lay: ConeLayout, s, z, mu) -> ScalingSnapshot:
    nn0, nnd = lay.nn0, lay.nonneg_dim
    sn, zn = s[nn0:nn0 + nnd], z[nn0:nn0 + nnd]
    if nnd and (np.any(sn <= 0.0) or np.any(zn <= 0.0)):
        raise ScalingFailure("nonnegative block lost the cone interior")
    st = ScalingSnapshot(lay, mu, sn / zn if nnd else np.zeros(0),
                         np.sqrt(sn / zn) if nnd else np.zeros(0),
                         np.sqrt(sn * zn) if nnd else np.zeros(0))
    for off, d in lay.socs:
        st.socs.append(soc_nt(s[off:off + d], z[off:off + d]))
    for kind, off, a in lay.nsym():
        st.nsyms.append(nsym_scale(kind, a, s[off:off + 3], z[off:off + 3], mu))
    for off, side in lay.psds:
        d = tri(side)
        st.psds.append(psd_nt(s[off:off + d], z[off:off + d], side))
    return st


def apply_h(st: ScalingSnapshot, v):
    lay = st.lay
    out = np.zeros_like(v)
    nn0, nnd = lay.nn0, lay.nonneg_dim
    out[nn0:nn0 + nnd] = st.nn_h * v[nn0:nn0 + nnd]
    for (off, d), sc in zip(lay.socs, st.socs):
        blk = v[off:off + d]
        jb = -blk.copy()
        jb[0] = blk[0]
        out[off:off + d] = sc.eta ** 2 * (2.0 * sc.w * float(sc.w @ blk) - jb)
    offs = list(lay.exps) + [o for o, _ in lay.pows]
    for off, ns in zip(offs, st.nsyms):
        out[off:off + 3] = ns.h @ v[off:off + 3]
    for (off, side), (r, _, _) in zip(lay.psds, st.psds):
        d = tri(side)
        q = r @ r.T
        out[off:off + d] = svec(q @ smat(v[off:off + d], side) @ q)
    return out


def combined_ds(st: ScalingSnapshot, s, z, dz_a, ds_a, sigma, mu):
    lay = st.lay
    out = np.zeros(lay.m)
    nn0, nnd = lay.nn0, lay.nonneg_dim
    if nnd:
        lam2 = s[nn0:nn0 + nnd] * z[nn0:nn0 + nnd]
        eta = ds_a[nn0:nn0 + nnd] * dz_a[nn0:nn0 + nnd]
        out[nn0:nn0 + nnd] = st.nn_w * (lam2 + eta - sigma * mu) / st.nn_lam
    for (off, d), sc in zip(lay.socs, st.socs):
        wi_ds = wbar_apply(sc.w, ds_a[off:off + d], inverse=True) / sc.eta
        w_dz = sc.eta * wbar_apply(sc.w, dz_a[off:off + d])
        rhs = jordan(sc.lam, sc.lam) + jordan(wi_ds, w_dz)
        rhs[0] -= sigma * mu
        out[off:off + d] = sc.eta * wbar_apply(sc.w, arrow_solve(sc.lam, rhs))
    for (kind, off, a), ns in zip(lay.nsym(), st.nsyms):
        zb, ub = z[off:off + 3], dz_a[off:off + 3]
        third = exp_third(zb, ub) if kind == EXP else pow_third(zb, ub, a)
        try:
            eta = -0.5 * third @ np.linalg.solve(ns.hess, ds_a[off:off + 3])
        except np.linalg.LinAlgError:
            eta = 0.0
        out[off:off + 3] = s[off:off + 3] + sigma * mu * ns.grad + eta
    for (off, side), (r, rinv, lam) in zip(lay.psds, st.psds):
        d = tri(side)
        a_m = rinv @ smat(ds_a[off:off + d], side) @ rinv.T
        b_m = r.T @ smat(dz_a[off:off + d], side) @ r
        eta_m = 0.5 * (a_m @ b_m + b_m @ a_m)
        rhs_m = np.diag(lam ** 2) + eta_m - sigma * mu * np.eye(side)
        u = 2.0 * rhs_m / np.add.outer(lam, lam)
        out[off:off + d] = svec(r @ u @ r.T)
    return out


def neighborhood_ok(lay: ConeLayout, s, z, mu, beta) -> bool:
    thresh = beta * mu
    nn0, nnd = lay.nn0, lay.nonneg_dim
    if nnd:
        sn, zn = s[nn0:nn0 + nnd], z[nn0:nn0 + nnd]
        if np.any(sn <= 0.0) or np.any(zn <= 0.0):
            raise DomainError("nonnegative block not strictly interior")
        with np.errstate(over="ignore", divide="ignore"):
            if nnd / float(np.sum(1.0 / (sn * zn))) < thresh:
                return False
    for off, d in lay.socs:
        sb, zb = s[off:off + d], z[off:off + d]
        rs, rz = soc_res(sb), soc_res(zb)
        if rs <= 0.0 or rz <= 0.0 or sb[0] <= 0.0 or zb[0] <= 0.0:
            raise DomainError("second-order block not strictly interior")
        if rs * rz / float(sb @ zb) < thresh:
            return False
    for kind, off, a in lay.nsym():
        if kind == EXP:
            zt = exp_conj(s[off:off + 3])
            st = -exp_grad(z[off:off + 3])
        else:
            zt = pow_conj(s[off:off + 3], a)
            st = -pow_grad(z[off:off + 3], a)
        if 3.0 / float(st @ zt) < thresh:
            return False
    for off, side in lay.psds:
        d = tri(side)
        try:
            si = np.linalg.inv(smat(s[off:off + d], side))
            zi = np.linalg.inv(smat(z[off:off + d], side))
        except np.linalg.LinAlgError:
            raise DomainError("PSD block not strictly interior") from None
        if side / float(np.sum(si * zi.T)) < thresh:
            return False
    return True


# ---------------------------------------------------------------------------
# step lengths
# ---------------------------------------------------------------------------

def ray_bound(v, dv) -> float:
    neg = dv < 0.0
    if not np.any(neg):
        return np.inf
    return float(np.min(-v[neg] / dv[neg]))


def soc_bound(v, dv) -> float:
    c = float(v[0] * v[0] - np.dot(v[1:], v[1:]))
    b = 2.0 * float(v[0] * dv[0] - np.dot(v[1:], dv[1:]))
    aa = float(dv[0] * dv[0] - np.dot(dv[1:], dv[1:]))
    roots = []
    if aa == 0.0:
        if b < 0.0:
            roots.append(-c / b)
    else:
        disc = b * b - 4.0 * aa * c
        if disc >= 0.0:
            sq = np.sqrt(disc)
            qq = -0.5 * (b + np.copysign(sq, b)) if b != 0.0 else 0.5 * sq * (1 if aa > 0 else -1)
            if qq != 0.0:
                roots.extend([qq / aa, c / qq])
            else:
                roots.append(0.0)
    pos = [r for r in roots if r > 0.0]
    bound = min(pos) if pos else np.inf
    if dv[0] < 0.0:
        bound = min(bound, -v[0] / dv[0])
    return bound


def nsym_feasible(lay: ConeLayout, s, z, ds, dz, alpha) -> bool:
    for off in lay.exps:
        st = s[off:off + 3] + alpha * ds[off:off + 3]
        zt = z[off:off + 3] + alpha * dz[off:off + 3]
        if not (exp_primal_ok(st) and exp_dual_ok(zt)):
            return False
    for off, a in lay.pows:
        st = s[off:off + 3] + alpha * ds[off:off + 3]
        zt = z[off:off + 3] + alpha * dz[off:off + 3]
        if not (pow_primal_ok(st, a) and pow_dual_ok(zt, a)):
            return False
    return True


def step_length(lay: ConeLayout, z, s, dz, ds, tau, kappa, dtau, dkappa,
                alpha_max=1.0, backtrack=0.8) -> float:
    alpha = alpha_max
    if dtau < 0.0:
        alpha = min(alpha, -tau / dtau)
    if dkappa < 0.0:
        alpha = min(alpha, -kappa / dkappa)
    nn0, nnd = lay.nn0, lay.nonneg_dim
    if nnd:
        alpha = min(alpha, ray_bound(z[nn0:nn0 + nnd], dz[nn0:nn0 + nnd]),
                    ray_bound(s[nn0:nn0 + nnd], ds[nn0:nn0 + nnd]))
    for off, d in lay.socs:
        alpha = min(alpha, soc_bound(z[off:off + d], dz[off:off + d]),
                    soc_bound(s[off:off + d], ds[off:off + d]))
    for off, side in lay.psds:
        d = tri(side)
        alpha = min(alpha, psd_step(z[off:off + d], dz[off:off + d], side),
                    psd_step(s[off:off + d], ds[off:off + d], side))
    if alpha < MIN_STEP:
        raise StepTooSmall(f"step length collapsed to {alpha:.3e}")
    if lay.exps or lay.pows:
        while alpha >= MIN_STEP:
            if nsym_feasible(lay, s, z, ds, dz, alpha):
                break
            alpha *= backtrack
        else:
            raise StepTooSmall("backtracking line search fell below the minimum step")
    return float(alpha)


def soc_residuals_fixed_order(dims, offsets, x) -> np.ndarray:
    """t² − Σu² with the reference's chunks-of-8 + pairwise tree order (steps.py:136-175)."""
    out = np.empty(len(dims))
    for i, (off, d) in enumerate(zip(offsets, dims)):
        nu = d - 1
        parts = []
        for c in range((nu + 7) // 8):
            lo = off + 1 + 8 * c
            hi = min(lo + 8, off + 1 + nu)
            acc = 0.0
            for k in range(lo, hi):
                acc = acc + x[k] * x[k]
            parts.append(acc)
        while len(parts) > 1:
            nxt = [parts[2 * c] + parts[2 * c + 1] for c in range(len(parts) // 2)]
            if len(parts) % 2 == 1:
                nxt.append(parts[-1])
            parts = nxt
        t = x[off]
        out[i] = t * t - parts[0] if nu > 0 else t * t
    return out
