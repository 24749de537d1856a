// Exponential / power cone device math (thread per cone).
//
// Restates cones/barriers.py (dual barriers, third-order terms, conjugate
// points via ×10 bracketing + Brent) and the rank-3 BFGS scaling with its
// fallback chain from cones/scaling.py:112-175.  Brent is scipy's brentq
// (the function the reference calls, barriers.py:298-302) restated for the
// device with the same xtol / rtol / maxiter.
#pragma once
#include <cmath>

namespace cipm {

constexpr double kBfgsGuard = 1e-8;
constexpr int kConjMaxIters = 100;

struct V3 { double v[3]; };
struct M3 { double a[9]; };   // row-major

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// ---- predicates (barriers.py:82-86, 147-151, 170-175, 248-252) ----
__device__ __forceinline__ bool exp_dual_ok(const double* z) {
    if (z[0] >= 0.0 || z[2] <= 0.0) return false;
    return z[1] - z[0] - z[0] * log(z[2] / -z[0]) > 0.0;
}
__device__ __forceinline__ bool exp_primal_ok(const double* s) {
    if (s[1] <= 0.0 || s[2] <= 0.0) return false;
    return s[1] * log(s[2] / s[1]) - s[0] > 0.0;
}
__device__ __forceinline__ bool pow_dual_ok(const double* z, double a) {
    if (z[0] <= 0.0 || z[1] <= 0.0) return false;
    double lw = 2.0 * a * log(z[0] / a) + 2.0 * (1.0 - a) * log(z[1] / (1.0 - a));
    return exp(lw) - z[2] * z[2] > 0.0;
}
__device__ __forceinline__ bool pow_primal_ok(const double* s, double a) {
    if (s[0] <= 0.0 || s[1] <= 0.0) return false;
    return exp(2.0 * a * log(s[0]) + 2.0 * (1.0 - a) * log(s[1])) - s[2] * s[2] > 0.0;
}
// strict membership used by take_step (cones/set.py:125-163)
__device__ __forceinline__ bool exp_member(const double* s) {
    return s[1] > 0.0 && s[2] > 0.0 && log(s[1]) + s[0] / s[1] < log(s[2]);
}
__device__ __forceinline__ bool exp_dual_member(const double* z) {
    return z[0] < 0.0 && z[2] > 0.0 && log(-z[0]) + z[1] / z[0] < 1.0 + log(z[2]);
}
__device__ __forceinline__ bool pow_member(double x, double y, double zz, double a) {
    if (x <= 0.0 || y <= 0.0) return false;
    if (zz == 0.0) return true;
    return a * log(x) + (1.0 - a) * log(y) > log(fabs(zz));
}

// ---- exp dual barrier (barriers.py:89-144) ----
struct ExpTerms { double z1, z2, z3, l, psi; bool ok; };
__device__ __forceinline__ ExpTerms exp_terms(const double* z) {
    ExpTerms t;
    t.z1 = z[0]; t.z2 = z[1]; t.z3 = z[2];
    t.ok = !(t.z1 >= 0.0 || t.z3 <= 0.0);
    if (!t.ok) return t;
    t.l = log(t.z3 / -t.z1);
    t.psi = t.z2 - t.z1 - t.z1 * t.l;
    t.ok = t.psi > 0.0;
    return t;
}
__device__ inline bool exp_grad(const double* z, double* g) {
    ExpTerms t = exp_terms(z);
    if (!t.ok) return false;
    double r = 1.0 / t.psi;
    g[0] = r * t.l - 1.0 / t.z1;
    g[1] = -r;
    g[2] = r * t.z1 / t.z3 - 1.0 / t.z3;
    return true;
}
__device__ inline bool exp_hess(const double* z, double* h) {
    ExpTerms t = exp_terms(z);
    if (!t.ok) return false;
    double r = 1.0 / t.psi;
    double g[3] = {-t.l, 1.0, -t.z1 / t.z3};
    double hp[9] = {1.0 / t.z1, 0.0, -1.0 / t.z3, 0.0, 0.0, 0.0, -1.0 / t.z3, 0.0, t.z1 / (t.z3 * t.z3)};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) h[3 * i + j] = r * r * (g[i] * g[j]) - r * hp[3 * i + j];
    h[0] += 1.0 / (t.z1 * t.z1);
    h[8] += 1.0 / (t.z3 * t.z3);
    return true;
}
__device__ inline bool exp_third(const double* z, const double* u, double* out) {
    ExpTerms t = exp_terms(z);
    if (!t.ok) return false;
    double u1 = u[0], u3 = u[2];
    double r = 1.0 / t.psi;
    double g[3] = {-t.l, 1.0, -t.z1 / t.z3};
    double hp[9] = {1.0 / t.z1, 0.0, -1.0 / t.z3, 0.0, 0.0, 0.0, -1.0 / t.z3, 0.0, t.z1 / (t.z3 * t.z3)};
    double z33 = t.z3 * t.z3;
    double tu[9] = {-u1 / (t.z1 * t.z1), 0.0, u3 / z33, 0.0, 0.0, 0.0, u3 / z33, 0.0,
                    u1 / z33 - 2.0 * t.z1 * u3 / (t.z3 * t.z3 * t.z3)};
    double gu = g[0] * u[0] + g[1] * u[1] + g[2] * u[2];
    double hu[3];
    for (int i = 0; i < 3; ++i) hu[i] = hp[3 * i] * u[0] + hp[3 * i + 1] * u[1] + hp[3 * i + 2] * u[2];
    double r3 = r * r * r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = -2.0 * r3 * gu * (g[i] * g[j]);
            v += r * r * ((hu[i] * g[j] + g[i] * hu[j]) + gu * hp[3 * i + j]);
            v -= r * tu[3 * i + j];
            out[3 * i + j] = v;
        }
    out[0] += -2.0 * u1 / (t.z1 * t.z1 * t.z1);
    out[8] += -2.0 * u3 / (t.z3 * t.z3 * t.z3);
    return true;
}

// ---- pow dual barrier (barriers.py:178-245) ----
struct PowTerms { double z1, z2, z3, b, om, phi; bool ok; };
__device__ __forceinline__ PowTerms pow_terms(const double* z, double a) {
    PowTerms t;
    t.z1 = z[0]; t.z2 = z[1]; t.z3 = z[2];
    t.ok = !(t.z1 <= 0.0 || t.z2 <= 0.0);
    if (!t.ok) return t;
    t.b = 1.0 - a;
    t.om = exp(2.0 * a * log(t.z1 / a) + 2.0 * t.b * log(t.z2 / t.b));
    t.phi = t.om - t.z3 * t.z3;
    t.ok = t.phi > 0.0;
    return t;
}
__device__ __forceinline__ void pow_hphi(const PowTerms& t, double a, double* hp) {
    hp[0] = 2.0 * a * (2 * a - 1) * t.om / (t.z1 * t.z1);
    hp[1] = 4.0 * a * t.b * t.om / (t.z1 * t.z2);
    hp[2] = 0.0;
    hp[3] = hp[1];
    hp[4] = 2.0 * t.b * (2 * t.b - 1) * t.om / (t.z2 * t.z2);
    hp[5] = 0.0;
    hp[6] = 0.0; hp[7] = 0.0; hp[8] = -2.0;
}
__device__ inline bool pow_grad(const double* z, double a, double* g) {
    PowTerms t = pow_terms(z, a);
    if (!t.ok) return false;
    double r = 1.0 / t.phi;
    double gp[3] = {2.0 * a * t.om / t.z1, 2.0 * t.b * t.om / t.z2, -2.0 * t.z3};
    double add[3] = {-t.b / t.z1, -a / t.z2, 0.0};
    for (int i = 0; i < 3; ++i) g[i] = -r * gp[i] + add[i];
    return true;
}
__device__ inline bool pow_hess(const double* z, double a, double* h) {
    PowTerms t = pow_terms(z, a);
    if (!t.ok) return false;
    double r = 1.0 / t.phi;
    double gp[3] = {2.0 * a * t.om / t.z1, 2.0 * t.b * t.om / t.z2, -2.0 * t.z3};
    double hp[9];
    pow_hphi(t, a, hp);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) h[3 * i + j] = r * r * (gp[i] * gp[j]) - r * hp[3 * i + j];
    h[0] += t.b / (t.z1 * t.z1);
    h[4] += a / (t.z2 * t.z2);
    return true;
}
__device__ inline bool pow_third(const double* z, const double* u, double a, double* out) {
    PowTerms t = pow_terms(z, a);
    if (!t.ok) return false;
    double u1 = u[0], u2 = u[1];
    double r = 1.0 / t.phi;
    double b = t.b, om = t.om, z1 = t.z1, z2 = t.z2;
    double gp[3] = {2.0 * a * om / z1, 2.0 * b * om / z2, -2.0 * t.z3};
    double hp[9];
    pow_hphi(t, a, hp);
    double p111 = 2 * a * (2 * a - 1) * (2 * a - 2) * om / (z1 * z1 * z1);
    double p112 = 4 * a * (2 * a - 1) * b * om / (z1 * z1 * z2);
    double p122 = 4 * a * b * (2 * b - 1) * om / (z1 * z2 * z2);
    double p222 = 2 * b * (2 * b - 1) * (2 * b - 2) * om / (z2 * z2 * z2);
    double tu[9] = {p111 * u1 + p112 * u2, p112 * u1 + p122 * u2, 0.0,
                    p112 * u1 + p122 * u2, p122 * u1 + p222 * u2, 0.0, 0.0, 0.0, 0.0};
    double gu = gp[0] * u[0] + gp[1] * u[1] + gp[2] * u[2];
    double hu[3];
    for (int i = 0; i < 3; ++i) hu[i] = hp[3 * i] * u[0] + hp[3 * i + 1] * u[1] + hp[3 * i + 2] * u[2];
    double r3 = r * r * r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = -2.0 * r3 * gu * (gp[i] * gp[j]);
            v += r * r * ((hu[i] * gp[j] + gp[i] * hu[j]) + gu * hp[3 * i + j]);
            v -= r * tu[3 * i + j];
            out[3 * i + j] = v;
        }
    out[0] += -2.0 * b * u1 / (z1 * z1 * z1);
    out[4] += -2.0 * a * u2 / (z2 * z2 * z2);
    return true;
}

// ---- conjugate points: scalar monotone equations + scipy brentq ----
struct ConjFn {
    int kind;          // 0 exp, 1 pow
    double s1, s2, s3, a, b, cst;
    __device__ double operator()(double t) const {
        if (kind == 0) return s2 * (log1p(s2 * t) - log(s3 * t)) + 1.0 / t + s1;
        double u = 1.0 + t;
        return 2.0 * a * log(2.0 * a * u + b) + 2.0 * b * log(2.0 * b * u + a) - log(u) - log(t) + cst;
    }
};

// scipy/optimize/Zeros/brentq.c semantics (xtol, rtol, maxiter)
__device__ inline double brentq(const ConjFn& f, double xa, double xb, double xtol, double rtol, int iter, bool* ok) {
    double xpre = xa, xcur = xb, xblk = 0.0, fpre, fcur, fblk = 0.0, spre = 0.0, scur = 0.0, sbis;
    double delta, stry, dpre, dblk;
    *ok = true;
    fpre = f(xpre);
    fcur = f(xcur);
    if (fpre == 0) return xpre;
    if (fcur == 0) return xcur;
    if (signbit(fpre) == signbit(fcur)) { *ok = false; return 0.0; }
    for (int i = 0; i < iter; i++) {
        if (fpre != 0 && fcur != 0 && (signbit(fpre) != signbit(fcur))) {
            xblk = xpre;
            fblk = fpre;
            spre = scur = xcur - xpre;
        }
        if (fabs(fblk) < fabs(fcur)) {
            xpre = xcur; xcur = xblk; xblk = xpre;
            fpre = fcur; fcur = fblk; fblk = fpre;
        }
        delta = (xtol + rtol * fabs(xcur)) / 2;
        sbis = (xblk - xcur) / 2;
        if (fcur == 0 || fabs(sbis) < delta) return xcur;
        if (fabs(spre) > delta && fabs(fcur) < fabs(fpre)) {
            if (xpre == xblk) {
                stry = -fcur * (xcur - xpre) / (fcur - fpre);
            } else {
                dpre = (fpre - fcur) / (xpre - xcur);
                dblk = (fblk - fcur) / (xblk - xcur);
                stry = -fcur * (fblk * dblk - fpre * dpre) / (dblk * dpre * (fblk - fpre));
            }
            if (2 * fabs(stry) < fmin(fabs(spre), 3 * fabs(sbis) - delta)) {
                spre = scur;
                scur = stry;
            } else {
                spre = sbis;
                scur = sbis;
            }
        } else {
            spre = sbis;
            scur = sbis;
        }
        xpre = xcur;
        fpre = fcur;
        if (fabs(scur) > delta) xcur += scur;
        else xcur += (sbis > 0 ? delta : -delta);
        fcur = f(xcur);
    }
    *ok = false;     // scipy raises RuntimeError("Failed to converge")
    return xcur;
}

// root of a decreasing f on (0, inf): ×10 bracketing then Brent (barriers.py:280-302)
__device__ inline bool solve_decreasing(const ConjFn& f, double t0, double* root) {
    double lo = t0, hi = t0;
    int i;
    for (i = 0; i < kConjMaxIters; ++i) {
        if (f(lo) > 0.0) break;
        lo /= 10.0;
        if (lo < 1e-300) return false;
    }
    for (i = 0; i < kConjMaxIters; ++i) {
        if (f(hi) < 0.0) break;
        hi *= 10.0;
        if (hi > 1e300) return false;
    }
    bool ok;
    *root = brentq(f, lo, hi, 1e-300, 4.0 * 2.220446049250313e-16, kConjMaxIters, &ok);
    return ok;
}

// w = -∇f*(s): returns 0 ok, CIPM_E_DOMAIN if s is not interior, CIPM_E_SCALING on bracket failure
__device__ inline int exp_conj(const double* s, double* w) {
    if (!exp_primal_ok(s)) return CIPM_E_DOMAIN;
    ConjFn f;
    f.kind = 0; f.s1 = s[0]; f.s2 = s[1]; f.s3 = s[2]; f.a = f.b = f.cst = 0.0;
    double t;
    if (!solve_decreasing(f, 1.0 / (1.0 + fabs(s[0]) + s[1] + s[2]), &t)) return CIPM_E_SCALING;
    double w1 = -t;
    double w3 = (1.0 + s[1] * t) / s[2];
    double w2 = 1.0 / s[1] + w1 + w1 * log(w3 / t);
    w[0] = w1; w[1] = w2; w[2] = w3;
    return 0;
}

__device__ inline int pow_conj(const double* s, double a, double* w) {
    if (!pow_primal_ok(s, a)) return CIPM_E_DOMAIN;
    double b = 1.0 - a;
    if (s[2] == 0.0) {
        w[0] = (1.0 + a) / s[0]; w[1] = (2.0 - a) / s[1]; w[2] = 0.0;
        return 0;
    }
    ConjFn f;
    f.kind = 1; f.s1 = s[0]; f.s2 = s[1]; f.s3 = s[2]; f.a = a; f.b = b;
    f.cst = (2.0 * log(fabs(s[2])) - 2.0 * a * log(a * s[0]) - 2.0 * b * log(b * s[1])) - log(4.0);
    double v;
    if (!solve_decreasing(f, 1.0, &v)) return CIPM_E_SCALING;
    double u = 1.0 + v;
    w[0] = (2.0 * a * u + b) / s[0];
    w[1] = (2.0 * b * u + a) / s[1];
    w[2] = -2.0 * v / s[2];
    return 0;
}

// ---- small dense helpers ----
// LAPACK dpotrf-style PD test of a symmetric 3x3 (lower triangle read)
__device__ inline bool chol3_ok(const double* h) {
    double l[9] = {0};
    for (int j = 0; j < 3; ++j) {
        double ajj = h[3 * j + j];
        for (int k = 0; k < j; ++k) ajj -= l[3 * j + k] * l[3 * j + k];
        if (!(ajj > 0.0)) return false;
        ajj = sqrt(ajj);
        l[3 * j + j] = ajj;
        for (int i = j + 1; i < 3; ++i) {
            double v = h[3 * i + j];
            for (int k = 0; k < j; ++k) v -= l[3 * i + k] * l[3 * j + k];
            l[3 * i + j] = v / ajj;
        }
    }
    return true;
}

// LU with partial pivoting (dgesv) of an n x n (n <= 3) system with nrhs columns;
// returns false on an exactly zero pivot (LinAlgError)
__device__ inline bool lu_solve(double* a, int n, double* bm, int nrhs) {
    int piv[3];
    for (int k = 0; k < n; ++k) {
        int p = k;
        double mx = fabs(a[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (fabs(a[i * n + k]) > mx) { mx = fabs(a[i * n + k]); p = i; }
        piv[k] = p;
        if (a[p * n + k] == 0.0) return false;
        if (p != k) {
            for (int j = 0; j < n; ++j) { double t = a[k * n + j]; a[k * n + j] = a[p * n + j]; a[p * n + j] = t; }
        }
        for (int i = k + 1; i < n; ++i) {
            a[i * n + k] /= a[k * n + k];
            for (int j = k + 1; j < n; ++j) a[i * n + j] -= a[i * n + k] * a[k * n + j];
        }
    }
    for (int c = 0; c < nrhs; ++c) {
        for (int k = 0; k < n; ++k) {
            int p = piv[k];
            if (p != k) { double t = bm[k * nrhs + c]; bm[k * nrhs + c] = bm[p * nrhs + c]; bm[p * nrhs + c] = t; }
        }
        for (int i = 1; i < n; ++i)
            for (int k = 0; k < i; ++k) bm[i * nrhs + c] -= a[i * n + k] * bm[k * nrhs + c];
        for (int i = n - 1; i >= 0; --i) {
            double v = bm[i * nrhs + c];
            for (int k = i + 1; k < n; ++k) v -= a[i * n + k] * bm[k * nrhs + c];
            bm[i * nrhs + c] = v / a[i * n + i];
        }
    }
    return true;
}

// rank-3 BFGS scaling with fallbacks (scaling.py:112-156); returns false on ScalingFailure
__device__ inline bool bfgs_block(const double* s, const double* z, double mu, const double* grad,
                                  const double* hess, const double* zt, double* h) {
    double st[3] = {-grad[0], -grad[1], -grad[2]};
    double sz = dot3(s, z);
    double mu_c = sz / 3.0;
    double ds[3], dz[3];
    for (int i = 0; i < 3; ++i) { ds[i] = s[i] - mu_c * st[i]; dz[i] = z[i] - mu_c * zt[i]; }
    double dot_d = dot3(ds, dz);
    double nrm = sqrt(dot3(ds, ds)) * sqrt(dot3(dz, dz));
    double ha[9], h1[9];
    for (int i = 0; i < 9; ++i) ha[i] = mu * hess[i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) h1[3 * i + j] = (s[i] * s[j]) / sz;
    bool have = false;
    if (dot_d > kBfgsGuard * nrm && nrm > 0.0) {
        double haz[6];   // 3x2: columns ha@z, ha@dz
        for (int i = 0; i < 3; ++i) {
            haz[2 * i] = ha[3 * i] * z[0] + ha[3 * i + 1] * z[1] + ha[3 * i + 2] * z[2];
            haz[2 * i + 1] = ha[3 * i] * dz[0] + ha[3 * i + 1] * dz[1] + ha[3 * i + 2] * dz[2];
        }
        double zb[6] = {z[0], dz[0], z[1], dz[1], z[2], dz[2]};   // 3x2
        double m2[4];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                m2[2 * a + b] = zb[a] * haz[b] + zb[2 + a] * haz[2 + b] + zb[4 + a] * haz[4 + b];
        double off = 0.5 * (m2[1] + m2[2]);
        m2[0] = 0.5 * (m2[0] + m2[0]);
        m2[3] = 0.5 * (m2[3] + m2[3]);
        m2[1] = off;
        m2[2] = off;
        double X[6];   // 2x3 = haz^T
        for (int a = 0; a < 2; ++a)
            for (int j = 0; j < 3; ++j) X[3 * a + j] = haz[2 * j + a];
        if (lu_solve(m2, 2, X, 3)) {
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double t3 = ha[3 * i + j] - (haz[2 * i] * X[j] + haz[2 * i + 1] * X[3 + j]);
                    h[3 * i + j] = (h1[3 * i + j] + (ds[i] * ds[j]) / dot_d) + t3;
                }
            for (int i = 0; i < 3; ++i)
                for (int j = i + 1; j < 3; ++j) {
                    double v = 0.5 * (h[3 * i + j] + h[3 * j + i]);
                    h[3 * i + j] = v;
                    h[3 * j + i] = v;
                }
            for (int i = 0; i < 3; ++i) h[4 * i] = 0.5 * (h[4 * i] + h[4 * i]);
            have = chol3_ok(h);
        }
    }
    if (!have) {
        double hz[3];
        for (int i = 0; i < 3; ++i) hz[i] = ha[3 * i] * z[0] + ha[3 * i + 1] * z[1] + ha[3 * i + 2] * z[2];
        double zhz = dot3(z, hz);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) h[3 * i + j] = (ha[3 * i + j] - (hz[i] * hz[j]) / zhz) + h1[3 * i + j];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j <= i; ++j) {
                double v = 0.5 * (h[3 * i + j] + h[3 * j + i]);
                h[3 * i + j] = v;
                h[3 * j + i] = v;
            }
        if (!chol3_ok(h)) {
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j <= i; ++j) {
                    double v = 0.5 * (ha[3 * i + j] + ha[3 * j + i]);
                    h[3 * i + j] = v;
                    h[3 * j + i] = v;
                }
            if (!chol3_ok(h)) return false;
        }
    }
    return true;
}

}  // namespace cipm
