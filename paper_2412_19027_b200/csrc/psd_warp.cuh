// PSD-cone dense kernels: a lane GROUP per cone — G = 8, 16 or 32 lanes (the
// smallest power of two >= the largest side, so 4, 2 or 1 cones per warp) —
// lane i of a group owns row i of every n x n matrix of its cone; the matrices
// live in the group's shared-memory slice (row-major, leading dimension
// ld = n_max | 1), reductions are fixed-order xor shuffles inside the group, and
// every loop that contains a shuffle or a warp barrier runs to the warp-uniform
// bound (the largest side of the warp's cones) so the groups stay in lockstep.
// Restates cones/psdcone.py:21-133 and the PSD parts of cones/scaling.py: NT
// factor via Cholesky + one-sided Jacobi SVD of Lz' Ls, congruence H = Q (x)s Q,
// step to the boundary via the minimum eigenvalue of L^-1 dS L^-T, neighbourhood
// trace tr(S^-1 Z^-1).  svec = column-major lower triangle, sqrt(2) off-diagonal.
#pragma once
#include <cmath>

namespace cipm {

namespace pw {

constexpr double kR2 = 1.4142135623730951;

// per-lane view of the group: row index, own side, warp-uniform side bound, group width
struct Grp {
    int i;      // lane within the group (= row)
    int n;      // side of this group's cone (0 when the group has no cone)
    int nu;     // largest side over the warp's groups (uniform loop bound)
    int g;      // group width
};

__device__ __forceinline__ int svec_index(int i, int j, int n) {   // i >= j
    return j * n - j * (j - 1) / 2 + (i - j);
}

__device__ __forceinline__ double gsum(double v, int g) {
    for (int o = g >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double gmin(double v, int g) {
    for (int o = g >> 1; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// X = smat(v) (full symmetric)
__device__ __forceinline__ void smat(const Grp& G, const double* v, double* X, int ld) {
    const int i = G.i, n = G.n;
    if (i < n)
        for (int j = 0; j < n; ++j) {
            const int a = i > j ? i : j, b = i > j ? j : i;
            const double e = v[svec_index(a, b, n)];
            X[i * ld + j] = a == b ? e : e / kR2;
        }
    __syncwarp();
}

// v = svec(X) (lower triangle of X)
__device__ __forceinline__ void svec(const Grp& G, const double* X, int ld, double* v) {
    const int i = G.i, n = G.n;
    if (i < n)
        for (int j = 0; j <= i; ++j) v[svec_index(i, j, n)] = i == j ? X[i * ld + i] : kR2 * X[i * ld + j];
    __syncwarp();
}

// lower Cholesky in place (upper part zeroed); false if not positive definite
__device__ __forceinline__ bool chol(const Grp& G, double* A, int ld) {
    const int i = G.i, n = G.n;
    bool ok = true;
    for (int j = 0; j < G.nu; ++j) {
        const bool act = j < n;
        const double d = act ? A[j * ld + j] : 1.0;
        if (act && !(d > 0.0)) ok = false;
        const double l = sqrt(d);
        __syncwarp();
        if (act && i == j) A[j * ld + j] = l;
        if (act && i > j && i < n) A[i * ld + j] = A[i * ld + j] / l;
        __syncwarp();
        if (act && i > j && i < n) {
            const double lij = A[i * ld + j];
            for (int c = j + 1; c <= i; ++c) A[i * ld + c] -= lij * A[c * ld + j];
        }
        __syncwarp();
    }
    if (i < n)
        for (int c = i + 1; c < n; ++c) A[i * ld + c] = 0.0;
    __syncwarp();
    // the group's verdict (lanes beyond n report true)
    for (int o = G.g >> 1; o > 0; o >>= 1) ok = ok && __shfl_xor_sync(0xffffffffu, (int)ok, o);
    return ok;
}

// C = op(A) op(B): op 0 = A B, 1 = A' B, 2 = A B'  (C must not alias A or B)
__device__ __forceinline__ void mm(const Grp& G, const double* A, const double* B, int ld, double* C, int op) {
    const int i = G.i, n = G.n;
    if (i < n)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) {
                const double a = op == 1 ? A[k * ld + i] : A[i * ld + k];
                const double b = op == 2 ? B[j * ld + k] : B[k * ld + j];
                acc += a * b;
            }
            C[i * ld + j] = acc;
        }
    __syncwarp();
}

// Li = L^-1 (lower), column-parallel forward substitution (lane j = column j)
__device__ __forceinline__ void tri_inv(const Grp& G, const double* L, int ld, double* Li) {
    const int j = G.i, n = G.n;
    if (j < n) {
        for (int i = 0; i < j; ++i) Li[i * ld + j] = 0.0;
        for (int i = j; i < n; ++i) {
            double v = i == j ? 1.0 : 0.0;
            for (int k = j; k < i; ++k) v -= L[i * ld + k] * Li[k * ld + j];
            Li[i * ld + j] = v / L[i * ld + i];
        }
    }
    __syncwarp();
}

// one-sided cyclic Jacobi: U <- U V with orthogonal columns, sig = column norms
__device__ __forceinline__ void jacobi_svd(const Grp& G, double* U, int ld, double* V, double* sig) {
    const int k = G.i, n = G.n;
    if (k < n)
        for (int c = 0; c < n; ++c) V[k * ld + c] = k == c ? 1.0 : 0.0;
    __syncwarp();
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rot = false;
        for (int p = 0; p < G.nu - 1; ++p)
            for (int q = p + 1; q < G.nu; ++q) {
                const bool act = q < n;
                const double up = (act && k < n) ? U[k * ld + p] : 0.0, uq = (act && k < n) ? U[k * ld + q] : 0.0;
                const double al = gsum(up * up, G.g), be = gsum(uq * uq, G.g), ga = gsum(up * uq, G.g);
                if (!act || fabs(ga) <= 1e-15 * sqrt(al * be) || ga == 0.0) continue;
                rot = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                if (k < n) {
                    U[k * ld + p] = c * up - s * uq;
                    U[k * ld + q] = s * up + c * uq;
                    const double vp = V[k * ld + p], vq = V[k * ld + q];
                    V[k * ld + p] = c * vp - s * vq;
                    V[k * ld + q] = s * vp + c * vq;
                }
            }
        __syncwarp();
        if (!__any_sync(0xffffffffu, rot)) break;
    }
    for (int c = 0; c < G.nu; ++c) {
        const double u = (k < n && c < n) ? U[k * ld + c] : 0.0;
        const double s2 = gsum(u * u, G.g);
        if (k == 0 && c < n) sig[c] = sqrt(s2);
    }
    __syncwarp();
}

// cyclic two-sided Jacobi eigenvalues of a symmetric matrix (A overwritten); min eigenvalue
__device__ __forceinline__ double sym_min_eig(const Grp& G, double* A, int ld) {
    const int k = G.i, n = G.n;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        if (k < n)
            for (int j = 0; j < n; ++j) {
                const double a2 = A[k * ld + j] * A[k * ld + j];
                tot += a2;
                if (j != k) off += a2;
            }
        off = gsum(off, G.g);
        tot = gsum(tot, G.g);
        const bool done = n == 0 || off <= 1e-32 * tot || off == 0.0;
        if (__all_sync(0xffffffffu, done)) break;
        for (int p = 0; p < G.nu - 1; ++p)
            for (int q = p + 1; q < G.nu; ++q) {
                const bool act = !done && q < n;
                const double apq = act ? A[p * ld + q] : 0.0;
                double c = 1.0, s = 0.0;
                const bool rot = act && apq != 0.0;
                if (rot) {
                    const double app = A[p * ld + p], aqq = A[q * ld + q];
                    const double theta = (aqq - app) / (2.0 * apq);
                    const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                    c = 1.0 / sqrt(1.0 + t * t);
                    s = t * c;
                }
                __syncwarp();
                if (rot && k < n) {                      // columns p, q
                    const double akp = A[k * ld + p], akq = A[k * ld + q];
                    A[k * ld + p] = c * akp - s * akq;
                    A[k * ld + q] = s * akp + c * akq;
                }
                __syncwarp();
                if (rot && k < n) {                      // rows p, q
                    const double apk = A[p * ld + k], aqk = A[q * ld + k];
                    A[p * ld + k] = c * apk - s * aqk;
                    A[q * ld + k] = s * apk + c * aqk;
                }
                __syncwarp();
                if (rot && k == 0) { A[p * ld + q] = 0.0; A[q * ld + p] = 0.0; }
            }
        __syncwarp();
    }
    return gmin(k < n ? A[k * ld + k] : INFINITY, G.g);
}

// Same eigenvalues by parallel-ordered two-sided Jacobi: a sweep is mu - 1 rounds
// of the round-robin tournament over mu = nu rounded up to even indices; the
// rotations of one round act on disjoint index pairs, so they are applied
// together (all column pairs, then all row pairs) — the sequential chain per
// sweep is mu - 1 rotation solves instead of mu (mu - 1) / 2.  The rotation of
// each pair is the cyclic one (same angle formula, zeroes its a_pq), and the
// stopping test is the same.  scr: 3 * mu doubles of the group's slice.
__device__ __forceinline__ double sym_min_eig_par(const Grp& G, double* A, int ld, double* scr) {
    const int k = G.i, n = G.n;
    const int mu = (G.nu + 1) & ~1, m1 = mu - 1, half = mu >> 1;
    double* pc = scr;
    double* ps = scr + mu;
    int* pq = reinterpret_cast<int*>(scr + 2 * mu);
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        if (k < n)
            for (int j = 0; j < n; ++j) {
                const double a2 = A[k * ld + j] * A[k * ld + j];
                tot += a2;
                if (j != k) off += a2;
            }
        off = gsum(off, G.g);
        tot = gsum(tot, G.g);
        const bool done = n == 0 || off <= 1e-32 * tot || off == 0.0;
        if (__all_sync(0xffffffffu, done)) break;
        for (int rnd = 0; rnd < m1; ++rnd) {
            // partner of index k in round rnd (index mu - 1 is the fixed player)
            int q = -1;
            if (k < mu) {
                if (k == mu - 1) q = (rnd * half) % m1;
                else {
                    q = ((rnd - k) % m1 + m1) % m1;
                    if (q == k) q = mu - 1;
                }
            }
            double c = 1.0, sn = 0.0;
            if (k < mu) {
                const int p0 = k < q ? k : q, q0 = k < q ? q : k;
                const bool act = !done && q0 < n;
                const double apq = act ? A[p0 * ld + q0] : 0.0;
                if (act && apq != 0.0) {
                    const double app = A[p0 * ld + p0], aqq = A[q0 * ld + q0];
                    const double theta = (aqq - app) / (2.0 * apq);
                    const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                    c = 1.0 / sqrt(1.0 + t * t);
                    sn = t * c;
                }
                pc[k] = c;
                ps[k] = sn;
                pq[2 * k] = q;
            }
            __syncwarp();
            if (!done && k < n) {                       // columns: A[k][p], A[k][q] for every pair
                for (int p = 0; p < n; ++p) {
                    const int qq = pq[2 * p];
                    if (qq <= p || qq >= n) continue;
                    const double cc = pc[p], ss = ps[p];
                    const double akp = A[k * ld + p], akq = A[k * ld + qq];
                    A[k * ld + p] = cc * akp - ss * akq;
                    A[k * ld + qq] = ss * akp + cc * akq;
                }
            }
            __syncwarp();
            if (!done && k < n) {                       // rows: A[p][k], A[q][k] for every pair
                for (int p = 0; p < n; ++p) {
                    const int qq = pq[2 * p];
                    if (qq <= p || qq >= n) continue;
                    const double cc = pc[p], ss = ps[p];
                    const double apk = A[p * ld + k], aqk = A[qq * ld + k];
                    A[p * ld + k] = cc * apk - ss * aqk;
                    A[qq * ld + k] = ss * apk + cc * aqk;
                }
            }
            __syncwarp();
            if (!done && k < n && q > k && q < n && ps[k] != 0.0) {   // the rotated pairs' a_pq = 0
                A[k * ld + q] = 0.0;
                A[q * ld + k] = 0.0;
            }
            __syncwarp();
        }
    }
    return gmin(k < n ? A[k * ld + k] : INFINITY, G.g);
}

// NT factor (psdcone.py:98-117): R = Ls V diag(sig^-1/2), R^-1 = diag(sig^1/2) V' Ls^-1,
// lam = sig; uses the work matrices W0..W3 of the group slice
__device__ __forceinline__ bool nt_factor(const Grp& G, const double* s, const double* z, int ld, double* W0,
                                          double* W1, double* W2, double* W3, double* R, double* Rinv, double* lam) {
    if (G.n > 0) smat(G, s, W0, ld);
    else __syncwarp();
    bool ok = chol(G, W0, ld);                     // Ls
    if (G.n > 0) smat(G, z, W1, ld);
    else __syncwarp();
    ok = chol(G, W1, ld) && ok;                    // Lz
    Grp H = G;                                     // a failed group idles through the rest
    if (!ok) H.n = 0;
    const int i = H.i, n = H.n;
    mm(H, W1, W0, ld, W2, 1);                      // M = Lz' Ls
    jacobi_svd(H, W2, ld, W3, lam);                // V in W3, sig in lam
    bool pos = true;
    for (int c = 0; c < n; ++c) pos = pos && lam[c] > 0.0;
    ok = ok && pos;
    mm(H, W0, W3, ld, R, 0);                       // Ls V
    if (i < n)
        for (int c = 0; c < n; ++c) R[i * ld + c] /= sqrt(lam[c]);
    __syncwarp();
    tri_inv(H, W0, ld, W1);                        // Ls^-1
    mm(H, W3, W1, ld, Rinv, 1);                    // V' Ls^-1
    if (i < n) {
        const double sq = sqrt(lam[i]);
        for (int c = 0; c < n; ++c) Rinv[i * ld + c] *= sq;
    }
    __syncwarp();
    return ok;
}

}  // namespace pw
}  // namespace cipm
