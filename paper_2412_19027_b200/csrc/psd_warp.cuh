// PSD-cone dense kernels, one warp per cone, side n <= 32: lane i owns row i of
// every n x n matrix, the matrices live in the warp's shared-memory slice
// (row-major, leading dimension ld = n_max | 1 so a column walk is bank-conflict
// free), and every reduction is a fixed-order warp shuffle — restating
// cones/psdcone.py:21-133 and the PSD parts of cones/scaling.py (NT factor via
// Cholesky + one-sided Jacobi SVD of Lz' Ls, congruence H = Q (x)s Q, step to the
// boundary via the minimum eigenvalue of L^-1 dS L^-T, neighbourhood trace).
// svec = column-major lower triangle with sqrt(2) off the diagonal.
#pragma once
#include <cmath>

namespace cipm {

namespace pw {

constexpr double kR2 = 1.4142135623730951;

__device__ __forceinline__ int svec_index(int i, int j, int n) {   // i >= j
    return j * n - j * (j - 1) / 2 + (i - j);
}

__device__ __forceinline__ double wsum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// X = smat(v) (full symmetric)
__device__ __forceinline__ void smat(const double* v, int n, double* X, int ld) {
    const int i = threadIdx.x & 31;
    if (i < n)
        for (int j = 0; j < n; ++j) {
            const int a = i > j ? i : j, b = i > j ? j : i;
            const double e = v[svec_index(a, b, n)];
            X[i * ld + j] = a == b ? e : e / kR2;
        }
    __syncwarp();
}

// v = svec(X) (lower triangle of X)
__device__ __forceinline__ void svec(const double* X, int n, int ld, double* v) {
    const int i = threadIdx.x & 31;
    if (i < n)
        for (int j = 0; j <= i; ++j) v[svec_index(i, j, n)] = i == j ? X[i * ld + i] : kR2 * X[i * ld + j];
    __syncwarp();
}

// lower Cholesky in place (upper part zeroed); false if not positive definite
__device__ __forceinline__ bool chol(double* A, int n, int ld) {
    const int i = threadIdx.x & 31;
    bool ok = true;
    for (int j = 0; j < n; ++j) {
        const double d = A[j * ld + j];
        if (!(d > 0.0)) ok = false;
        const double l = sqrt(d);
        __syncwarp();
        if (i == j) A[j * ld + j] = l;
        if (i > j && i < n) A[i * ld + j] = A[i * ld + j] / l;
        __syncwarp();
        if (i > j && i < n) {
            const double lij = A[i * ld + j];
            for (int c = j + 1; c <= i; ++c) A[i * ld + c] -= lij * A[c * ld + j];
        }
        __syncwarp();
    }
    if (i < n)
        for (int c = i + 1; c < n; ++c) A[i * ld + c] = 0.0;
    __syncwarp();
    return __all_sync(0xffffffffu, ok);
}

// C = op(A) op(B): op 0 = A B, 1 = A' B, 2 = A B'
// (C must not alias A or B: lane i writes row i of C while the others read A, B)
__device__ __forceinline__ void mm(const double* A, const double* B, int n, int ld, double* C, int op) {
    const int i = threadIdx.x & 31;
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
__device__ __forceinline__ void tri_inv(const double* L, int n, int ld, double* Li) {
    const int j = threadIdx.x & 31;
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
__device__ __forceinline__ void jacobi_svd(double* U, int n, int ld, double* V, double* sig) {
    const int k = threadIdx.x & 31;
    if (k < n)
        for (int c = 0; c < n; ++c) V[k * ld + c] = k == c ? 1.0 : 0.0;
    __syncwarp();
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rot = false;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double up = k < n ? U[k * ld + p] : 0.0, uq = k < n ? U[k * ld + q] : 0.0;
                const double al = wsum(up * up), be = wsum(uq * uq), ga = wsum(up * uq);
                if (fabs(ga) <= 1e-15 * sqrt(al * be) || ga == 0.0) continue;
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
                __syncwarp();
            }
        if (!rot) break;
    }
    for (int c = 0; c < n; ++c) {
        const double u = k < n ? U[k * ld + c] : 0.0;
        const double s2 = wsum(u * u);
        if (k == 0) sig[c] = sqrt(s2);
    }
    __syncwarp();
}

// cyclic two-sided Jacobi eigenvalues of a symmetric matrix (A overwritten); min eigenvalue
__device__ __forceinline__ double sym_min_eig(double* A, int n, int ld) {
    const int k = threadIdx.x & 31;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        if (k < n)
            for (int j = 0; j < n; ++j) {
                const double a2 = A[k * ld + j] * A[k * ld + j];
                tot += a2;
                if (j != k) off += a2;
            }
        off = wsum(off);
        tot = wsum(tot);
        if (off <= 1e-32 * tot || off == 0.0) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A[p * ld + q];
                if (apq == 0.0) continue;
                const double app = A[p * ld + p], aqq = A[q * ld + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                __syncwarp();
                if (k < n) {                     // columns p, q
                    const double akp = A[k * ld + p], akq = A[k * ld + q];
                    A[k * ld + p] = c * akp - s * akq;
                    A[k * ld + q] = s * akp + c * akq;
                }
                __syncwarp();
                if (k < n) {                     // rows p, q
                    const double apk = A[p * ld + k], aqk = A[q * ld + k];
                    A[p * ld + k] = c * apk - s * aqk;
                    A[q * ld + k] = s * apk + c * aqk;
                }
                __syncwarp();
                if (k == 0) { A[p * ld + q] = 0.0; A[q * ld + p] = 0.0; }
                __syncwarp();
            }
    }
    double mn = k < n ? A[k * ld + k] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    return mn;
}

// NT factor (psdcone.py:98-117): R = Ls V diag(sig^-1/2), R^-1 = diag(sig^1/2) V' Ls^-1,
// lam = sig; uses 4 work matrices W0..W3 of the warp slice
__device__ __forceinline__ bool nt_factor(const double* s, const double* z, int n, int ld, double* W0, double* W1,
                                          double* W2, double* W3, double* R, double* Rinv, double* lam) {
    const int i = threadIdx.x & 31;
    smat(s, n, W0, ld);
    if (!chol(W0, n, ld)) return false;            // Ls
    smat(z, n, W1, ld);
    if (!chol(W1, n, ld)) return false;            // Lz
    mm(W1, W0, n, ld, W2, 1);                      // M = Lz' Ls
    jacobi_svd(W2, n, ld, W3, lam);                // V in W3, sig in lam
    bool ok = true;
    if (i == 0)
        for (int c = 0; c < n; ++c) ok = ok && lam[c] > 0.0;
    if (!__shfl_sync(0xffffffffu, ok, 0)) return false;
    mm(W0, W3, n, ld, R, 0);                       // Ls V
    if (i < n)
        for (int c = 0; c < n; ++c) R[i * ld + c] /= sqrt(lam[c]);
    __syncwarp();
    tri_inv(W0, n, ld, W1);                        // Ls^-1
    mm(W3, W1, n, ld, Rinv, 1);                    // V' Ls^-1
    if (i < n) {
        const double sq = sqrt(lam[i]);
        for (int c = 0; c < n; ++c) Rinv[i * ld + c] *= sq;
    }
    __syncwarp();
    return true;
}

}  // namespace pw
}  // namespace cipm
