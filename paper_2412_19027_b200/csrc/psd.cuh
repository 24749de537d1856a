// Small dense PSD-cone kernels (thread per cone, side <= MAXS), restating
// cones/psdcone.py:21-133 and the PSD parts of cones/scaling.py.
//
// Storage: svec = column-major lower triangle with √2 on off-diagonals
// (psdcone.py:21-46).  Matrices are local row-major arrays M[i*MAXS + j].
// The NT factor uses Cholesky factors of S and Z and a one-sided Jacobi SVD of
// Lz' Ls (the reference uses LAPACK gesdd; H = Q ⊗s Q with Q = R R' and the
// corrector are invariant to the order and signs of the singular pairs).
#pragma once
#include <cmath>

namespace cipm {

constexpr double kSqrt2 = 1.4142135623730951;

template <int MS>
__device__ inline void smat(const double* v, int n, double* X) {
    int k = 0;
    for (int j = 0; j < n; ++j) {
        X[j * MS + j] = v[k++];
        for (int i = j + 1; i < n; ++i) {
            double t = v[k++] / kSqrt2;
            X[i * MS + j] = t;
            X[j * MS + i] = t;
        }
    }
}

template <int MS>
__device__ inline void svec(const double* X, int n, double* v) {
    int k = 0;
    for (int j = 0; j < n; ++j) {
        v[k++] = X[j * MS + j];
        for (int i = j + 1; i < n; ++i) v[k++] = kSqrt2 * X[i * MS + j];
    }
}

// lower Cholesky (dpotrf semantics); false if not PD
template <int MS>
__device__ inline bool chol(const double* A, int n, double* L) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) L[i * MS + j] = 0.0;
    for (int j = 0; j < n; ++j) {
        double ajj = A[j * MS + j];
        for (int k = 0; k < j; ++k) ajj -= L[j * MS + k] * L[j * MS + k];
        if (!(ajj > 0.0)) return false;
        ajj = sqrt(ajj);
        L[j * MS + j] = ajj;
        for (int i = j + 1; i < n; ++i) {
            double v = A[i * MS + j];
            for (int k = 0; k < j; ++k) v -= L[i * MS + k] * L[j * MS + k];
            L[i * MS + j] = v / ajj;
        }
    }
    return true;
}

// inverse of a lower-triangular matrix
template <int MS>
__device__ inline void tri_inv(const double* L, int n, double* Li) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) Li[i * MS + j] = 0.0;
    for (int j = 0; j < n; ++j) {
        Li[j * MS + j] = 1.0 / L[j * MS + j];
        for (int i = j + 1; i < n; ++i) {
            double v = 0.0;
            for (int k = j; k < i; ++k) v -= L[i * MS + k] * Li[k * MS + j];
            Li[i * MS + j] = v / L[i * MS + i];
        }
    }
}

// C = A * B (op: 0 = A B, 1 = A' B, 2 = A B')
template <int MS>
__device__ inline void mm(const double* A, const double* B, int n, double* C, int op) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) {
                double a = op == 1 ? A[k * MS + i] : A[i * MS + k];
                double b = op == 2 ? B[j * MS + k] : B[k * MS + j];
                acc += a * b;
            }
            C[i * MS + j] = acc;
        }
}

// cyclic Jacobi eigenvalues of a symmetric matrix (A overwritten); returns min
template <int MS>
__device__ inline double sym_min_eig(double* A, int n) {
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double a2 = A[i * MS + j] * A[i * MS + j];
                tot += a2;
                if (i != j) off += a2;
            }
        if (off <= 1e-32 * tot || off == 0.0) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double apq = A[p * MS + q];
                if (apq == 0.0) continue;
                double app = A[p * MS + p], aqq = A[q * MS + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < n; ++k) {
                    double akp = A[k * MS + p], akq = A[k * MS + q];
                    A[k * MS + p] = c * akp - s * akq;
                    A[k * MS + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    double apk = A[p * MS + k], aqk = A[q * MS + k];
                    A[p * MS + k] = c * apk - s * aqk;
                    A[q * MS + k] = s * apk + c * aqk;
                }
                A[p * MS + q] = 0.0;
                A[q * MS + p] = 0.0;
            }
    }
    double mn = A[0];
    for (int i = 1; i < n; ++i) mn = fmin(mn, A[i * MS + i]);
    return mn;
}

// one-sided Jacobi SVD: on exit U = M V has orthogonal columns, sig = column norms
template <int MS>
__device__ inline void jacobi_svd(double* U, int n, double* V, double* sig) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) V[i * MS + j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rot = false;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int k = 0; k < n; ++k) {
                    double up = U[k * MS + p], uq = U[k * MS + q];
                    al += up * up;
                    be += uq * uq;
                    ga += up * uq;
                }
                if (fabs(ga) <= 1e-15 * sqrt(al * be) || ga == 0.0) continue;
                rot = true;
                double zeta = (be - al) / (2.0 * ga);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int k = 0; k < n; ++k) {
                    double up = U[k * MS + p], uq = U[k * MS + q];
                    U[k * MS + p] = c * up - s * uq;
                    U[k * MS + q] = s * up + c * uq;
                    double vp = V[k * MS + p], vq = V[k * MS + q];
                    V[k * MS + p] = c * vp - s * vq;
                    V[k * MS + q] = s * vp + c * vq;
                }
            }
        if (!rot) break;
    }
    for (int j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc += U[k * MS + j] * U[k * MS + j];
        sig[j] = sqrt(acc);
    }
}

// NT factor (psdcone.py:98-117): R = Ls V diag(σ^-1/2), R^-1 = diag(σ^1/2) V' Ls^-1
template <int MS>
__device__ inline int psd_nt(const double* s, const double* z, int n, double* R, double* Rinv, double* lam) {
    double A[MS * MS], Ls[MS * MS], Lz[MS * MS], M[MS * MS], V[MS * MS];
    smat<MS>(s, n, A);
    if (!chol<MS>(A, n, Ls)) return CIPM_E_SCALING;
    smat<MS>(z, n, A);
    if (!chol<MS>(A, n, Lz)) return CIPM_E_SCALING;
    mm<MS>(Lz, Ls, n, M, 1);                 // Lz' Ls
    jacobi_svd<MS>(M, n, V, lam);
    for (int j = 0; j < n; ++j)
        if (!(lam[j] > 0.0)) return CIPM_E_SCALING;
    mm<MS>(Ls, V, n, R, 0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) R[i * MS + j] /= sqrt(lam[j]);
    tri_inv<MS>(Ls, n, A);                   // Ls^-1
    mm<MS>(V, A, n, Rinv, 1);                // V' Ls^-1
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) Rinv[i * MS + j] *= sqrt(lam[i]);
    return 0;
}

// sup{a >= 0: mat(v) + a mat(dv) PSD} (psdcone.py:120-133); returns <0 on DomainError
template <int MS>
__device__ inline double psd_step(const double* v, const double* dv, int n) {
    double X[MS * MS], L[MS * MS], Li[MS * MS], D[MS * MS], T[MS * MS];
    smat<MS>(v, n, X);
    if (!chol<MS>(X, n, L)) return -1.0;
    tri_inv<MS>(L, n, Li);
    smat<MS>(dv, n, D);
    mm<MS>(Li, D, n, T, 0);
    mm<MS>(T, Li, n, X, 2);                  // Li D Li'
    double lmin = sym_min_eig<MS>(X, n);
    return lmin >= 0.0 ? INFINITY : -1.0 / lmin;
}

// tr(S^-1 Z^-1) for the neighbourhood test; returns false if not PD
template <int MS>
__device__ inline bool psd_trace_inv(const double* s, const double* z, int n, double* tr) {
    double X[MS * MS], L[MS * MS], Li[MS * MS], Si[MS * MS], Zi[MS * MS];
    smat<MS>(s, n, X);
    if (!chol<MS>(X, n, L)) return false;
    tri_inv<MS>(L, n, Li);
    mm<MS>(Li, Li, n, Si, 1);                // L^-T L^-1 = S^-1
    smat<MS>(z, n, X);
    if (!chol<MS>(X, n, L)) return false;
    tri_inv<MS>(L, n, Li);
    mm<MS>(Li, Li, n, Zi, 1);
    double acc = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) acc += Si[i * MS + j] * Zi[j * MS + i];
    *tr = acc;
    return true;
}

template <int MS>
__device__ inline bool psd_is_pd(const double* v, int n) {
    double X[MS * MS], L[MS * MS];
    smat<MS>(v, n, X);
    return chol<MS>(X, n, L);
}

}  // namespace cipm
