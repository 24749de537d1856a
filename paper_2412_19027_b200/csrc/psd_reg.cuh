// PSD-cone kernels for small equal sides (N <= 8, the C5a shape): one THREAD per
// cone, every matrix in registers as a compile-time-indexed packed lower triangle
// (no shared memory, no warp barriers), the whole cone kernel unrolled for N.
// Same algorithms as psd_warp.cuh (psdcone.py:21-133): Cholesky, triangular
// inverse, congruences, two-sided Jacobi (round-robin order) for the minimum eigenvalue.
#pragma once
#include <cmath>

namespace cipm {
namespace pr {

constexpr double kR2 = 1.4142135623730951;

template <int N>
struct Tri {
    static constexpr int T = N * (N + 1) / 2;
};

// packed lower triangle, row-major: (i, j), i >= j
__host__ __device__ constexpr int P(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }
// svec position (column-major lower, problem.py): (i, j), i >= j
__host__ __device__ constexpr int SV(int i, int j, int n) { return j * n - j * (j - 1) / 2 + (i - j); }

// S = smat(v)
template <int N>
__device__ __forceinline__ void smat(const double* __restrict__ v, double (&S)[Tri<N>::T]) {
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = j; i < N; ++i) {
            const double e = v[SV(i, j, N)];
            S[P(i, j)] = i == j ? e : e / kR2;
        }
}

template <int N>
__device__ __forceinline__ void svec_store(const double (&S)[Tri<N>::T], double* __restrict__ v) {
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = j; i < N; ++i) v[SV(i, j, N)] = i == j ? S[P(i, i)] : kR2 * S[P(i, j)];
}

// A = L L' in place (lower); false when not positive definite
template <int N>
__device__ __forceinline__ bool chol(double (&A)[Tri<N>::T]) {
    bool ok = true;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double d = A[P(j, j)];
#pragma unroll
        for (int k = 0; k < j; ++k) d -= A[P(j, k)] * A[P(j, k)];
        ok = ok && d > 0.0;
        const double l = sqrt(ok ? d : 1.0);
        A[P(j, j)] = l;
#pragma unroll
        for (int i = j + 1; i < N; ++i) {
            double v = A[P(i, j)];
#pragma unroll
            for (int k = 0; k < j; ++k) v -= A[P(i, k)] * A[P(j, k)];
            A[P(i, j)] = v / l;
        }
    }
    return ok;
}

// Li = L^-1 (lower)
template <int N>
__device__ __forceinline__ void tri_inv(const double (&L)[Tri<N>::T], double (&Li)[Tri<N>::T]) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
        Li[P(j, j)] = 1.0 / L[P(j, j)];
#pragma unroll
        for (int i = j + 1; i < N; ++i) {
            double v = 0.0;
#pragma unroll
            for (int k = j; k < i; ++k) v -= L[P(i, k)] * Li[P(k, j)];
            Li[P(i, j)] = v / L[P(i, i)];
        }
    }
}

// M = Li D Li' (symmetric), Li lower, D symmetric
template <int N>
__device__ __forceinline__ void congr_lower(const double (&Li)[Tri<N>::T], const double (&D)[Tri<N>::T],
                                            double (&M)[Tri<N>::T]) {
    double T[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int l = 0; l < N; ++l) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k <= i; ++k) v += Li[P(i, k)] * D[P(k, l)];
            T[i][l] = v;
        }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = 0.0;
#pragma unroll
            for (int l = 0; l <= j; ++l) v += T[i][l] * Li[P(j, l)];
            M[P(i, j)] = v;
        }
}

// Y = Q X Q (all symmetric)
template <int N>
__device__ __forceinline__ void congr_sym(const double (&Q)[Tri<N>::T], const double (&X)[Tri<N>::T],
                                          double (&Y)[Tri<N>::T]) {
    double T[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int l = 0; l < N; ++l) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) v += Q[P(i, k)] * X[P(k, l)];
            T[i][l] = v;
        }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = 0.0;
#pragma unroll
            for (int l = 0; l < N; ++l) v += T[i][l] * Q[P(l, j)];
            Y[P(i, j)] = v;
        }
}

// round-robin partner of index k in round r of the M-player tournament (M even)
__host__ __device__ constexpr int rr_partner(int k, int r, int M) {
    return k == M - 1 ? (r * (M / 2)) % (M - 1)
                      : (((r - k) % (M - 1) + (M - 1)) % (M - 1) == k ? M - 1 : ((r - k) % (M - 1) + (M - 1)) % (M - 1));
}

// one two-sided Jacobi rotation of the (p, q) pair (the rotation of pw::sym_min_eig),
// zeroing a_pq; the parameters depend only on a_pp, a_qq, a_pq
template <int N>
__device__ __forceinline__ void jrot(double (&A)[Tri<N>::T], int p, int q) {
    const double apq = A[P(p, q)];
    if (apq == 0.0) return;
    const double app = A[P(p, p)], aqq = A[P(q, q)];
    const double theta = (aqq - app) / (2.0 * apq);
    const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
    const double c = 1.0 / sqrt(1.0 + t * t);
    const double s = t * c;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (k == p || k == q) continue;
        const double akp = A[P(k, p)], akq = A[P(k, q)];
        A[P(k, p)] = c * akp - s * akq;
        A[P(k, q)] = s * akp + c * akq;
    }
    A[P(p, p)] = c * c * app - 2.0 * s * c * apq + s * s * aqq;
    A[P(q, q)] = s * s * app + 2.0 * s * c * apq + c * c * aqq;
    A[P(p, q)] = 0.0;
}

// two-sided Jacobi on a packed symmetric matrix, sweeps in round-robin order: the
// N/2 rotations of a round act on disjoint pairs, so their angle computations
// (the sqrt / division chains) are independent and overlap; same stopping rule as
// pw::sym_min_eig.  Returns the minimum eigenvalue.
template <int N>
__device__ __forceinline__ double sym_min_eig(double (&A)[Tri<N>::T]) {
    constexpr int M = (N + 1) & ~1;
#pragma unroll 1
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double a2 = A[P(i, j)] * A[P(i, j)];
                tot += a2;
                if (i != j) off += a2;
            }
        if (off <= 1e-32 * tot || off == 0.0) break;
#pragma unroll
        for (int r = 0; r < M - 1; ++r)
#pragma unroll
            for (int k = 0; k < M; ++k) {
                const int q = rr_partner(k, r, M);
                if (k < q && q < N) jrot<N>(A, k, q);
            }
    }
    double m = A[P(0, 0)];
#pragma unroll
    for (int i = 1; i < N; ++i) m = fmin(m, A[P(i, i)]);
    return m;
}

// sup{alpha >= 0: mat(v) + alpha mat(dv) PSD} (psdcone.py:120-133); < 0 when mat(v) is not PD
template <int N>
__device__ __forceinline__ double step_bound(const double* __restrict__ v, const double* __restrict__ dv) {
    double L[Tri<N>::T], Li[Tri<N>::T], D[Tri<N>::T], M[Tri<N>::T];
    smat<N>(v, L);
    if (!chol<N>(L)) return -1.0;
    tri_inv<N>(L, Li);
    smat<N>(dv, D);
    congr_lower<N>(Li, D, M);
    const double lmin = sym_min_eig<N>(M);
    return lmin >= 0.0 ? INFINITY : -1.0 / lmin;
}

// S^-1 = L^-T L^-1 into packed symmetric form; false when not PD
template <int N>
__device__ __forceinline__ bool sym_inv(const double* __restrict__ v, double (&Si)[Tri<N>::T]) {
    double L[Tri<N>::T], Li[Tri<N>::T];
    smat<N>(v, L);
    const bool ok = chol<N>(L);
    tri_inv<N>(L, Li);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = i; k < N; ++k) s += Li[P(k, i)] * Li[P(k, j)];
            Si[P(i, j)] = s;
        }
    return ok;
}

}  // namespace pr
}  // namespace cipm
