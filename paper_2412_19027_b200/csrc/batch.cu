// Batched independent instances (C5b: 8 x 256 MPC QPs): one CTA runs one
// instance's whole homogeneous-embedding IPM (Algorithm 1, reference
// ipm.py:411-496) on the device — no host round trip per iteration.
//
// All instances share one sparsity pattern, so the pattern tables (P, A, A',
// the permuted KKT CSC, the elimination schedule) live once in global memory
// (L1/L2 resident, read by every CTA) and every per-instance vector lives in
// the CTA's shared memory (or in a per-instance global workspace when an
// instance is too large for 227 KB).
//
// Scope: zero + nonnegative cones (LP / QP), the MPC family of the paper's
// §4.6.  Arithmetic follows the reference step for step:
//   residuals / termination / infeasibility   ipm.py:233-280 (fused scaled-G form)
//   stall, best iterate, almost-optimal        ipm.py:429-457, :489-496
//   nonneg NT scaling                          cones/scaling.py:231-240
//   KKT values + ±δs, up-looking LDL' with the
//     dynamic-regularisation bump              kkt/system.py:246-263, kkt/ldl.py:37-88
//   iterative refinement                       kkt/system.py:279-314
//   directions (two-column, P-norm Δτ)         ipm.py:309-338
//   step length (τ/κ + ray) and neighbourhood  cones/steps.py:79-116, ipm.py:350-366
//   take_step + membership                     ipm.py:368-379
// The factorisation uses the reference's own minimum-degree order and the
// reference's up-looking visiting order (precomputed schedule), single thread,
// FMA contraction off (built with -fmad=false), so D and L round like the
// CPU solver's.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "batch.hpp"

namespace cipm {

namespace {

constexpr int BT = 256;            // threads per instance CTA
constexpr int NW = BT / 32;

enum BStatus {
    BS_OPTIMAL = 0, BS_PRIMAL_INF = 1, BS_DUAL_INF = 2, BS_ALMOST = 3, BS_MAXIT = 4,
    BS_INSUFFICIENT = 6, BS_NUMERICAL = 7
};

struct Red {
    double* buf;   // NW * 16 doubles in shared memory
};

// block-wide fixed-order reduction of K values (sum / max per op mask bit: 1 = max)
template <int K>
__device__ __forceinline__ void breduce(double (&v)[K], unsigned maxmask, double* sbuf) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double a = v[k];
        for (int o = 16; o > 0; o >>= 1) {
            const double b = __shfl_down_sync(0xffffffffu, a, o);
            a = ((maxmask >> k) & 1u) ? fmax(a, b) : a + b;
        }
        if (lane == 0) sbuf[warp * K + k] = a;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double a = sbuf[k];
        for (int w = 1; w < NW; ++w) a = ((maxmask >> k) & 1u) ? fmax(a, sbuf[w * K + k]) : a + sbuf[w * K + k];
        v[k] = a;
    }
    __syncthreads();
}

struct Inst {
    // shared-memory (or workspace) vectors
    double *x, *z, *s, *dx[2], *dz[2], *ds[2], *gx, *gz, *col2, *sol, *rb, *rx, *rr, *rbest, *t, *dsc, *h, *w, *lam,
        *V, *lx, *d, *y, *qs, *bs;
};

__device__ __forceinline__ double csr_dot(const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                                          int i) {
    double acc = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) acc += v[p] * x[ci[p]];
    return acc;
}

// A' row i: values live in V (A part) at at_src
__device__ __forceinline__ double csrt_dot(const int32_t* rp, const int32_t* ci, const int32_t* src,
                                           const double* va, const double* x, int i) {
    double acc = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) acc += va[src[p]] * x[ci[p]];
    return acc;
}

__device__ void carve(const BatchPattern& pt, double* base, Inst& I) {
    const int n = pt.n, m = pt.m, dim = n + m;
    double* p = base;
    auto take = [&](int cnt) { double* q = p; p += (cnt + 1) & ~1; return q; };
    I.x = take(n); I.z = take(m); I.s = take(m);
    for (int k = 0; k < 2; ++k) { I.dx[k] = take(n); I.dz[k] = take(m); I.ds[k] = take(m); }
    I.gx = take(n); I.gz = take(m);
    I.col2 = take(dim); I.sol = take(dim);
    I.rb = take(dim); I.rx = take(dim); I.rr = take(dim); I.rbest = take(dim); I.t = take(dim);
    I.dsc = take(m); I.h = take(m); I.w = take(m); I.lam = take(m);
    I.V = take(pt.nnz_p + pt.nnz_a);
    I.lx = take(pt.use_groups ? pt.panel_total + pt.inbox_total : pt.nnz_l); I.d = take(dim); I.y = take(dim);
    I.qs = take(n); I.bs = take(m);
}

// ------------------------- factorisation (thread 0) -------------------------
// reference kkt/ldl.py:37-88 restated over the precomputed up-looking schedule
__device__ int factor_seq(const BatchPattern& pt, Inst& I, double delta_s, double delta_d) {
    const int dim = pt.n + pt.m;
    double* y = I.y;
    double run_max = 0.0;
    int bumped = 0;
    for (int j = 0; j < dim; ++j) y[j] = 0.0;
    for (int j = 0; j < dim; ++j) {
        for (int p = pt.cp[j]; p < pt.cp[j + 1]; ++p) {
            const int i = pt.ci[p];
            const int src = pt.csrc[p];
            double v = 0.0;
            if (src >= 0) v = I.V[src];
            else if (src <= -2) v = -I.h[-src - 2];
            if (i == j) v = v + (pt.sign[j] > 0 ? delta_s : -delta_s);
            y[i] += v;
        }
        double dj = y[j];
        y[j] = 0.0;
        for (int u = pt.up_ptr[j]; u < pt.up_ptr[j + 1]; ++u) {
            const int i = pt.up_i[u];
            const int p2 = pt.up_p2[u];
            const double yi = y[i];
            y[i] = 0.0;
            for (int p = pt.lp[i]; p < p2; ++p) y[pt.li[p]] -= I.lx[p] * yi;
            const double l_ji = yi / I.d[i];
            dj -= l_ji * yi;
            I.lx[p2] = l_ji;
        }
        const double bound = delta_s + delta_d * run_max;
        if (fabs(dj) < bound) {
            dj = pt.sign[j] > 0 ? bound : -bound;
            ++bumped;
        }
        if (dj == 0.0) return -1;
        I.d[j] = dj;
        if (fabs(dj) > run_max) run_max = fabs(dj);
    }
    return bumped;
}

// x += solve(r): permute, L / D / L' sweeps (kkt/ldl.py:91-104), permute back (thread 0)
__device__ void ldl_solve_add(const BatchPattern& pt, Inst& I, const double* r, double* x) {
    const int dim = pt.n + pt.m;
    double* t = I.t;
    for (int k = 0; k < dim; ++k) t[k] = r[pt.perm[k]];
    for (int j = 0; j < dim; ++j) {
        const double xj = t[j];
        for (int p = pt.lp[j]; p < pt.lp[j + 1]; ++p) t[pt.li[p]] -= I.lx[p] * xj;
    }
    for (int j = 0; j < dim; ++j) t[j] /= I.d[j];
    for (int j = dim - 1; j >= 0; --j) {
        double acc = t[j];
        for (int p = pt.lp[j]; p < pt.lp[j + 1]; ++p) acc -= I.lx[p] * t[pt.li[p]];
        t[j] = acc;
    }
    for (int k = 0; k < dim; ++k) x[pt.perm[k]] += t[k];
}

// ------------------- CTA-parallel factorisation (use_groups) -------------------
// The same L D L' as kkt/ldl.py:37-88 (same elimination order: the groups are
// independent subtrees, so eliminating them first or interleaved gives the same
// factor up to rounding), computed by all threads of the instance's CTA:
//   1. base values of every group panel and of the dense root block scattered from
//      V / -h with the static regularisation on the diagonal (system.py:253);
//   2. one thread per group: dense right-looking LDL' of its panel (w <= 16),
//      its contribution block L_off D L_off' into private inbox slots;
//   3. root entries gather their inbox slots (fixed order, no atomics);
//   4. root: blocked right-looking LDL' with 32-column blocks — warp 0 factors the
//      diagonal block in registers (shuffles), one thread per row below solves
//      against it, the trailing update is parallel over entries;
//   5. every diagonal block is replaced by its unit-lower inverse (solve form:
//      the blocked triangular solves become GEMVs).
// Dynamic regularisation (ldl.py:79-87): groups use their own running max, the
// root starts from the max over all group pivots (delta_d * runmax is O(eps^2)).
constexpr int RB = 32;             // root block width

__device__ __forceinline__ double root_bump(double dd, double ds, double dd_coef, double runmax, int8_t sg,
                                            int& bumped) {
    const double bound = ds + dd_coef * runmax;
    if (fabs(dd) < bound) {
        ++bumped;
        return sg > 0 ? bound : -bound;
    }
    return dd;
}

__device__ int group_ldl(const BatchPattern& pt, double* P, int r, int w, const int32_t* cols, double* d,
                         double ds, double ddc, double& runmax) {
    int bumped = 0;
    for (int j = 0; j < w; ++j) {
        double dj = root_bump(P[j * r + j], ds, ddc, runmax, pt.sign[cols[j]], bumped);
        if (dj == 0.0) return -1;
        d[cols[j]] = dj;
        runmax = fmax(runmax, fabs(dj));
        const double inv = 1.0 / dj;
        for (int i = j + 1; i < r; ++i) {
            const double lij = P[j * r + i] * inv;          // a_ij unscaled -> l_ij
            const int cend = i < w - 1 ? i : w - 1;
            for (int c = j + 1; c <= cend; ++c) P[c * r + i] -= lij * P[j * r + c];
        }
        for (int i = j + 1; i < r; ++i) P[j * r + i] *= inv;
        P[j * r + j] = 1.0;
    }
    return bumped;
}

// all threads; returns (in *s_err) 1 on a zero pivot
__device__ void bfactor_cta(const BatchPattern& pt, Inst& I, double ds, double ddc, double* sblk, int* s_err,
                            double* sred) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = pt.W, s0 = pt.s;
    double* PS = I.lx;                       // group panels, then the root block (col-major W x W)
    double* R = PS + pt.root_off;
    double* inbox = PS + pt.panel_total;
    for (int k = tid; k < pt.panel_total; k += BT) PS[k] = 0.0;
    __syncthreads();
    for (int k = tid; k < pt.nbsc; k += BT) {
        const int src = pt.bsc_src[k];
        PS[pt.bsc_slot[k]] = src >= 0 ? I.V[src] : -I.h[-src - 2];
    }
    __syncthreads();
    for (int k = tid; k < pt.nbdg; k += BT) {
        const int slot = pt.bdg_slot[k];
        PS[slot] = PS[slot] + (pt.sign[pt.bdg_col[k]] > 0 ? ds : -ds);
    }
    __syncthreads();
    // 2. groups
    double gmax[1] = {0.0};
    for (int g = tid; g < pt.ngroups; g += BT) {
        const int32_t* gi = pt.g_info + 8 * g;
        const int w = gi[1], r = gi[2], o = r - w;
        double* P = PS + gi[3];
        double runmax = 0.0;
        if (group_ldl(pt, P, r, w, pt.g_cols + gi[0], I.d, ds, ddc, runmax) < 0) *s_err = 1;
        gmax[0] = fmax(gmax[0], runmax);
        double* ib = inbox + gi[4];
        int tb = 0;
        for (int b = 0; b < o; ++b) {
            for (int a = b; a < o; ++a) {
                double acc = 0.0;
                for (int k = 0; k < w; ++k) acc += P[k * r + w + a] * I.d[pt.g_cols[gi[0] + k]] * P[k * r + w + b];
                ib[tb + (a - b)] = acc;
            }
            tb += o - b;
        }
    }
    breduce<1>(gmax, 1u, sred);
    // 3. root assembly: R(e) -= sum of its inbox slots
    for (int k = tid; k < pt.nrg; k += BT) {
        double acc = 0.0;
        for (int p = pt.rg_ptr[k]; p < pt.rg_ptr[k + 1]; ++p) acc += inbox[pt.rg_idx[p]];
        R[pt.rg_tgt[k]] -= acc;
    }
    __syncthreads();
    // 4. root blocked LDL'
    double runmax = gmax[0];
    int bumped = 0;
    for (int k0 = 0; k0 < W; k0 += RB) {
        const int nbk = min(RB, W - k0), k1 = k0 + nbk;
        if (warp == 0) {
            double x[RB];
#pragma unroll
            for (int c = 0; c < RB; ++c) x[c] = (c < nbk && lane < nbk && c <= lane) ? R[(k0 + c) * W + k0 + lane] : 0.0;
            // column j is published through shared memory (one store, broadcast loads;
            // double-buffered in sblk, which the block's L11 overwrites afterwards)
            // instead of 32 shuffles on the pivot chain — the same values
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                if (j < nbk) {
                    double* col = sblk + (j & 1) * 32;
                    col[lane] = x[j];
                    __syncwarp();
                    double dj = col[j];
                    dj = root_bump(dj, ds, ddc, runmax, pt.sign[s0 + k0 + j], bumped);
                    if (dj == 0.0 && lane == 0) *s_err = 1;
                    runmax = fmax(runmax, fabs(dj));
                    const double inv = 1.0 / dj;
                    if (lane == 0) {
                        I.d[s0 + k0 + j] = dj;
                        sblk[RB * RB + j] = inv;
                    }
                    const double xj = x[j];
#pragma unroll
                    for (int c = j + 1; c < RB; ++c) {
                        const double acj = col[c] * inv;
                        if (lane >= c) x[c] -= xj * acj;
                    }
                    x[j] = lane > j ? xj * inv : (lane == j ? 1.0 : 0.0);
                }
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < RB; ++c) {
                if (c < nbk && lane < nbk && c <= lane) R[(k0 + c) * W + k0 + lane] = x[c];
                sblk[c * RB + lane] = (c < lane && lane < nbk) ? x[c] : 0.0;   // sblk[c][i] = l_ic
            }
        }
        __syncthreads();
        // rows below the diagonal block: x_i L11' = a_i (right-looking on the row)
        for (int i = k1 + tid; i < W; i += BT) {
            double x[RB];
#pragma unroll
            for (int c = 0; c < RB; ++c) x[c] = c < nbk ? R[(k0 + c) * W + i] : 0.0;
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                const double xj = x[j];
#pragma unroll
                for (int c = j + 1; c < RB; ++c) x[c] -= xj * sblk[j * RB + c];
                x[j] = xj * sblk[RB * RB + j];
            }
#pragma unroll
            for (int c = 0; c < RB; ++c)
                if (c < nbk) R[(k0 + c) * W + i] = x[c];
        }
        __syncthreads();
        // trailing update of the lower triangle
        // (d_k l_ck for the warp's column c formed once per column in the warp's slice of
        // sblk — free between the row solve and the next diagonal block — not per row i)
        for (int c = k1 + warp; c < W; c += NW) {
            double* dl = sblk + warp * RB;
            if (lane < nbk) dl[lane] = I.d[s0 + k0 + lane] * R[(k0 + lane) * W + c];
            __syncwarp();
            for (int i = c + lane; i < W; i += 32) {
                double acc = 0.0;
                for (int k = 0; k < nbk; ++k) acc += R[(k0 + k) * W + i] * dl[k];
                R[c * W + i] -= acc;
            }
            __syncwarp();
        }
        __syncthreads();
    }
    // 5. diagonal blocks -> unit-lower inverses (column-parallel substitution, lane j = column j)
    for (int kb = warp; kb * RB < W; kb += NW) {
        const int k0 = kb * RB, nbk = min(RB, W - k0);
        double v[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            double acc = 0.0;
            if (i < nbk)
#pragma unroll
                for (int k = 0; k < i; ++k) acc += R[(k0 + k) * W + k0 + i] * v[k];
            v[i] = (i < nbk && lane < nbk) ? (i == lane ? 1.0 : (i < lane ? 0.0 : -acc)) : 0.0;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < RB; ++i)
            if (lane < nbk && i < nbk) R[(k0 + lane) * W + k0 + i] = v[i];   // column lane, zeros above the diagonal
        __syncwarp();
    }
    __syncthreads();
    (void)bumped;
}

// x += solve(r) (permuted, groups + blocked root, kkt/ldl.py:91-104); all threads
__device__ void bsolve_cta(const BatchPattern& pt, Inst& I, const double* r, double* x, double* sblk) {
    const int tid = threadIdx.x;
    const int dim = pt.n + pt.m, W = pt.W, s0 = pt.s;
    double* t = I.t;
    double* PS = I.lx;
    const double* R = PS + pt.root_off;
    double* vin = PS + pt.panel_total;       // the factor inbox is free during solves
    for (int k = tid; k < dim; k += BT) t[k] = r[pt.perm[k]];
    __syncthreads();
    // groups, forward
    for (int g = tid; g < pt.ngroups; g += BT) {
        const int32_t* gi = pt.g_info + 8 * g;
        const int w = gi[1], rr = gi[2], o = rr - w;
        const double* P = PS + gi[3];
        const int32_t* cols = pt.g_cols + gi[0];
        double y[16];
        for (int c = 0; c < w; ++c) {
            double acc = t[cols[c]];
            for (int k = 0; k < c; ++k) acc -= P[k * rr + c] * y[k];
            y[c] = acc;
            t[cols[c]] = acc;
        }
        for (int a = 0; a < o; ++a) {
            double acc = 0.0;
            for (int k = 0; k < w; ++k) acc += P[k * rr + w + a] * y[k];
            vin[gi[5] + a] = acc;
        }
    }
    __syncthreads();
    for (int i = tid; i < W; i += BT) {
        double acc = 0.0;
        for (int p = pt.rv_ptr[i]; p < pt.rv_ptr[i + 1]; ++p) acc += vin[pt.rv_idx[p]];
        t[s0 + i] -= acc;
    }
    __syncthreads();
    // root, forward: y_b = inv(L_bb) (t_b - sum_{k<b} L_bk y_k).  The block GEMVs run
    // as NW (diagonal block) / RP (rows below) strided partial sums per row, combined
    // in a fixed order, instead of one 32-term chain per thread on 32-56 threads
    constexpr int RP = BT / 64;                                    // partials per row below
    static_assert(NW * RB <= RB * RB && RP * 64 <= RB * RB, "sblk holds the partials");
    const int prow = tid & (RB - 1), part = tid / RB;
    for (int k0 = 0; k0 < W; k0 += RB) {
        const int nbk = min(RB, W - k0), k1 = k0 + nbk;
        {
            double acc = 0.0;
            if (prow < nbk)
                for (int k = part; k <= prow; k += NW) acc += R[(k0 + k) * W + k0 + prow] * t[s0 + k0 + k];
            sblk[part * RB + prow] = acc;
        }
        __syncthreads();
        if (tid < nbk) {
            double acc = 0.0;
            for (int q = 0; q < NW; ++q) acc += sblk[q * RB + tid];
            t[s0 + k0 + tid] = acc;
        }
        __syncthreads();
        for (int i0 = k1; i0 < W; i0 += 64) {
            const int i = i0 + (tid & 63), q = tid >> 6;
            double acc = 0.0;
            if (i < W)
                for (int k = q; k < nbk; k += RP) acc += R[(k0 + k) * W + i] * t[s0 + k0 + k];
            sblk[q * 64 + (tid & 63)] = acc;
            __syncthreads();
            if (tid < 64 && i0 + tid < W) {
                double a2 = 0.0;
                for (int qq = 0; qq < RP; ++qq) a2 += sblk[qq * 64 + tid];
                t[s0 + i0 + tid] -= a2;
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < W; i += BT) t[s0 + i] /= I.d[s0 + i];
    __syncthreads();
    // root, backward: x_b = inv(L_bb)' (t_b - sum_{i>=k1} L_ib' x_i), last block first
    const int nb = (W + RB - 1) / RB;
    double* bvec = sblk + NW * RB;                     // the block's right-hand side
    for (int kb = nb - 1; kb >= 0; --kb) {
        const int k0 = kb * RB, nbk = min(RB, W - k0), k1 = k0 + nbk;
        {
            double acc = 0.0;
            if (prow < nbk) {
                const double* Ck = R + (k0 + prow) * W;
                for (int i = k1 + part; i < W; i += NW) acc += Ck[i] * t[s0 + i];
            }
            sblk[part * RB + prow] = acc;
        }
        __syncthreads();
        if (tid < nbk) {
            double acc = 0.0;
            for (int q = 0; q < NW; ++q) acc += sblk[q * RB + tid];
            bvec[tid] = t[s0 + k0 + tid] - acc;
        }
        __syncthreads();
        {
            double acc = 0.0;
            if (prow < nbk) {
                const double* Cj = R + (k0 + prow) * W + k0;   // column prow of the inverse block
                for (int i = prow + part; i < nbk; i += NW) acc += Cj[i] * bvec[i];
            }
            sblk[part * RB + prow] = acc;
        }
        __syncthreads();
        if (tid < nbk) {
            double acc = 0.0;
            for (int q = 0; q < NW; ++q) acc += sblk[q * RB + tid];
            t[s0 + k0 + tid] = acc;
        }
        __syncthreads();
    }
    // groups, backward: x_c = y_c / d_c - L_off' x_R - sum_{k>c} l_kc x_k
    for (int g = tid; g < pt.ngroups; g += BT) {
        const int32_t* gi = pt.g_info + 8 * g;
        const int w = gi[1], rr = gi[2], o = rr - w;
        const double* P = PS + gi[3];
        const int32_t* cols = pt.g_cols + gi[0];
        const int32_t* rows = pt.g_rows + gi[6];
        double xv[16];
        for (int c = w - 1; c >= 0; --c) {
            double acc = t[cols[c]] / I.d[cols[c]];
            for (int a = 0; a < o; ++a) acc -= P[c * rr + w + a] * t[s0 + rows[a]];
            for (int k = c + 1; k < w; ++k) acc -= P[c * rr + k] * xv[k];
            xv[c] = acc;
            t[cols[c]] = acc;
        }
    }
    __syncthreads();
    for (int k = tid; k < dim; k += BT) x[pt.perm[k]] += t[k];
    __syncthreads();
}

struct Ctl {
    double tau, kappa, mu, gtau, sigma;
    double dtau[2], dkappa[2];
    double alpha;
    int err;          // 0 ok, else numerical error
    int done;
    int steps;
};

// ---------------------------- the kernel -----------------------------------
__global__ void __launch_bounds__(BT) batch_ipm(BatchPattern pt, BatchData bd, int count) {
    extern __shared__ __align__(16) double bsm[];
    __shared__ double sred[NW * 16];
    __shared__ Ctl C;
    __shared__ double sblk[RB * RB + RB];   // root: L11 of the current block + 1/d (factor), block vector (solve)
    const int inst = blockIdx.x;
    if (inst >= count) return;
    const int tid = threadIdx.x;
    const int n = pt.n, m = pt.m, dim = n + m;
    const int z0 = pt.zero_dim, nnd = pt.nonneg_dim;
    Inst I;
    carve(pt, bd.use_smem ? bsm : bd.workspace + (int64_t)inst * bd.ws_stride, I);
    const double* gV = bd.V + (int64_t)inst * (pt.nnz_p + pt.nnz_a);
    const double* q_in = bd.q + (int64_t)inst * n;
    const double* b_in = bd.b + (int64_t)inst * m;
    double* dr = bd.dr + (int64_t)inst * m;
    double* dc = bd.dc + (int64_t)inst * n;
    double* bx = bd.best_x + (int64_t)inst * n;
    double* bz_ = bd.best_z + (int64_t)inst * m;
    double* bs = bd.best_s + (int64_t)inst * m;
    const double* Va = I.V + pt.nnz_p;
    double* Vw = I.V + pt.nnz_p;
    const double nu1 = (double)nnd + 1.0;
    const double eps_feas = bd.eps_feas, eps_inf = bd.eps_inf;
    double* q = I.qs;
    double* b = I.bs;
    double cobj, norm_q, norm_b;

    if (bd.device_setup) {
        // raw user-order data: cone reordering + Ruiz equilibration in the CTA
        // (problem.py:177-284, the reference's elementwise arithmetic, no FMA contraction)
        for (int k = tid; k < pt.nnz_p; k += BT) I.V[k] = gV[k];
        for (int k = tid; k < pt.nnz_a; k += BT) Vw[k] = gV[pt.nnz_p + pt.a_src[k]];
        for (int k = tid; k < n; k += BT) q[k] = q_in[k];
        for (int k = tid; k < m; k += BT) b[k] = b_in[pt.b_src[k]];
        double nq[2] = {0.0, 0.0};
        for (int k = tid; k < n; k += BT) nq[0] = fmax(nq[0], fabs(q_in[k]));
        for (int k = tid; k < m; k += BT) nq[1] = fmax(nq[1], fabs(b_in[k]));
        breduce<2>(nq, 3u, sred);
        norm_q = n ? nq[0] : 0.0;
        norm_b = m ? nq[1] : 0.0;
        double* cnorm = I.rb;            // scratch (the refinement vectors are free before the loop)
        double* rnorm = I.rb + n;
        double* cstep = I.rx;
        double* rstep = I.rx + n;
        double* dcol = I.rr;
        double* drow = I.rr + n;
        for (int k = tid; k < n; k += BT) dcol[k] = 1.0;
        for (int k = tid; k < m; k += BT) drow[k] = 1.0;
        __syncthreads();
        if (bd.equilibrate) {
            for (int it = 0; it < 10; ++it) {
                for (int j = tid; j < n; j += BT) {
                    double c = 0.0;
                    for (int p = pt.p_rp[j]; p < pt.p_rp[j + 1]; ++p) c = fmax(c, fabs(I.V[p]));
                    for (int p = pt.at_rp[j]; p < pt.at_rp[j + 1]; ++p) c = fmax(c, fabs(Vw[pt.at_src[p]]));
                    cnorm[j] = c;
                }
                for (int r = tid; r < m; r += BT) {
                    double c = 0.0;
                    for (int p = pt.a_rp[r]; p < pt.a_rp[r + 1]; ++p) c = fmax(c, fabs(Vw[p]));
                    rnorm[r] = c;
                }
                __syncthreads();
                for (int j = tid; j < n; j += BT) {
                    const double st = cnorm[j] > 0.0 ? 1.0 / sqrt(cnorm[j]) : 1.0;
                    const double nd = fmin(fmax(dcol[j] * st, 1e-4), 1e4);
                    cstep[j] = nd / dcol[j];
                    dcol[j] = nd;
                }
                for (int r = tid; r < m; r += BT) {
                    const double st = rnorm[r] > 0.0 ? 1.0 / sqrt(rnorm[r]) : 1.0;
                    const double nd = fmin(fmax(drow[r] * st, 1e-4), 1e4);
                    rstep[r] = nd / drow[r];
                    drow[r] = nd;
                }
                __syncthreads();
                for (int j = tid; j < n; j += BT) {
                    const double cj = cstep[j];
                    for (int p = pt.p_rp[j]; p < pt.p_rp[j + 1]; ++p) I.V[p] = (cj * I.V[p]) * cstep[pt.p_ci[p]];
                    q[j] *= cj;
                }
                for (int r = tid; r < m; r += BT) {
                    const double ri = rstep[r];
                    for (int p = pt.a_rp[r]; p < pt.a_rp[r + 1]; ++p) Vw[p] = (ri * Vw[p]) * cstep[pt.a_ci[p]];
                    b[r] *= ri;
                }
                __syncthreads();
            }
            double qm[1] = {0.0};
            for (int k = tid; k < n; k += BT) qm[0] = fmax(qm[0], fabs(q[k]));
            breduce<1>(qm, 1u, sred);
            const double qmax = n ? qm[0] : 0.0;
            cobj = qmax == 0.0 ? 1.0 : fmin(fmax(1.0 / qmax, 1e-4), 1e4);
            for (int k = tid; k < pt.nnz_p; k += BT) I.V[k] = I.V[k] * cobj;
            for (int k = tid; k < n; k += BT) q[k] = q[k] * cobj;
        } else {
            cobj = 1.0;
        }
        for (int k = tid; k < n; k += BT) dc[k] = dcol[k];
        for (int k = tid; k < m; k += BT) dr[k] = drow[k];
        if (tid == 0) bd.out_cobj[inst] = cobj;
    } else {
        for (int k = tid; k < pt.nnz_p + pt.nnz_a; k += BT) I.V[k] = gV[k];
        for (int k = tid; k < n; k += BT) q[k] = q_in[k];
        for (int k = tid; k < m; k += BT) b[k] = b_in[k];
        cobj = bd.c_obj[inst];
        norm_q = bd.norm_q[inst];
        norm_b = bd.norm_b[inst];
    }
    __syncthreads();
    // unit start (set.py:91-112): x = 0, zero block 0, nonneg 1
    for (int k = tid; k < n; k += BT) I.x[k] = 0.0;
    for (int k = tid; k < m; k += BT) {
        const double u = (k >= z0 && k < z0 + nnd) ? 1.0 : 0.0;
        I.s[k] = u;
        I.z[k] = u;
        I.h[k] = 0.0;
    }
    __syncthreads();
    {
        double v[1] = {0.0};
        for (int k = tid; k < m; k += BT) v[0] += I.s[k] * I.z[k];
        breduce<1>(v, 0u, sred);
        if (tid == 0) {
            C.tau = 1.0;
            C.kappa = 1.0;
            C.mu = (v[0] + 1.0) / nu1;
            C.err = 0;
            C.done = 0;
        }
    }
    __syncthreads();
    const double mu0 = C.mu;
    double best_score = INFINITY;
    double best_r[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // g_p g_d rp rd tau kappa mu valid r1 r2 r3
    double cur_r[4] = {0, 0, 0, 0};
    double st_mu = INFINITY, st_rp = INFINITY, st_rd = INFINITY;
    int stall = 0;
    int status = -1;
    int iterations = 0;

    for (int it = 0; it <= bd.max_iter; ++it) {
        // ---- residuals through the scaled G rows (vec.cu resid_n / resid_m) ----
        const double tau = C.tau, kappa = C.kappa, mu = C.mu;
        double vn[6] = {0, 0, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int i = tid; i < n; i += BT) {
            const double px = csr_dot(pt.p_rp, pt.p_ci, I.V, I.x, i);
            const double atz = csrt_dot(pt.at_rp, pt.at_ci, pt.at_src, Va, I.z, i);
            const double g = -((px + atz) + q[i] * tau);
            I.gx[i] = g;
            const double xi = I.x[i], dci = dc[i];
            vn[0] += xi * px;
            vn[1] += q[i] * xi;
            vn[2] = fmax(vn[2], fabs(g / dci));
            vn[3] = fmax(vn[3], fabs(atz / dci));
            vn[4] = fmax(vn[4], fabs(px / dci));
            vn[5] = fmax(vn[5], fabs(dci * xi));
        }
        breduce<6>(vn, 0x3cu, sred);
        double vm[5] = {0, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int i = tid; i < m; i += BT) {
            const double ax = csr_dot(pt.a_rp, pt.a_ci, Va, I.x, i);
            const double si = I.s[i], dri = dr[i];
            const double g = (si + ax) - b[i] * tau;
            I.gz[i] = g;
            vm[0] += b[i] * I.z[i];
            vm[1] = fmax(vm[1], fabs(g / dri));
            vm[2] = fmax(vm[2], fabs((ax + si) / dri));
            vm[3] = fmax(vm[3], fabs(dri * I.z[i]));
            vm[4] = fmax(vm[4], fabs(si / dri));
        }
        breduce<5>(vm, 0x1eu, sred);
        const double xpx = vn[0], qx = vn[1], bzv = vm[0];
        const double nrm_xu = n ? vn[5] : 0.0, nrm_zu = m ? vm[3] : 0.0, nrm_su = m ? vm[4] : 0.0;
        const double gtau = ((kappa + qx) + bzv) + xpx / tau;
        const double hq = 0.5 * xpx / (cobj * tau * tau);
        const double g_p = hq + qx / (cobj * tau), g_d = -hq - bzv / (cobj * tau);
        const double rp = (m ? vm[1] : 0.0) / tau, rd = (n ? vn[2] : 0.0) / (cobj * tau);
        const double xbar = nrm_xu / tau, sbar = nrm_su / tau, zbar = nrm_zu / (cobj * tau);
        const double gap = fabs(g_p - g_d);
        const double r1 = rp / fmax(1.0, norm_b + xbar + sbar);
        const double r2 = rd / fmax(1.0, norm_q + xbar + zbar);
        const double r3 = gap / fmax(1.0, fmin(fabs(g_p), fabs(g_d)));
        const double score = fmax(r1, fmax(r2, r3));
        cur_r[0] = g_p; cur_r[1] = g_d; cur_r[2] = rp; cur_r[3] = rd;
        if (score < best_score || best_r[7] == 0.0) {
            if (score < best_score) best_score = score;
            best_r[0] = g_p; best_r[1] = g_d; best_r[2] = rp; best_r[3] = rd;
            best_r[4] = tau; best_r[5] = kappa; best_r[6] = mu; best_r[7] = 1.0;
            best_r[8] = r1; best_r[9] = r2; best_r[10] = r3;
            for (int k = tid; k < n; k += BT) bx[k] = I.x[k];
            for (int k = tid; k < m; k += BT) { bz_[k] = I.z[k]; bs[k] = I.s[k]; }
        }
        if (r1 < eps_feas && r2 < eps_feas && r3 < eps_feas) { status = BS_OPTIMAL; break; }
        {   // Eq.(9) (ipm.py:263-280) on the unscaled, un-normalised iterate
            const double bz_u = bzv / cobj, qx_u = qx / cobj;
            const double nx = nrm_xu, nz = nrm_zu / cobj, ns = nrm_su;
            const double atz = n ? vn[3] / cobj : 0.0;
            if (atz < -eps_inf * fmax(1.0, nx + nz) * bz_u && bz_u < -eps_inf) { status = BS_PRIMAL_INF; break; }
            const double pxn = n ? vn[4] / cobj : 0.0;
            const double axs = m ? vm[2] : 0.0;
            if (pxn < -eps_inf * fmax(1.0, nx) * bz_u && axs < -eps_inf * fmax(1.0, nx + ns) * qx_u &&
                qx_u < -eps_inf) { status = BS_DUAL_INF; break; }
        }
        if (it >= bd.max_iter) { status = BS_MAXIT; break; }
        {
            const bool improved = mu < STALL_IMP * st_mu || rp < STALL_IMP * st_rp || rd < STALL_IMP * st_rd;
            st_mu = fmin(st_mu, mu);
            st_rp = fmin(st_rp, rp);
            st_rd = fmin(st_rd, rd);
            stall = improved ? 0 : stall + 1;
            if (stall >= 5) { status = BS_INSUFFICIENT; break; }
        }
        // ---- nonneg NT scaling (scaling.py:231-240) ----
        for (int k = tid; k < nnd; k += BT) {
            const double sk = I.s[z0 + k], zk = I.z[z0 + k];
            if (!(sk > 0.0) || !(zk > 0.0)) C.err = 1;
            I.h[z0 + k] = sk / zk;
            I.w[z0 + k] = sqrt(sk / zk);
            I.lam[z0 + k] = sqrt(sk * zk);
        }
        __syncthreads();
        if (C.err) { status = BS_NUMERICAL; break; }
        // ---- numeric factorisation ----
        if (pt.use_groups) {
            bfactor_cta(pt, I, bd.delta_s, bd.delta_d, sblk, &C.err, sred);
        } else if (tid == 0) {
            const int bumped = factor_seq(pt, I, bd.delta_s, bd.delta_d);
            if (bumped < 0) C.err = 1;
        }
        __syncthreads();
        if (C.err) { status = BS_NUMERICAL; break; }

        // refined solve of K x = rb into `out` (system.py:279-314); K x from P, A, H
        auto refined = [&](double* out) {
            double bn[1] = {-INFINITY};
            for (int k = tid; k < dim; k += BT) {
                bn[0] = fmax(bn[0], fabs(I.rb[k]));
                I.rx[k] = 0.0;
                I.rr[k] = I.rb[k];
                out[k] = 0.0;
            }
            breduce<1>(bn, 1u, sred);
            const double target = bd.refine_abs + bd.refine_rel * (dim ? bn[0] : 0.0);
            double best = INFINITY, prev = INFINITY;
            int ups = 0;
            for (int step = 1; step <= bd.refine_max; ++step) {
                if (pt.use_groups) bsolve_cta(pt, I, I.rr, I.rx, sblk);
                else if (tid == 0) ldl_solve_add(pt, I, I.rr, I.rx);
                __syncthreads();
                double rn[1] = {-INFINITY};
                for (int i = tid; i < n; i += BT) {
                    const double kx = csr_dot(pt.p_rp, pt.p_ci, I.V, I.rx, i) +
                                      csrt_dot(pt.at_rp, pt.at_ci, pt.at_src, Va, I.rx + n, i);
                    const double r = I.rb[i] - kx;
                    I.rr[i] = r;
                    rn[0] = fmax(rn[0], fabs(r));
                }
                for (int i = tid; i < m; i += BT) {
                    double r = I.rb[n + i] - csr_dot(pt.a_rp, pt.a_ci, Va, I.rx, i);
                    r = r + I.h[i] * I.rx[n + i];
                    I.rr[n + i] = r;
                    rn[0] = fmax(rn[0], fabs(r));
                }
                breduce<1>(rn, 1u, sred);
                const double r = dim ? rn[0] : 0.0;
                if (r < best) {
                    best = r;
                    for (int k = tid; k < dim; k += BT) out[k] = I.rx[k];
                }
                if (r <= target) {
                    for (int k = tid; k < dim; k += BT) out[k] = I.rx[k];
                    break;
                }
                if (r > prev) {
                    if (++ups >= 2) break;
                } else {
                    ups = 0;
                }
                prev = r;
                __syncthreads();
            }
            __syncthreads();
        };

        // col2 = K \ [-q; b]
        for (int k = tid; k < dim; k += BT) I.rb[k] = k < n ? -q[k] : b[k - n];
        __syncthreads();
        refined(I.col2);
        // τ-step denominator pieces (fixed per iteration)
        double dn[5] = {0, 0, 0, 0, 0};
        for (int i = tid; i < n; i += BT) {
            double pdiff = 0.0, pdx2 = 0.0;
            for (int p = pt.p_rp[i]; p < pt.p_rp[i + 1]; ++p) {
                const int jx = pt.p_ci[p];
                pdiff += I.V[p] * (I.col2[jx] - I.x[jx] / tau);
                pdx2 += I.V[p] * I.col2[jx];
            }
            dn[0] += (I.col2[i] - I.x[i] / tau) * pdiff;
            dn[1] += I.col2[i] * pdx2;
            dn[2] += q[i] * I.col2[i];
        }
        for (int i = tid; i < m; i += BT) dn[3] += b[i] * I.col2[n + i];
        breduce<5>(dn, 0u, sred);
        const double den = (((kappa / tau + dn[0]) - dn[1]) - dn[2]) - dn[3];
        if (fabs(den) < 1e-14 || !(den == den)) { status = BS_NUMERICAL; break; }

        // direction recovery (ipm.py:309-338); which 0 affine, 1 combined
        auto recover = [&](int which, double d_tau, double d_kappa, const double* d_s) {
            double dd[3] = {0, 0, 0};
            for (int i = tid; i < n; i += BT) {
                const double pd = csr_dot(pt.p_rp, pt.p_ci, I.V, I.sol, i);
                dd[0] += q[i] * I.sol[i];
                dd[1] += (I.x[i] / tau) * pd;
            }
            for (int i = tid; i < m; i += BT) dd[2] += b[i] * I.sol[n + i];
            breduce<3>(dd, 0u, sred);
            const double num = (((d_tau - d_kappa / tau) + dd[0]) + dd[2]) + 2.0 * dd[1];
            const double dt = num / den;
            const double dk = -(d_kappa + kappa * dt) / tau;
            for (int k = tid; k < n; k += BT) I.dx[which][k] = I.sol[k] + dt * I.col2[k];
            for (int k = tid; k < m; k += BT) {
                const double dzk = I.sol[n + k] + dt * I.col2[n + k];
                I.dz[which][k] = dzk;
                I.ds[which][k] = -d_s[k] - I.h[k] * dzk;     // Δs = -d_s - H Δz
            }
            if (tid == 0) { C.dtau[which] = dt; C.dkappa[which] = dk; }
            __syncthreads();
        };
        // step to the boundary (steps.py:79-116): τ/κ + nonneg ray
        auto step_length = [&](int which) -> double {
            const double dt = C.dtau[which], dk = C.dkappa[which];
            double a = 1.0;
            if (dt < 0.0) a = fmin(a, -tau / dt);
            if (dk < 0.0) a = fmin(a, -kappa / dk);
            double v[1] = {INFINITY};
            for (int k = tid; k < nnd; k += BT) {
                const double dzk = I.dz[which][z0 + k], dsk = I.ds[which][z0 + k];
                if (dzk < 0.0) v[0] = fmin(v[0], -I.z[z0 + k] / dzk);
                if (dsk < 0.0) v[0] = fmin(v[0], -I.s[z0 + k] / dsk);
            }
            // min-reduction (max of negatives)
            v[0] = -v[0];
            breduce<1>(v, 1u, sred);
            return fmin(a, -v[0]);
        };

        // ---- affine direction ----
        for (int k = tid; k < dim; k += BT) I.rb[k] = k < n ? I.gx[k] : -(I.gz[k - n] - I.s[k - n]);
        __syncthreads();
        refined(I.sol);
        recover(0, gtau, kappa * tau, I.s);
        const double alpha_a = step_length(0);
        if (alpha_a < 1e-11) { status = BS_NUMERICAL; break; }
        const double sigma = pow(1.0 - alpha_a, 3.0);
        const double f = 1.0 - sigma;
        // ---- combined d_s (scaling.py:277-320, nonneg part) ----
        for (int k = tid; k < m; k += BT) {
            double o = 0.0;
            if (k >= z0 && k < z0 + nnd) {
                const double lam2 = I.s[k] * I.z[k];
                const double eta = I.ds[0][k] * I.dz[0][k];
                o = I.w[k] * ((lam2 + eta) - sigma * mu) / I.lam[k];
            }
            I.dsc[k] = o;
        }
        __syncthreads();
        const double dkap_c = (kappa * tau + C.dkappa[0] * C.dtau[0]) - sigma * mu;
        for (int k = tid; k < dim; k += BT) I.rb[k] = k < n ? f * I.gx[k] : -(f * I.gz[k - n] - I.dsc[k - n]);
        __syncthreads();
        refined(I.sol);
        recover(1, f * gtau, dkap_c, I.dsc);
        double alpha = step_length(1);
        if (alpha < 1e-11) { status = BS_NUMERICAL; break; }
        // ---- neighbourhood backtracking (ipm.py:350-366, scaling.py:364-374) ----
        bool ok = false;
        for (int tries = 0; tries < 4096; ++tries) {
            const double a = bd.step_scale * alpha;
            double v[3] = {0.0, 0.0, 0.0};
            for (int k = tid; k < m; k += BT) {
                const double st = I.s[k] + a * I.ds[1][k], zt = I.z[k] + a * I.dz[1][k];
                const double pz = st * zt;
                v[0] += pz;
                if (k >= z0 && k < z0 + nnd) {
                    if (!(st > 0.0) || !(zt > 0.0)) v[2] = 1.0;
                    v[1] += 1.0 / pz;
                }
            }
            breduce<3>(v, 0u, sred);
            if (v[2] != 0.0) break;   // DomainError
            const double mu_t = (v[0] + (tau + a * C.dtau[1]) * (kappa + a * C.dkappa[1])) / nu1;
            if (!(nnd && (double)nnd / v[1] < bd.beta * mu_t)) { ok = true; break; }
            alpha *= bd.backtrack;
            if (alpha < 1e-11) break;
        }
        if (!ok) { status = BS_NUMERICAL; break; }
        // ---- take_step (ipm.py:368-379) ----
        const double a = bd.step_scale * alpha;
        for (int k = tid; k < n; k += BT) I.x[k] = I.x[k] + a * I.dx[1][k];
        double mv[2] = {0.0, 0.0};
        for (int k = tid; k < m; k += BT) {
            const double zk = I.z[k] + a * I.dz[1][k];
            const double sk = I.s[k] + a * I.ds[1][k];
            I.z[k] = zk;
            I.s[k] = sk;
            if (k < z0 && sk != 0.0) mv[1] = 1.0;
            if (k >= z0 && k < z0 + nnd && (!(sk > 0.0) || !(zk > 0.0))) mv[1] = 1.0;
            mv[0] += sk * zk;
        }
        breduce<2>(mv, 0u, sred);
        const double nt = tau + a * C.dtau[1], nk = kappa + a * C.dkappa[1];
        if (!(nt > 0.0) || !(nk > 0.0) || mv[1] != 0.0) { status = BS_NUMERICAL; break; }
        if (tid == 0) {
            C.tau = nt;
            C.kappa = nk;
            C.mu = (mv[0] + nt * nk) / nu1;
        }
        __syncthreads();
        iterations = it + 1;
    }
    __syncthreads();
    // ---- outputs: the host recovers (unscale, un-permute, certificates) ----
    const bool terminal = status == BS_OPTIMAL || status == BS_PRIMAL_INF || status == BS_DUAL_INF;
    int final_status = status;
    const double* px = I.x;
    const double* pz = I.z;
    const double* ps = I.s;
    double res[9];
    if (terminal) {
        res[0] = cur_r[0]; res[1] = cur_r[1]; res[2] = cur_r[2]; res[3] = cur_r[3];
        res[4] = C.tau; res[5] = C.kappa; res[6] = C.mu;
    } else {
        // best iterate; ALMOST_OPTIMAL if it meets 10ε (ipm.py:489-496)
        px = bx; pz = bz_; ps = bs;
        for (int k = 0; k < 7; ++k) res[k] = best_r[k];
        const double e10 = 10.0 * eps_feas;
        if (best_r[7] != 0.0 && best_r[8] < e10 && best_r[9] < e10 && best_r[10] < e10) final_status = BS_ALMOST;
    }
    res[7] = mu0;
    res[8] = (double)iterations;
    __syncthreads();
    double* ox = bd.out_x + (int64_t)inst * n;
    double* oz = bd.out_z + (int64_t)inst * m;
    double* os = bd.out_s + (int64_t)inst * m;
    if (bd.device_setup) {
        // recovery on the device (ipm.py:383-407): unscale x = Dc x, z = Dr z / c, s = s / Dr,
        // divide by tau unless an infeasibility certificate, back to the user's row order
        const bool cert = final_status == BS_PRIMAL_INF || final_status == BS_DUAL_INF;
        const double tau_f = res[4];
        for (int k = tid; k < n; k += BT) {
            const double v = dc[k] * px[k];
            ox[k] = cert ? v : v / tau_f;
        }
        for (int k = tid; k < m; k += BT) {
            const double zu = dr[k] * pz[k] / cobj, su = ps[k] / dr[k];
            const int u = pt.b_src[k];
            oz[u] = cert ? zu : zu / tau_f;
            os[u] = cert ? su : su / tau_f;
        }
    } else {
        for (int k = tid; k < n; k += BT) ox[k] = px[k];
        for (int k = tid; k < m; k += BT) { oz[k] = pz[k]; os[k] = ps[k]; }
    }
    if (tid == 0) {
        bd.out_status[inst] = final_status;
        for (int k = 0; k < 9; ++k) bd.out_res[(int64_t)inst * 9 + k] = res[k];
    }
}

}  // namespace

size_t batch_smem_doubles(const BatchPattern& pt) {
    const int64_t n = pt.n, m = pt.m, dim = n + m;
    auto r2 = [](int64_t c) { return (c + 1) & ~int64_t(1); };
    const int64_t nl = pt.use_groups ? (int64_t)pt.panel_total + pt.inbox_total : pt.nnz_l;
    return (size_t)(r2(n) * 5 + r2(m) * 13 + r2(dim) * 7 + r2(pt.nnz_p + pt.nnz_a) + r2(nl) + r2(dim) * 2);
}

int batch_launch(const BatchPattern& pt, const BatchData& bd, int count, cudaStream_t stream, int smem_bytes) {
    if (smem_bytes > 0) {
        CIPM_CUDA(cudaFuncSetAttribute(batch_ipm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
    }
    batch_ipm<<<count, BT, smem_bytes > 0 ? smem_bytes : 0, stream>>>(pt, bd, count);
    CIPM_CUDA(cudaGetLastError());
    return CIPM_OK;
}

}  // namespace cipm

// ===========================================================================
// host side: pattern analysis (once) + the C ABI (include/cipm.h cipm_batch_*)
// ===========================================================================
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "symbolic.hpp"

struct cipm_batch {
    cipm::BatchPattern pt;
    cipm::BatchData bd;
    int count = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool have_raw = false;        // raw V / q / b uploaded once (NULL keeps them)
    int smem_bytes = 0;
    std::vector<void*> allocs;
    std::vector<int32_t> h_perm;
    int64_t h2d = 0, d2h = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

template <typename T>
int bup(cipm_batch* h, const T** dst, const std::vector<T>& v) {
    void* p = nullptr;
    CIPM_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(v.size(), 1)));
    h->allocs.push_back(p);
    if (!v.empty()) {
        CIPM_CUDA(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, h->stream));
        CIPM_CUDA(cudaStreamSynchronize(h->stream));
    }
    *dst = (const T*)p;
    return CIPM_OK;
}

template <typename T>
int balloc(cipm_batch* h, T** dst, int64_t count) {
    void* p = nullptr;
    CIPM_CUDA(cudaMalloc(&p, sizeof(T) * std::max<int64_t>(count, 1)));
    h->allocs.push_back(p);
    *dst = (T*)p;
    return CIPM_OK;
}

}  // namespace

extern "C" {

int cipm_batch_create(const cipm_problem_desc* d, int count, const cipm_settings* st, double eps_feas,
                      double eps_inf, int max_iter, cipm_batch** out) {
    CIPM_NVTX("cipm_batch_create");
    using namespace cipm;
    if (!d || !st || !out || count <= 0) return CIPM_E_ARG;
    if (d->n_soc || d->n_exp || d->n_pow || d->n_psd) {
        fprintf(stderr, "[cipm] batched instances support zero + nonnegative cones only\n");
        return CIPM_E_ARG;
    }
    if (st->precision != CIPM_FULL) {
        fprintf(stderr, "[cipm] batched instances run the full-precision factorisation\n");
        return CIPM_E_ARG;
    }
    const int64_t n = d->n, m = d->m, dim = n + m;
    const int64_t nnzp = d->p_rowptr[n], nnza = d->a_rowptr[m];
    auto* h = new cipm_batch();
    h->count = count;
    h->device = st->device;
    CIPM_CUDA(cudaSetDevice(h->device));
    if (st->stream) {
        h->stream = (cudaStream_t)st->stream;
    } else {
        CIPM_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    // K upper pattern with value sources (kkt/system.py:87-148)
    std::vector<int64_t> key;
    std::vector<int32_t> ksrc;
    key.reserve(n + nnzp + nnza + m);
    std::vector<std::pair<int64_t, int32_t>> ent;
    for (int64_t i = 0; i < n; ++i) ent.emplace_back(i * dim + i, -1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = d->p_rowptr[i]; p < d->p_rowptr[i + 1]; ++p)
            if (d->p_colidx[p] >= i) ent.emplace_back(i * dim + d->p_colidx[p], (int32_t)p);
    for (int64_t r = 0; r < m; ++r)
        for (int64_t p = d->a_rowptr[r]; p < d->a_rowptr[r + 1]; ++p)
            ent.emplace_back(d->a_colidx[p] * dim + (n + r), (int32_t)(nnzp + p));
    for (int64_t i = 0; i < m; ++i) ent.emplace_back((n + i) * dim + (n + i), (int32_t)(-2 - i));
    std::stable_sort(ent.begin(), ent.end(), [](auto& a, auto& b) { return a.first < b.first; });
    // unique keys; a P diagonal entry overrides the structural x-diagonal slot
    std::vector<int64_t> kr, kc;
    std::vector<int32_t> src;
    for (size_t e = 0; e < ent.size(); ++e) {
        if (!key.empty() && key.back() == ent[e].first) {
            if (ent[e].second != -1) src.back() = ent[e].second;
            continue;
        }
        key.push_back(ent[e].first);
        src.push_back(ent[e].second);
    }
    std::vector<int64_t> krp(dim + 1, 0), kci(key.size());
    for (size_t e = 0; e < key.size(); ++e) {
        krp[key[e] / dim + 1]++;
        kci[e] = key[e] % dim;
    }
    for (int64_t i = 0; i < dim; ++i) krp[i + 1] += krp[i];
    // the reference's minimum-degree order of that pattern (ordering.py:15-53)
    std::vector<int32_t> perm(dim);
    {
        int rc = cipm_min_degree(dim, krp.data(), kci.data(), perm.data());
        if (rc) { delete h; return rc; }
    }
    std::vector<int32_t> iperm(dim);
    for (int64_t k = 0; k < dim; ++k) iperm[perm[k]] = (int32_t)k;
    // permuted upper CSC sorted by (column, row) (system.py:198-219)
    const int64_t nk = (int64_t)key.size();
    std::vector<int64_t> rr(nk), cc(nk), ord(nk);
    for (int64_t e = 0; e < nk; ++e) {
        const int64_t pi = iperm[key[e] / dim], pj = iperm[key[e] % dim];
        rr[e] = std::min(pi, pj);
        cc[e] = std::max(pi, pj);
    }
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return cc[a] != cc[b] ? cc[a] < cc[b] : rr[a] < rr[b]; });
    std::vector<int32_t> cp(dim + 1, 0), ci(nk), csrc(nk);
    for (int64_t t = 0; t < nk; ++t) {
        ci[t] = (int32_t)rr[ord[t]];
        csrc[t] = src[ord[t]];
        cp[cc[ord[t]] + 1]++;
    }
    for (int64_t j = 0; j < dim; ++j) cp[j + 1] += cp[j];
    std::vector<int8_t> sign(dim);
    for (int64_t k = 0; k < dim; ++k) sign[k] = perm[k] < n ? 1 : -1;
    // etree + column counts (ldl.py:20-34), then the up-looking visiting schedule (ldl.py:37-88)
    std::vector<int32_t> parent(dim, -1), flag(dim, -1), lnz(dim, 0);
    for (int64_t j = 0; j < dim; ++j) {
        flag[j] = (int32_t)j;
        for (int32_t p = cp[j]; p < cp[j + 1]; ++p)
            for (int32_t i = ci[p]; flag[i] != j; i = parent[i]) {
                if (parent[i] == -1) parent[i] = (int32_t)j;
                lnz[i]++;
                flag[i] = (int32_t)j;
            }
    }
    std::vector<int32_t> lp(dim + 1, 0);
    for (int64_t j = 0; j < dim; ++j) lp[j + 1] = lp[j] + lnz[j];
    const int64_t nnzl = lp[dim];
    std::vector<int32_t> li(nnzl), upp(dim + 1, 0), upi, up2, cnt(dim, 0), pattern(dim);
    upi.reserve(nnzl);
    up2.reserve(nnzl);
    std::fill(flag.begin(), flag.end(), -1);
    for (int64_t j = 0; j < dim; ++j) {
        int64_t top = dim;
        flag[j] = (int32_t)j;
        for (int32_t p = cp[j]; p < cp[j + 1]; ++p) {
            int32_t i = ci[p];
            int64_t len = 0;
            while (flag[i] != j) { pattern[len++] = i; flag[i] = (int32_t)j; i = parent[i]; }
            while (len > 0) pattern[--top] = pattern[--len];
        }
        for (int64_t t = top; t < dim; ++t) {
            const int32_t i = pattern[t];
            const int32_t p2 = lp[i] + cnt[i];
            upi.push_back(i);
            up2.push_back(p2);
            li[p2] = (int32_t)j;
            cnt[i]++;
        }
        upp[j + 1] = (int32_t)upi.size();
    }
    // ---- CTA-parallel factorisation plan (BatchPattern::use_groups) ----
    // Groups = maximal subtrees of the elimination tree with <= 16 columns and <= 48
    // panel rows (independent: no K or L entries between disjoint subtrees); every
    // other column joins the dense root block (<= 128 columns), the Schur complement
    // of the groups.  The elimination order becomes [groups..., root] (the same L D L'
    // up to rounding: each group is closed under descendants), so the root is the
    // contiguous range [s, dim) of the new order.
    std::vector<int32_t> g_info, g_cols, g_rows, bsc_slot, bsc_src, bdg_slot, bdg_col, rg_tgt, rg_ptr, rg_idx,
        rv_ptr, rv_idx, perm_g, sign_g_i;
    std::vector<int8_t> sign_g;
    int64_t plan_s = dim, plan_W = 0, plan_ng = 0, panel_total = 0, root_off = 0, inbox_total = 0;
    bool plan_ok = false;
    if (!getenv("CIPM_BATCH_SEQ") && dim > 0) {
        std::vector<std::vector<int32_t>> kids(dim);
        std::vector<int32_t> ssize(dim, 1);
        for (int64_t j = 0; j < dim; ++j)
            if (parent[j] >= 0) kids[parent[j]].push_back((int32_t)j);
        for (int64_t j = 0; j < dim; ++j)
            if (parent[j] >= 0) ssize[parent[j]] += ssize[j];     // children precede parents
        std::vector<int32_t> gid(dim, -1);
        std::vector<std::vector<int32_t>> gcols, groots_old;
        std::vector<int32_t> rootc;
        std::vector<int32_t> stack;
        for (int64_t j = dim - 1; j >= 0; --j)
            if (parent[j] < 0) stack.push_back((int32_t)j);
        while (!stack.empty()) {
            const int32_t j = stack.back();
            stack.pop_back();
            bool grp = false;
            if (ssize[j] <= 16) {
                std::vector<int32_t> cols, sub{j}, offr;
                while (!sub.empty()) {
                    const int32_t u = sub.back();
                    sub.pop_back();
                    cols.push_back(u);
                    for (int32_t k : kids[u]) sub.push_back(k);
                }
                std::sort(cols.begin(), cols.end());
                for (int32_t u : cols)
                    for (int32_t p = lp[u]; p < lp[u + 1]; ++p)
                        if (!std::binary_search(cols.begin(), cols.end(), li[p])) offr.push_back(li[p]);
                std::sort(offr.begin(), offr.end());
                offr.erase(std::unique(offr.begin(), offr.end()), offr.end());
                if (cols.size() + offr.size() <= 48) {
                    grp = true;
                    for (int32_t u : cols) gid[u] = (int32_t)gcols.size();
                    gcols.push_back(cols);
                    groots_old.push_back(offr);
                }
            }
            if (!grp) {
                rootc.push_back(j);
                for (int32_t k : kids[j]) stack.push_back(k);
            }
        }
        std::sort(rootc.begin(), rootc.end());
        const int64_t W = (int64_t)rootc.size(), ng = (int64_t)gcols.size();
        bool ok = W <= 128;
        for (int64_t g = 0; g < ng && ok; ++g)
            for (int32_t r : groots_old[g])
                if (gid[r] >= 0) ok = false;                      // off rows must be root columns
        if (ok) {
            // new elimination order: groups (ascending old index inside), then the root
            std::vector<int32_t> sigma, inv(dim);
            for (auto& cols : gcols)
                for (int32_t u : cols) sigma.push_back(u);
            const int64_t s0 = (int64_t)sigma.size();
            for (int32_t u : rootc) sigma.push_back(u);
            for (int64_t k = 0; k < dim; ++k) inv[sigma[k]] = (int32_t)k;
            perm_g.resize(dim);
            sign_g.resize(dim);
            for (int64_t k = 0; k < dim; ++k) { perm_g[k] = perm[sigma[k]]; sign_g[k] = sign[sigma[k]]; }
            std::vector<std::vector<int32_t>> groots(ng);     // root-local off rows, ascending
            for (int64_t g = 0; g < ng; ++g) {
                for (int32_t r : groots_old[g]) groots[g].push_back(inv[r] - (int32_t)s0);
                std::sort(groots[g].begin(), groots[g].end());
            }
            std::vector<int32_t> lrow(dim, -1);                // new index -> local row in its group panel
            int64_t off = 0, ib = 0, vb = 0;
            g_info.assign((size_t)ng * 8, 0);
            for (int64_t g = 0; g < ng; ++g) {
                const int64_t w = (int64_t)gcols[g].size(), o = (int64_t)groots[g].size(), r = w + o;
                int32_t* gi = &g_info[(size_t)g * 8];
                gi[0] = (int32_t)g_cols.size();
                gi[1] = (int32_t)w;
                gi[2] = (int32_t)r;
                gi[3] = (int32_t)off;
                gi[4] = (int32_t)ib;
                gi[5] = (int32_t)vb;
                gi[6] = (int32_t)g_rows.size();
                for (int64_t c = 0; c < w; ++c) {
                    const int32_t nc = inv[gcols[g][c]];
                    g_cols.push_back(nc);
                    lrow[nc] = (int32_t)c;
                }
                for (int32_t rr : groots[g]) g_rows.push_back(rr);
                off += r * w;
                ib += o * (o + 1) / 2;
                vb += o;
            }
            root_off = off;
            panel_total = off + W * W;
            inbox_total = std::max<int64_t>(ib, vb);
            // base scatter: K entry (old i <= old j) is the lower entry (max, min) of the new order
            for (int64_t j = 0; j < dim; ++j)
                for (int32_t p = cp[j]; p < cp[j + 1]; ++p) {
                    const int64_t a0 = inv[ci[p]], b0 = inv[j];
                    const int64_t row = std::max(a0, b0), col = std::min(a0, b0);
                    int64_t slot;
                    if (col >= s0) {
                        slot = root_off + (col - s0) * W + (row - s0);
                    } else {
                        const int64_t g = gid[sigma[col]];
                        const int32_t* gi = &g_info[(size_t)g * 8];
                        const int64_t r = gi[2], w = gi[1];
                        int64_t lr;
                        if (row < s0) lr = lrow[row];
                        else lr = w + (std::lower_bound(groots[g].begin(), groots[g].end(), (int32_t)(row - s0)) -
                                       groots[g].begin());
                        slot = gi[3] + (int64_t)lrow[col] * r + lr;
                    }
                    if (csrc[p] != -1) { bsc_slot.push_back((int32_t)slot); bsc_src.push_back(csrc[p]); }
                    if (a0 == b0) { bdg_slot.push_back((int32_t)slot); bdg_col.push_back((int32_t)col); }
                }
            // root gather of the contribution inboxes, and of the solve's vector inbox per root row
            std::vector<std::pair<int32_t, int32_t>> tg;
            std::vector<std::vector<int32_t>> vrows(W);
            for (int64_t g = 0; g < ng; ++g) {
                const int32_t* gi = &g_info[(size_t)g * 8];
                const int64_t o = (int64_t)groots[g].size();
                int64_t tb = 0;
                for (int64_t b = 0; b < o; ++b) {
                    for (int64_t a = b; a < o; ++a)
                        tg.emplace_back((int32_t)(groots[g][b] * W + groots[g][a]), (int32_t)(gi[4] + tb + (a - b)));
                    tb += o - b;
                }
                for (int64_t a = 0; a < o; ++a) vrows[groots[g][a]].push_back((int32_t)(gi[5] + a));
            }
            std::stable_sort(tg.begin(), tg.end(), [](auto& x, auto& y) { return x.first < y.first; });
            for (size_t e = 0; e < tg.size(); ++e) {
                if (e == 0 || tg[e].first != tg[e - 1].first) { rg_tgt.push_back(tg[e].first); rg_ptr.push_back((int32_t)e); }
                rg_idx.push_back(tg[e].second);
            }
            rg_ptr.push_back((int32_t)tg.size());
            rv_ptr.push_back(0);
            for (int64_t i = 0; i < W; ++i) {
                for (int32_t v : vrows[i]) rv_idx.push_back(v);
                rv_ptr.push_back((int32_t)rv_idx.size());
            }
            plan_s = s0;
            plan_W = W;
            plan_ng = ng;
            plan_ok = true;
        }
        if (getenv("CIPM_BATCH_DEBUG"))
            fprintf(stderr, "[cipm] batch plan: dim %lld root W %lld groups %lld ok %d\n", (long long)dim, (long long)W,
                    (long long)ng, (int)ok);
    }
    // CSR / transposed patterns (int32)
    std::vector<int32_t> prp(d->p_rowptr, d->p_rowptr + n + 1), pci(d->p_colidx, d->p_colidx + nnzp);
    std::vector<int32_t> arp(d->a_rowptr, d->a_rowptr + m + 1), aci(d->a_colidx, d->a_colidx + nnza);
    std::vector<int32_t> trp(n + 1, 0), tci(nnza), tsrc(nnza);
    for (int64_t p = 0; p < nnza; ++p) trp[aci[p] + 1]++;
    for (int64_t j = 0; j < n; ++j) trp[j + 1] += trp[j];
    {
        std::vector<int32_t> fill(trp.begin(), trp.end() - 1);
        for (int64_t r = 0; r < m; ++r)
            for (int32_t p = arp[r]; p < arp[r + 1]; ++p) {
                const int32_t t = fill[aci[p]]++;
                tci[t] = (int32_t)r;
                tsrc[t] = p;
            }
    }
    BatchPattern& pt = h->pt;
    pt.n = (int)n;
    pt.m = (int)m;
    pt.zero_dim = (int)d->zero_dim;
    pt.nonneg_dim = (int)d->nonneg_dim;
    pt.nnz_p = (int)nnzp;
    pt.nnz_a = (int)nnza;
    pt.nnz_l = (int)nnzl;
    int rc = 0;
#define BTRY(x)           \
    do {                  \
        rc = (x);         \
        if (rc) {         \
            cipm_batch_destroy(h); \
            return rc;    \
        }                 \
    } while (0)
    BTRY(bup(h, &pt.p_rp, prp));
    BTRY(bup(h, &pt.p_ci, pci));
    BTRY(bup(h, &pt.a_rp, arp));
    BTRY(bup(h, &pt.a_ci, aci));
    BTRY(bup(h, &pt.at_rp, trp));
    BTRY(bup(h, &pt.at_ci, tci));
    BTRY(bup(h, &pt.at_src, tsrc));
    BTRY(bup(h, &pt.cp, cp));
    BTRY(bup(h, &pt.ci, ci));
    BTRY(bup(h, &pt.csrc, csrc));
    BTRY(bup(h, &pt.sign, sign));
    BTRY(bup(h, &pt.perm, perm));
    BTRY(bup(h, &pt.lp, lp));
    BTRY(bup(h, &pt.li, li));
    BTRY(bup(h, &pt.up_ptr, upp));
    BTRY(bup(h, &pt.up_i, upi));
    BTRY(bup(h, &pt.up_p2, up2));
    h->h_perm = perm;
    if (plan_ok) {
        pt.s = (int)plan_s;
        pt.W = (int)plan_W;
        pt.ngroups = (int)plan_ng;
        pt.panel_total = (int)panel_total;
        pt.root_off = (int)root_off;
        pt.inbox_total = (int)inbox_total;
        pt.nbsc = (int)bsc_slot.size();
        pt.nbdg = (int)bdg_slot.size();
        pt.nrg = (int)rg_tgt.size();
        BTRY(bup(h, &pt.g_info, g_info));
        BTRY(bup(h, &pt.g_cols, g_cols));
        BTRY(bup(h, &pt.g_rows, g_rows));
        BTRY(bup(h, &pt.bsc_slot, bsc_slot));
        BTRY(bup(h, &pt.bsc_src, bsc_src));
        BTRY(bup(h, &pt.bdg_slot, bdg_slot));
        BTRY(bup(h, &pt.bdg_col, bdg_col));
        BTRY(bup(h, &pt.rg_tgt, rg_tgt));
        BTRY(bup(h, &pt.rg_ptr, rg_ptr));
        BTRY(bup(h, &pt.rg_idx, rg_idx));
        BTRY(bup(h, &pt.rv_ptr, rv_ptr));
        BTRY(bup(h, &pt.rv_idx, rv_idx));
        pt.use_groups = 1;
        if (batch_smem_doubles(pt) * sizeof(double) > 220 * 1024) {
            pt.use_groups = 0;                    // too large for one CTA: keep the sequential path
        } else {
            // the new elimination order: permutation and signs of the groups-then-root order
            BTRY(bup(h, &pt.perm, perm_g));
            BTRY(bup(h, &pt.sign, sign_g));
            h->h_perm = perm_g;
        }
    }
    // per-instance buffers
    BatchData& bd = h->bd;
    const int64_t nv = nnzp + nnza;
    double* tmp = nullptr;
    BTRY(balloc(h, &tmp, count * nv)); bd.V = tmp;
    BTRY(balloc(h, &tmp, count * n)); bd.q = tmp;
    BTRY(balloc(h, &tmp, count * m)); bd.b = tmp;
    BTRY(balloc(h, &bd.dr, count * m));
    BTRY(balloc(h, &bd.dc, count * n));
    BTRY(balloc(h, &tmp, count)); bd.c_obj = tmp;
    BTRY(balloc(h, &tmp, count)); bd.norm_q = tmp;
    BTRY(balloc(h, &tmp, count)); bd.norm_b = tmp;
    BTRY(balloc(h, &bd.out_cobj, count));
    BTRY(balloc(h, &bd.best_x, count * n));
    BTRY(balloc(h, &bd.best_z, count * m));
    BTRY(balloc(h, &bd.best_s, count * m));
    BTRY(balloc(h, &bd.out_x, count * n));
    BTRY(balloc(h, &bd.out_z, count * m));
    BTRY(balloc(h, &bd.out_s, count * m));
    BTRY(balloc(h, &bd.out_res, count * 9));
    BTRY(balloc(h, &bd.out_status, count));
    const size_t nd = batch_smem_doubles(pt);
    const size_t bytes = nd * sizeof(double);
    if (bytes <= 220 * 1024) {
        bd.use_smem = 1;
        h->smem_bytes = (int)bytes;
    } else {
        bd.use_smem = 0;
        bd.ws_stride = (int64_t)nd;
        BTRY(balloc(h, &bd.workspace, (int64_t)count * (int64_t)nd));
        h->smem_bytes = 0;
    }
    bd.eps_feas = eps_feas;
    bd.eps_inf = eps_inf;
    bd.max_iter = max_iter;
    bd.delta_s = st->delta_s;
    bd.delta_d = st->delta_d;
    bd.beta = st->beta;
    bd.backtrack = st->backtrack;
    bd.step_scale = st->step_scale;
    bd.refine_abs = st->refine_abs;
    bd.refine_rel = st->refine_rel;
    bd.refine_max = st->refine_max;
    CIPM_CUDA(cudaEventCreate(&h->ev0));
    CIPM_CUDA(cudaEventCreate(&h->ev1));
#undef BTRY
    *out = h;
    return CIPM_OK;
}

int cipm_batch_info(const cipm_batch* h, int64_t* info) {
    if (!h || !info) return CIPM_E_ARG;
    info[0] = h->count;
    info[1] = h->pt.n;
    info[2] = h->pt.m;
    info[3] = h->pt.nnz_l;
    info[4] = h->smem_bytes;
    info[5] = h->bd.use_smem;
    info[6] = h->pt.use_groups;
    info[7] = h->pt.W;
    info[8] = h->pt.ngroups;
    return CIPM_OK;
}

int cipm_batch_set_values(cipm_batch* h, const double* V, const double* q, const double* b, const double* dr,
                          const double* dc, const double* c_obj, const double* norm_q, const double* norm_b) {
    if (!h) return CIPM_E_ARG;
    const int64_t c = h->count, n = h->pt.n, m = h->pt.m, nv = (int64_t)h->pt.nnz_p + h->pt.nnz_a;
    CIPM_CUDA(cudaSetDevice(h->device));
    auto cp = [&](const double* dst, const double* src, int64_t cnt) -> int {
        CIPM_CUDA(cudaMemcpyAsync((void*)dst, src, sizeof(double) * cnt, cudaMemcpyHostToDevice, h->stream));
        h->h2d += (int64_t)sizeof(double) * cnt;
        return CIPM_OK;
    };
    int rc = cp(h->bd.V, V, c * nv);
    if (!rc) rc = cp(h->bd.q, q, c * n);
    if (!rc) rc = cp(h->bd.b, b, c * m);
    if (!rc) rc = cp(h->bd.dr, dr, c * m);
    if (!rc) rc = cp(h->bd.dc, dc, c * n);
    if (!rc) rc = cp(h->bd.c_obj, c_obj, c);
    if (!rc) rc = cp(h->bd.norm_q, norm_q, c);
    if (!rc) rc = cp(h->bd.norm_b, norm_b, c);
    h->bd.device_setup = 0;
    // bd.V / q / b now hold reordered, scaled values: a later raw update must
    // re-send every array (a NULL would reuse them as raw user-order data)
    h->have_raw = false;
    return rc;
}

int cipm_batch_set_reorder(cipm_batch* h, const int64_t* row_perm, const int64_t* a_src) {
    using namespace cipm;
    if (!h) return CIPM_E_ARG;
    const int64_t m = h->pt.m, nnza = h->pt.nnz_a;
    std::vector<int32_t> bs(row_perm, row_perm + m), as(a_src, a_src + nnza);
    int rc = bup(h, &h->pt.b_src, bs);
    if (!rc) rc = bup(h, &h->pt.a_src, as);
    return rc;
}

int cipm_batch_set_raw_values(cipm_batch* h, const double* V, const double* q, const double* b, int equilibrate) {
    CIPM_NVTX("cipm_batch_set_raw_values");
    if (!h || !h->pt.b_src) return CIPM_E_ARG;
    const int64_t c = h->count, n = h->pt.n, m = h->pt.m, nv = (int64_t)h->pt.nnz_p + h->pt.nnz_a;
    CIPM_CUDA(cudaSetDevice(h->device));
    // NULL keeps the previous raw array (the kernel reads them, never writes them):
    // a parametric update of q / b sends only q / b
    if ((!V && nv && !h->have_raw) || (!q && n && !h->have_raw) || (!b && m && !h->have_raw)) return CIPM_E_ARG;
    if (V && nv) {
        CIPM_CUDA(cudaMemcpyAsync((void*)h->bd.V, V, sizeof(double) * c * nv, cudaMemcpyHostToDevice, h->stream));
        h->h2d += (int64_t)sizeof(double) * c * nv;
    }
    if (q && n) {
        CIPM_CUDA(cudaMemcpyAsync((void*)h->bd.q, q, sizeof(double) * c * n, cudaMemcpyHostToDevice, h->stream));
        h->h2d += (int64_t)sizeof(double) * c * n;
    }
    if (b && m) {
        CIPM_CUDA(cudaMemcpyAsync((void*)h->bd.b, b, sizeof(double) * c * m, cudaMemcpyHostToDevice, h->stream));
        h->h2d += (int64_t)sizeof(double) * c * m;
    }
    h->have_raw = true;
    h->bd.device_setup = 1;
    h->bd.equilibrate = equilibrate ? 1 : 0;
    return CIPM_OK;
}

int cipm_batch_solve(cipm_batch* h, double* ms) {
    CIPM_NVTX("cipm_batch_solve");
    if (!h) return CIPM_E_ARG;
    CIPM_CUDA(cudaSetDevice(h->device));
    CIPM_CUDA(cudaEventRecord(h->ev0, h->stream));
    int rc = cipm::batch_launch(h->pt, h->bd, h->count, h->stream, h->smem_bytes);
    if (rc) return rc;
    CIPM_CUDA(cudaEventRecord(h->ev1, h->stream));
    CIPM_CUDA(cudaEventSynchronize(h->ev1));
    CIPM_CUDA(cudaGetLastError());
    if (ms) {
        float v = 0.f;
        CIPM_CUDA(cudaEventElapsedTime(&v, h->ev0, h->ev1));
        *ms = v;
    }
    return CIPM_OK;
}

int cipm_batch_results(cipm_batch* h, int32_t* status, double* res, double* x, double* z, double* s) {
    CIPM_NVTX("cipm_batch_results");
    if (!h) return CIPM_E_ARG;
    const int64_t c = h->count, n = h->pt.n, m = h->pt.m;
    CIPM_CUDA(cudaSetDevice(h->device));
    CIPM_CUDA(cudaStreamSynchronize(h->stream));
    if (status) CIPM_CUDA(cudaMemcpyAsync(status, h->bd.out_status, sizeof(int32_t) * c, cudaMemcpyDeviceToHost, h->stream));
    if (res) CIPM_CUDA(cudaMemcpyAsync(res, h->bd.out_res, sizeof(double) * c * 9, cudaMemcpyDeviceToHost, h->stream));
    if (x) CIPM_CUDA(cudaMemcpyAsync(x, h->bd.out_x, sizeof(double) * c * n, cudaMemcpyDeviceToHost, h->stream));
    if (z) CIPM_CUDA(cudaMemcpyAsync(z, h->bd.out_z, sizeof(double) * c * m, cudaMemcpyDeviceToHost, h->stream));
    if (s) CIPM_CUDA(cudaMemcpyAsync(s, h->bd.out_s, sizeof(double) * c * m, cudaMemcpyDeviceToHost, h->stream));
    CIPM_CUDA(cudaStreamSynchronize(h->stream));     // results land in the caller's buffers before return
    h->d2h += (int64_t)(status ? 4 * c : 0) + (int64_t)sizeof(double) * ((res ? 9 * c : 0) + (x ? c * n : 0) +
                                                                         (z ? c * m : 0) + (s ? c * m : 0));
    return CIPM_OK;
}

int cipm_batch_io_bytes(cipm_batch* h, int64_t* h2d, int64_t* d2h, int reset) {
    if (!h) return CIPM_E_ARG;
    if (h2d) *h2d = h->h2d;
    if (d2h) *d2h = h->d2h;
    if (reset) h->h2d = h->d2h = 0;
    return CIPM_OK;
}

void cipm_batch_destroy(cipm_batch* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (void* p : h->allocs) cudaFree(p);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

}  // extern "C"
