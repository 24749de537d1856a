// Dense "tail" of the supernodal LDL' (replaces the wide-supernode share of
// kkt/ldl.py:37-104 / kkt/system.py:246-271).
//
// Supernodes that are wide (w >= 64) or have a large contribution block
// (o >= 512) — and all their ancestors — are too big for one CTA of the
// persistent kernel in ldl.cu (the C1 LP's 1787-column root, the C4 exp/pow
// 5143-column root).  They run here after the persistent phase, one supernode
// at a time in topological order, as a blocked right-looking dense LDL' over
// the panel (r rows x w columns, column-major, ld = r) in HBM:
//
//   tail_gather   inbox -> panel (warp per row, fixed-order segmented sums)
//   for each 64-column block kb:
//     tail_diag   64x64 diagonal block: unblocked LDL' with the reference's
//                 dynamic-regularisation rule (ldl.py:79-87), one CTA, and the
//                 explicit inverse of its unit-lower factor
//     tail_gemm   rows below: L21 = A21 L11^-T D^-1 as a GEMM with that inverse
//     tail_gemm   trailing panel columns -= L21 D L21'   (FP64: DMMA
//                 mma.sync.m8n8k4 tensor-core tiles; FP32: FFMA tiles)
//   tail_gemm     contribution block C = L_off D L_off' pushed to the ancestors'
//                 inboxes (same GEMM, scatter epilogue)
//
// Triangular solves of a tail supernode are single multi-CTA launches: one CTA
// per 64-row block, ordered by an atomic ticket and synchronised with
// per-block release/acquire flags (a wavefront over the diagonal blocks);
// the diagonal solves are GEMVs with the precomputed block inverses.
#include <cuda_runtime.h>

#include <cstdlib>

#include <type_traits>

#include "common.cuh"
#include "ctx.hpp"

namespace cipm {

namespace {

constexpr int TB = 64;   // tail block size (columns / rows)

__device__ __forceinline__ void wait_flag(const int* p) { wait_ge(p, 1); }

// ---------------------------------------------------------------------------
// inbox gather: warp per panel row; entries of a row are sorted by target
// (column-major panel offset), equal targets contiguous (one per source).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) tail_gather(T* __restrict__ L, int r, const int64_t* __restrict__ irow,
                                                   const int32_t* __restrict__ tgt, const T* __restrict__ inbox) {
    const int lane = threadIdx.x & 31;
    const int tr = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tr >= r) return;
    const int64_t lo = irow[tr], hi = irow[tr + 1];
    int carry_t = -1;
    T carry = (T)0;
    // next chunk's entries are requested before the current one is scanned
    int tg_n = lo + lane < hi ? tgt[lo + lane] : -(lane + 2);
    T v_n = lo + lane < hi ? __ldcg(inbox + lo + lane) : (T)0;
    for (int64_t base = lo; base < hi; base += 32) {
        const int64_t e = base + lane;
        const bool valid = e < hi;
        const int tg = tg_n;
        T v = v_n;
        {
            const int64_t en = e + 32;
            tg_n = en < hi ? tgt[en] : -(lane + 2);
            v_n = en < hi ? __ldcg(inbox + en) : (T)0;
        }
        const int t0 = __shfl_sync(0xffffffffu, tg, 0);
        if (carry_t >= 0 && t0 != carry_t) {
            if (lane == 0) L[carry_t] -= carry;
            carry_t = -1;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int tp = __shfl_up_sync(0xffffffffu, tg, off);
            const T vp = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off && tp == tg) v += vp;
        }
        const int tn = __shfl_down_sync(0xffffffffu, tg, 1);
        const bool is_end = lane == 31 || tn != tg;
        const bool more = base + 32 < hi;
        T tot = v;
        if (valid && is_end && tg == carry_t) tot += carry;
        if (valid && is_end && !(lane == 31 && more)) L[tg] -= tot;
        const int t31 = __shfl_sync(0xffffffffu, tg, 31);
        const T v31 = __shfl_sync(0xffffffffu, tot, 31);
        if (more) {
            carry_t = t31;
            carry = v31;
        }
    }
}

// ---------------------------------------------------------------------------
// diagonal block: LDL' of the nb x nb block at (kb, kb) with the reference's
// dynamic-regularisation rule (ldl.py:79-87), then the explicit inverse of its
// unit lower factor — row-major for the solves, column-major as the B operand
// of the TRSM-as-GEMM (L21 = A21 L11^-T D^-1).
//
// The block sits column-major in shared memory (ld 64, zero outside the lower
// nb x nb triangle).  Blocked by 16 columns: (a) warp 0 factors the 16 x 16
// diagonal sub-block with lane i holding row i in registers (shuffles, no
// barriers), publishing L11' and 1/d; (b) one thread per row below applies the
// same right-looking elimination in registers; (c) rank-16 update of the
// trailing sub-matrix.  The inverse: one thread per column j of L^-1 holds that
// column in registers and eliminates right-looking down the 64 rows (column k
// of L is a contiguous, broadcast shared-memory read).
// ---------------------------------------------------------------------------
// (a) of tail_diag: LDL' of the 16 x 16 diagonal sub-block at k0 by warp 0, lane i
// owning row k0 + i in registers; FULL: nbk == SB (compile-time loop bounds)
template <typename T, bool FULL>
__device__ __forceinline__ void diag_sub(T* Sk, int k0, int nbk_rt, const int8_t* sSg, T* sCol, double delta_s,
                                         double delta_d, double* s_runmax_p, T* sD, T* sInv, T* dvec, int c0,
                                         int kb, int* err, int32_t* bumps, T* sLt) {
    constexpr int SB = 16;
    const int nbk = FULL ? SB : nbk_rt;
    const int lane = threadIdx.x & 31;
    double& s_runmax = *s_runmax_p;
    double runmax = s_runmax;
    // regularisation constants pinned in registers (not re-read from the constant
    // bank inside the pivot chain)
    double ds_r = delta_s, dd_r = delta_d;
    asm volatile("" : "+d"(ds_r), "+d"(dd_r));
    T x[SB];
#pragma unroll
    for (int c = 0; c < SB; ++c) x[c] = (lane < nbk && c <= lane) ? Sk[c * TB + k0 + lane] : (T)0;
    // the pivot chain holds only the shuffle, the regularisation select, the
    // reciprocal and the update; signs come from one ballot, and each lane
    // keeps its own column's d / 1/d / bump flag for a single store afterwards
    const unsigned pos = __ballot_sync(0xffffffffu, lane < nbk && sSg[k0 + lane] > 0);
    T d_mine = (T)0, inv_mine = (T)0;
    bool bump_mine = false;
#pragma unroll
    for (int j = 0; j < SB; ++j) {
        if (j < nbk) {
            // column j of the sub-block through shared memory (one store + one
            // broadcast load per operand instead of 15 shuffles): 1.7x shorter
            // pivot chain (tools/micro/diag16.cu)
            T* col = sCol + (j & 1) * 32;
            col[lane] = x[j];
            __syncwarp();
            // the whole column in one burst of 16-byte broadcast loads, so the
            // operands of the update are in flight with the pivot's own load
            // (tools/micro/diag_bench.cu: pivot chains -5 % FP64, -11 % FP32)
            T cc[SB];
            load_col<T, SB>(cc, col);
            double dd = (double)cc[j];
            const double bound = ds_r + dd_r * runmax;
            const bool bump = fabs(dd) < bound;
            dd = bump ? (((pos >> j) & 1u) ? bound : -bound) : dd;
            const T dt = (T)dd;
            runmax = fmax(runmax, fabs(dd));
            const T inv = (T)1 / dt;
            if (lane == j) {
                d_mine = dt;
                inv_mine = inv;
                bump_mine = bump;
            }
            const T lj = x[j] * inv;
#pragma unroll
            for (int c = j + 1; c < SB; ++c) {
                const T acj = cc[c];
                if (lane >= c) x[c] -= lj * acj;
            }
            x[j] = lane > j ? lj : (lane == j ? (T)1 : x[j]);
        }
    }
    if (lane < SB) {
        sInv[lane] = lane < nbk ? inv_mine : (T)0;
        if (lane < nbk) {
            sD[k0 + lane] = d_mine;
            dvec[c0 + kb + k0 + lane] = d_mine;
            if (d_mine == (T)0) set_error(err, CIPM_E_FACTOR);
        }
    }
    const unsigned nb_bumps = __popc(__ballot_sync(0xffffffffu, bump_mine));
    if (lane == 0 && nb_bumps) atomicAdd(bumps, (int)nb_bumps);
    int row = k0 + lane;
    asm volatile("" : "+r"(row));
#pragma unroll
    for (int c = 0; c < SB; ++c) {
        if (lane < nbk && c <= lane) Sk[c * TB + row] = x[c];
        if (lane < SB) sLt[c * SB + lane] = (c < lane && lane < nbk) ? x[c] : (T)0;
    }
    __syncwarp();
    if (lane == 0) s_runmax = runmax;
}

#ifdef CIPM_DIAG_TS
__device__ long long g_diag_ts[64];
#define DIAG_TS(k) do { if (threadIdx.x == 0) g_diag_ts[k] = clock64(); } while (0)
#else
#define DIAG_TS(k) do { } while (0)
#endif
template <typename T>
__global__ void __launch_bounds__(256) tail_diag(T* __restrict__ L, int r, int kb, int nb, int c0,
                                                 T* __restrict__ dvec, const int8_t* __restrict__ sign,
                                                 double* maxd, int32_t* bumps, int* err, double delta_s,
                                                 double delta_d, T* __restrict__ inv_rm, T* __restrict__ inv_cm) {
    constexpr int SB = 16;
    extern __shared__ __align__(16) unsigned char dsm_raw[];
    T* S = reinterpret_cast<T*>(dsm_raw);          // S[j * TB + i]: column-major block
    T* DL = S + TB * TB;                           // (TB - SB) x SB: d_k l_ck of the trailing columns
    __shared__ T sD[TB];
    __shared__ T sInv[SB];
    __shared__ __align__(16) T sLt[SB * SB];
    __shared__ __align__(16) T sCol[64];
    __shared__ int8_t sSg[TB];
    __shared__ double s_runmax;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    DIAG_TS(0);
    T* B = L + (int64_t)kb * r + kb;
    {
        // all 16 loads of a thread in flight at once (blockDim = 256)
        T v[TB * TB / 256];
#pragma unroll
        for (int u = 0; u < TB * TB / 256; ++u) {
            const int idx = tid + 256 * u, i = idx & (TB - 1), j = idx >> 6;
            v[u] = (i < nb && j < nb && i >= j) ? B[(int64_t)j * r + i] : (T)0;
        }
#pragma unroll
        for (int u = 0; u < TB * TB / 256; ++u) S[tid + 256 * u] = v[u];
    }
    if (tid < nb) sSg[tid] = sign[c0 + kb + tid];
    if (tid == 0) s_runmax = *maxd;
    __syncthreads();
    DIAG_TS(1);
    for (int k0 = 0; k0 < nb; k0 += SB) {
        const int nbk = min(SB, nb - k0);
        T* Sk = S + k0 * TB;                       // column k0
        // (a) diagonal sub-block, lane i owns row k0 + i
        if (wid == 0) {
            if (nbk == SB) diag_sub<T, true>(Sk, k0, nbk, sSg, sCol, delta_s, delta_d, &s_runmax, sD, sInv, dvec, c0, kb, err, bumps, sLt);
            else diag_sub<T, false>(Sk, k0, nbk, sSg, sCol, delta_s, delta_d, &s_runmax, sD, sInv, dvec, c0, kb, err, bumps, sLt);
        }
        __syncthreads();
        DIAG_TS(2 + 4 * (k0 / SB));
        const int c1 = k0 + nbk, rest = nb - c1;
        if (rest <= 0) break;
        // (b) rows below the sub-block
        for (int i = c1 + tid; i < nb; i += nt) {
            T x[SB];
#pragma unroll
            for (int c = 0; c < SB; ++c) x[c] = Sk[c * TB + i];
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                const T xj = x[j];
#pragma unroll
                for (int c = j + 1; c < SB; ++c) x[c] -= xj * sLt[j * SB + c];
                x[j] = xj * sInv[j];
            }
            int is = i;
            asm volatile("" : "+r"(is));
#pragma unroll
            for (int c = 0; c < SB; ++c) Sk[c * TB + is] = x[c];
        }
        // d_k l_ck of the trailing columns (reads the rows just finished: own thread only)
        __syncthreads();
        DIAG_TS(3 + 4 * (k0 / SB));
        for (int idx = tid; idx < rest * SB; idx += nt) {
            const int cc = idx / SB, k = idx - cc * SB;
            DL[idx] = sD[k0 + k] * Sk[k * TB + c1 + cc];
        }
        __syncthreads();
        // (c) trailing columns c >= c1, rows i >= c: A(i,c) -= sum_k l_ik d_k l_ck
        for (int c = c1 + wid; c < nb; c += nw) {
            const T* dl = DL + (c - c1) * SB;
            for (int i = c + lane; i < nb; i += 32) {
                T a0 = (T)0, a1 = (T)0, a2 = (T)0, a3 = (T)0;   // 4 independent chains
#pragma unroll
                for (int k = 0; k < SB; k += 4) {
                    a0 += Sk[k * TB + i] * dl[k];
                    a1 += Sk[(k + 1) * TB + i] * dl[k + 1];
                    a2 += Sk[(k + 2) * TB + i] * dl[k + 2];
                    a3 += Sk[(k + 3) * TB + i] * dl[k + 3];
                }
                S[c * TB + i] -= (a0 + a1) + (a2 + a3);
            }
        }
        __syncthreads();
        DIAG_TS(4 + 4 * (k0 / SB));
    }
    DIAG_TS(18);
    for (int idx = tid; idx < nb * nb; idx += nt) {
        const int i = idx % nb, j = idx / nb;
        if (i >= j) B[(int64_t)j * r + i] = S[j * TB + i];
    }
    if (tid == 0) *maxd = s_runmax;
    // inverse of the unit lower block by 16 x 16 blocks: X_ii = L_ii^-1 (thread per
    // column, registers), then block rows bi = 1..3: X_ij = -X_ii sum_{k=j}^{bi-1} L_ik X_kj.
    // Compact loops: this kernel runs once per diagonal block, from a cold i-cache.
    constexpr int XL = TB + 1;
    T* X = DL + (TB - SB) * SB;                    // X[col * XL + row]
    T* Tm = X + TB * XL;                           // 3 x 16 x 16 scratch
    if (tid < TB) {
        const int base = tid & ~(SB - 1), jj = tid & (SB - 1);
        T x[SB];
#pragma unroll
        for (int rr = 0; rr < SB; ++rr) x[rr] = rr == jj ? (T)1 : (T)0;
#pragma unroll
        for (int k = 0; k < SB - 1; ++k) {
            const T xk = x[k];
#pragma unroll
            for (int rr = k + 1; rr < SB; ++rr) x[rr] -= S[(base + k) * TB + base + rr] * xk;
        }
#pragma unroll
        for (int rr = 0; rr < SB; ++rr) X[(base + jj) * XL + base + rr] = x[rr];
    }
    __syncthreads();
    for (int bi = 1; bi < TB / SB; ++bi) {
        for (int e = tid; e < bi * SB * SB; e += nt) {
            const int bj = e >> 8, rr = e & (SB - 1), cc = (e >> 4) & (SB - 1);
            T a0 = (T)0, a1 = (T)0, a2 = (T)0, a3 = (T)0;
            for (int k = bj * SB; k < bi * SB; k += 4) {     // (bi - bj) * 16 terms, 4 chains
                a0 += S[k * TB + bi * SB + rr] * X[(bj * SB + cc) * XL + k];
                a1 += S[(k + 1) * TB + bi * SB + rr] * X[(bj * SB + cc) * XL + k + 1];
                a2 += S[(k + 2) * TB + bi * SB + rr] * X[(bj * SB + cc) * XL + k + 2];
                a3 += S[(k + 3) * TB + bi * SB + rr] * X[(bj * SB + cc) * XL + k + 3];
            }
            Tm[e] = (a0 + a1) + (a2 + a3);          // Tm[bj](rr, cc)
        }
        __syncthreads();
        for (int e = tid; e < bi * SB * SB; e += nt) {
            const int bj = e >> 8, rr = e & (SB - 1), cc = (e >> 4) & (SB - 1);
            const T* Tb = Tm + bj * SB * SB + cc * SB;
            T a0 = (T)0, a1 = (T)0, a2 = (T)0, a3 = (T)0;
#pragma unroll
            for (int m = 0; m < SB; m += 4) {
                a0 += X[(bi * SB + m) * XL + bi * SB + rr] * Tb[m];
                a1 += X[(bi * SB + m + 1) * XL + bi * SB + rr] * Tb[m + 1];
                a2 += X[(bi * SB + m + 2) * XL + bi * SB + rr] * Tb[m + 2];
                a3 += X[(bi * SB + m + 3) * XL + bi * SB + rr] * Tb[m + 3];
            }
            X[(bj * SB + cc) * XL + bi * SB + rr] = -((a0 + a1) + (a2 + a3));
        }
        __syncthreads();
    }
    DIAG_TS(19);
    for (int idx = tid; idx < TB * TB; idx += nt) {
        const int hi = idx >> 6, lo = idx & (TB - 1);
        // column-major copy: (row lo, column hi); row-major: (row hi, column lo)
        inv_cm[idx] = (lo < nb && (lo >> 4) >= (hi >> 4)) ? X[hi * XL + lo] : (T)0;
        inv_rm[idx] = (hi < nb && (hi >> 4) >= (lo >> 4)) ? X[lo * XL + hi] : (T)0;
    }
    DIAG_TS(20);
}

template <typename T>
constexpr int diag_smem() {
    return (int)sizeof(T) * (TB * TB + (TB - 16) * 16 + TB * (TB + 1) + 3 * 16 * 16);
}

// ---------------------------------------------------------------------------
// C (M x N, lower: i + diag_off >= j) op= A (M x K) * diag(d) * B (N x K)'
// A, B column-major with leading dimensions lda / ldb.  MODE 0: C -= acc in
// place (ld = ldc).  MODE 1: inbox[push_pos[i,j packed]] = acc.  MODE 2:
// C = acc / dscale[j] (the rows-below solve with a block inverse, in place).
// 64x64 CTA tile, 4 warps of 32x32, K staged in 16-deep slices through a
// 4-stage cp.async ring (all of a K = 64 update is in flight at once); the MODE 0
// tile of C is loaded (negated) into the accumulators before the K loop, so its
// read overlaps the operand loads.  FP64 uses DMMA m8n8k4; FP32 FFMA tiles.
// ---------------------------------------------------------------------------
constexpr int GB = 64, GK = 16, GP = GB + 4, GST = 4;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src, bool ok) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

template <typename T>
struct GemmSmem {
    T A[GST][GK][GP];
    T B[GST][GK][GP];
    T D[GST][GK];
};

template <typename T>
constexpr int gemm_smem() { return (int)sizeof(GemmSmem<T>); }

template <typename T, int MODE>
__global__ void __launch_bounds__(128) tail_gemm(const T* A, int lda, const T* __restrict__ Bm, int ldb,
                                                 const T* __restrict__ d, int M, int N, int K, int diag_off,
                                                 T* C, int ldc, const int64_t* __restrict__ push_pos,
                                                 T* __restrict__ inbox, const T* __restrict__ dscale) {
    const int m0 = blockIdx.x * GB, n0 = blockIdx.y * GB;
    if (m0 + GB - 1 + diag_off < n0) return;      // tile strictly above the diagonal
    extern __shared__ __align__(16) unsigned char gsm_raw[];
    GemmSmem<T>& sm = *reinterpret_cast<GemmSmem<T>*>(gsm_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int nk = (K + GK - 1) / GK;
    auto load_stage = [&](int kt) {
        const int slot = kt % GST, k0 = kt * GK;
#pragma unroll
        for (int u = 0; u < GK * GB / 128; ++u) {
            const int e = tid + 128 * u, k = e >> 6, mi = e & 63;
            const int gk = k0 + k;
            const bool kok = gk < K;
            const bool aok = kok && m0 + mi < M, bok = kok && n0 + mi < N;
            cp_async_elem(&sm.A[slot][k][mi], aok ? A + (int64_t)gk * lda + m0 + mi : A, aok);
            cp_async_elem(&sm.B[slot][k][mi], bok ? Bm + (int64_t)gk * ldb + n0 + mi : Bm, bok);
        }
        if (tid < GK) {
            const bool ok = d != nullptr && k0 + tid < K;
            cp_async_elem(&sm.D[slot][tid], ok ? d + k0 + tid : Bm, ok);
        }
    };
#pragma unroll
    for (int s = 0; s < GST - 1; ++s) {
        if (s < nk) load_stage(s);
        cp_async_commit();
    }
    T acc[4][4][2];                                 // FP64: DMMA accumulators; FP32: FFMA (true FP32, as the reference's factor)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = 0.0;
                if (MODE == 0) {
                    const int i = m0 + wm * 32 + a * 8 + (lane >> 2);
                    const int j = n0 + wn * 32 + b * 8 + (lane & 3) * 2 + e;
                    if (i < M && j < N && i + diag_off >= j) v = -(double)C[(int64_t)j * ldc + i];
                }
                acc[a][b][e] = v;
            }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<GST - 2>();
        __syncthreads();
        if (kt + GST - 1 < nk) load_stage(kt + GST - 1);
        cp_async_commit();
        const int slot = kt % GST;
        if constexpr (std::is_same<T, double>::value) {
#pragma unroll
            for (int kk = 0; kk < GK; kk += 4) {
                const int kr = kk + (lane & 3);
                const double dk = d ? sm.D[slot][kr] : 1.0;
                double af[4], bf[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) af[a] = sm.A[slot][kr][wm * 32 + a * 8 + (lane >> 2)];
#pragma unroll
                for (int b = 0; b < 4; ++b) bf[b] = sm.B[slot][kr][wn * 32 + b * 8 + (lane >> 2)] * dk;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
            }
        } else {
            // FP32 (mixed mode): same fragment ownership, FFMA accumulation
#pragma unroll 4
            for (int k = 0; k < GK; ++k) {
                const float dk = d ? sm.D[slot][k] : 1.0f;
                float af[4], bf[4][2];
#pragma unroll
                for (int a = 0; a < 4; ++a) af[a] = sm.A[slot][k][wm * 32 + a * 8 + (lane >> 2)];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    bf[b][0] = sm.B[slot][k][wn * 32 + b * 8 + (lane & 3) * 2] * dk;
                    bf[b][1] = sm.B[slot][k][wn * 32 + b * 8 + (lane & 3) * 2 + 1] * dk;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        acc[a][b][0] = fmaf(af[a], bf[b][0], acc[a][b][0]);
                        acc[a][b][1] = fmaf(af[a], bf[b][1], acc[a][b][1]);
                    }
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = m0 + wm * 32 + a * 8 + (lane >> 2);
                const int j = n0 + wn * 32 + b * 8 + (lane & 3) * 2 + e;
                if (i >= M || j >= N || i + diag_off < j) continue;
                if (MODE == 0) {
                    C[(int64_t)j * ldc + i] = (T)(-acc[a][b][e]);
                } else if (MODE == 2) {
                    C[(int64_t)j * ldc + i] = (T)acc[a][b][e] / dscale[j];
                } else {
                    const int64_t tpk = (int64_t)j * M - (int64_t)j * (j - 1) / 2 + (i - j);
                    inbox[push_pos[tpk]] = (T)acc[a][b][e];
                }
            }
}

__global__ void tail_finish(double* maxd, int32_t* count, int J, int parent) {
    if (parent >= 0) {
        const double v = maxd[J];
        atomicMax(reinterpret_cast<unsigned long long*>(maxd + parent), (unsigned long long)__double_as_longlong(v));
        atomicAdd(count + parent, 1);
    }
}

// ---------------------------------------------------------------------------
// triangular solves of one tail supernode
// ---------------------------------------------------------------------------
struct TailSolveArgs {
    int c0, w, r, nbd;
    int64_t dim, nv, cvo;
    const int32_t* rows;       // sn_rows + r0 (permuted row indices)
    const int64_t* vn_lo;      // non-tiny vector-inbox entries of each column (tiny ones are folded)
    const int64_t* vn_hi;
    const int32_t* vpush_pos;
    int* flags;                // nbd flags
    int* ticket;
    int* done;                 // backward: solve-done flag of the supernode (persistent-kernel protocol)
    int act0, act1;
    const double* rstate;      // refinement state: skip converged right-hand sides
};

// forward: CTA per row block (diag blocks 0..nbd-1, then off-row blocks).
// Everything static is fetched before the CTA waits: its inverse block into
// shared memory, and each block's L values into registers before that block's
// flag is polled, so the critical step after a flag is one load of the 64
// solved values, a GEMV from registers and (diag) a GEMV from shared memory.
template <typename T>
__global__ void __launch_bounds__(256) tail_fwd(TailSolveArgs a0, const T* __restrict__ L, const T* __restrict__ inv,
                                                T* x, T* vin) {
    TailSolveArgs a = a0;
    if (a.rstate) {
        a.act0 = a.act0 && a.rstate[4] == 0.0;
        a.act1 = a.act1 && a.rstate[12] == 0.0;
    }
    if (!a.act0 && !a.act1) return;
    __shared__ int s_b;
    __shared__ T acc[2][TB];
    __shared__ T xs[2][TB];
    __shared__ T part[4][2][TB];
    __shared__ __align__(16) T inv_s[TB * TB];
    const int tid = threadIdx.x, ri = tid & 63, kp = tid >> 6;
    if (tid == 0) s_b = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int b = s_b;
    const bool diag = b < a.nbd;
    const int row0 = diag ? b * TB : a.w + (b - a.nbd) * TB;
    const int rend = diag ? min(a.w, row0 + TB) : a.r;
    const int nrow = min(TB, rend - row0);
    const bool act[2] = {a.act0 != 0, a.act1 != 0};
    if (diag) {
        const T* I = inv + (int64_t)b * TB * TB;
#pragma unroll
        for (int e = tid; e < TB * TB; e += 256) inv_s[e] = I[e];
    }
    if (kp == 0) {
        for (int q = 0; q < 2; ++q) {
            T v = (T)0;
            if (act[q] && ri < nrow && diag) {
                const int col = a.c0 + row0 + ri;
                v = x[q * a.dim + col];
                const T* vq = vin + q * a.nv;
                const int64_t e1 = a.vn_hi[col];
                for (int64_t e0 = a.vn_lo[col]; e0 < e1; e0 += 4) {      // 4 entries in flight, fixed order
                    T u[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) u[k] = e0 + k < e1 ? __ldcg(vq + e0 + k) : (T)0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) v -= u[k];
                }
            }
            acc[q][ri] = v;
        }
    }
    const int nblk = diag ? b : a.nbd;
    for (int kb = 0; kb < nblk; ++kb) {
        const int kc = kb * TB, kn = min(TB, a.w - kc);
        T lv[TB / 4];
        const T* Lr = L + (int64_t)kc * a.r + row0 + ri;
#pragma unroll
        for (int u = 0; u < TB / 4; ++u) {
            const int k = kp + 4 * u;
            lv[u] = (ri < nrow && k < kn) ? Lr[(int64_t)k * a.r] : (T)0;
        }
        if (tid == 0) wait_flag(a.flags + kb);
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, k = tid & 63;
            xs[q][k] = (act[q] && k < kn) ? __ldcg(x + q * a.dim + a.c0 + kc + k) : (T)0;
        }
        __syncthreads();
        T p0 = (T)0, p1 = (T)0;
#pragma unroll
        for (int u = 0; u < TB / 4; ++u) {
            p0 += lv[u] * xs[0][kp + 4 * u];
            p1 += lv[u] * xs[1][kp + 4 * u];
        }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (kp == 0)          // acc row ri is only touched by this thread: no barrier after it
            for (int q = 0; q < 2; ++q)
                acc[q][ri] -= ((part[0][q][ri] + part[1][q][ri]) + part[2][q][ri]) + part[3][q][ri];
    }
    __syncthreads();
    if (diag) {
        // x_b = inv(L_bb) * acc (row-major lower inverse, staged in shared memory)
        T p0 = (T)0, p1 = (T)0;
        if (ri < nrow)
            for (int t = kp; t <= ri; t += 4) {
                const T iv = inv_s[ri * TB + t];
                p0 += iv * acc[0][t];
                p1 += iv * acc[1][t];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (kp == 0 && ri < nrow)
            for (int q = 0; q < 2; ++q)
                if (act[q]) x[q * a.dim + a.c0 + row0 + ri] = ((part[0][q][ri] + part[1][q][ri]) + part[2][q][ri]) + part[3][q][ri];
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release(a.flags + b, 1);
    } else if (kp == 0 && ri < nrow) {
        const int64_t pos = a.vpush_pos[a.cvo + (row0 + ri - a.w)];
        for (int q = 0; q < 2; ++q)
            if (act[q]) vin[q * a.nv + pos] = -acc[q][ri];
    }
}

// backward: CTA per column block, last block first.  Warp w owns columns
// j = w, w+8, ... (lanes over rows: coalesced column reads); each warp polls the
// flags itself, with that block's L values already in registers, so there is
// no CTA barrier per block; the inverse block is staged in shared memory.
template <typename T>
__global__ void __launch_bounds__(256) tail_bwd(TailSolveArgs a0, const T* __restrict__ L, const T* __restrict__ inv,
                                                const T* __restrict__ dvec, T* x) {
    TailSolveArgs a = a0;
    if (a.rstate) {
        a.act0 = a.act0 && a.rstate[4] == 0.0;
        a.act1 = a.act1 && a.rstate[12] == 0.0;
    }
    if (!a.act0 && !a.act1) return;
    __shared__ int s_b;
    __shared__ T acc[2][TB];
    __shared__ __align__(16) T inv_s[TB * TB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_b = a.nbd - 1 - atomicAdd(a.ticket, 1);
    __syncthreads();
    const int b = s_b;
    const int col0 = b * TB;
    const int ncol = min(TB, a.w - col0);
    const bool act[2] = {a.act0 != 0, a.act1 != 0};
    {
        const T* I = inv + (int64_t)b * TB * TB;
#pragma unroll
        for (int e = tid; e < TB * TB; e += 256) inv_s[e] = I[e];
    }
    // off rows (ancestors' x is final)
    for (int j = warp; j < ncol; j += 8) {
        const T* Lc = L + (int64_t)(col0 + j) * a.r;
        T s0 = (T)0, s1 = (T)0;
        // 8 rows per lane in flight: the index -> value gathers are latency-bound
        // (narrow tail supernodes have thousands of off rows)
        for (int i0 = a.w + lane; i0 < a.r; i0 += 32 * 8) {
            int gi[8];
            T l[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + 32 * u;
                gi[u] = i < a.r ? a.rows[i] : -1;
                l[u] = i < a.r ? Lc[i] : (T)0;
            }
            T v0[8], v1[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                v0[u] = (act[0] && gi[u] >= 0) ? __ldcg(x + gi[u]) : (T)0;
                v1[u] = (act[1] && gi[u] >= 0) ? __ldcg(x + a.dim + gi[u]) : (T)0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                s0 += l[u] * v0[u];
                s1 += l[u] * v1[u];
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_down_sync(0xffffffffu, s0, o);
            s1 += __shfl_down_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
            const int gc = a.c0 + col0 + j;
            const T dj = dvec[gc];
            acc[0][j] = act[0] ? __ldcg(x + gc) / dj - s0 : (T)0;
            acc[1][j] = act[1] ? __ldcg(x + a.dim + gc) / dj - s1 : (T)0;
        }
    }
    // later own blocks, last first
    for (int kb = a.nbd - 1; kb > b; --kb) {
        const int r0 = kb * TB, rn = min(TB, a.w - r0);
        T l0[TB / 8], l1[TB / 8];
#pragma unroll
        for (int c = 0; c < TB / 8; ++c) {
            const int j = warp + 8 * c;
            const T* Lc = L + (int64_t)(col0 + j) * a.r + r0;
            l0[c] = (j < ncol && lane < rn) ? Lc[lane] : (T)0;
            l1[c] = (j < ncol && lane + 32 < rn) ? Lc[lane + 32] : (T)0;
        }
        if (lane == 0) wait_flag(a.flags + kb);
        __syncwarp();
        T xa[2], xb[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            xa[q] = (act[q] && lane < rn) ? __ldcg(x + q * a.dim + a.c0 + r0 + lane) : (T)0;
            xb[q] = (act[q] && lane + 32 < rn) ? __ldcg(x + q * a.dim + a.c0 + r0 + lane + 32) : (T)0;
        }
        T s[TB / 8][2];
#pragma unroll
        for (int c = 0; c < TB / 8; ++c)
#pragma unroll
            for (int q = 0; q < 2; ++q) s[c][q] = l0[c] * xa[q] + l1[c] * xb[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int c = 0; c < TB / 8; ++c)
#pragma unroll
                for (int q = 0; q < 2; ++q) s[c][q] += __shfl_down_sync(0xffffffffu, s[c][q], o);
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < TB / 8; ++c) {
                const int j = warp + 8 * c;
                if (j < ncol) {
                    acc[0][j] -= s[c][0];
                    acc[1][j] -= s[c][1];
                }
            }
    }
    __syncthreads();
    // x_b = inv(L_bb)' * acc
    if (tid < 2 * TB) {
        const int q = tid >> 6, j = tid & 63;
        if (act[q] && j < ncol) {
            T v = (T)0;
            for (int t = j; t < ncol; ++t) v += inv_s[t * TB + j] * acc[q][t];
            x[q * a.dim + a.c0 + col0 + j] = v;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        st_release(a.flags + b, 1);
        if (b == 0) st_release(a.done, 1);
    }
}

// ---------------------------------------------------------------------------
// single dense ROOT (the whole tail is one supernode with no off rows, w <= 256:
// C2, C3, C5a): forward, D and backward solve of the root in ONE CTA of 1024
// threads, right-hand sides in shared memory — replaces the tail_fwd / tail_bwd
// pair (multi-CTA wavefronts that synchronise through global flags, ~20 us each
// for a 4-block root) with block GEMVs separated by CTA barriers.
//   forward  y_b = inv(L_bb) (t_b - sum_{k<b} L_bk y_k)      (inv row-major, per 64-block)
//   backward x_b = inv(L_bb)' (y_b / D_b - sum_{i>b} L_ib' x_i)
// Partial sums: 16 threads per row / column, fixed-order combination.
// ---------------------------------------------------------------------------
constexpr int RT = 1024, RP = RT / TB;      // threads, partial sums per row (16)

template <typename T>
__global__ void __launch_bounds__(RT) root_solve(TailSolveArgs a0, const T* __restrict__ L, const T* __restrict__ inv,
                                                 const T* __restrict__ dvec, T* x, const T* __restrict__ vin) {
    TailSolveArgs a = a0;
    if (a.rstate) {
        a.act0 = a.act0 && a.rstate[4] == 0.0;
        a.act1 = a.act1 && a.rstate[12] == 0.0;
    }
    const int tid = threadIdx.x;
    const int w = a.w, r = a.r;
    __shared__ T xs[2][256];
    __shared__ T acc[2][TB];
    __shared__ T part[RP][2][TB];
    if (!a.act0 && !a.act1) {
        if (tid == 0) st_release(a.done, 1);
        return;
    }
    const bool act[2] = {a.act0 != 0, a.act1 != 0};
    // 1. right-hand side of the root columns minus the non-tiny vector inbox
    for (int e = tid; e < 2 * w; e += RT) {
        const int q = e / w, j = e - q * w;
        T v = (T)0;
        if (act[q]) {
            const int col = a.c0 + j;
            v = x[q * a.dim + col];
            const T* vq = vin + q * a.nv;
            for (int64_t p = a.vn_lo[col]; p < a.vn_hi[col]; ++p) v -= __ldcg(vq + p);
        }
        xs[q][j] = v;
    }
    __syncthreads();
    const int ri = tid & (TB - 1), kp = tid >> 6;       // row / column within the block, partial index
    // 2. forward, block by block
    for (int b = 0; b < a.nbd; ++b) {
        const int row0 = b * TB, nb = min(TB, w - row0);
        T p0 = (T)0, p1 = (T)0;
        if (ri < nb)
            for (int k = kp; k < row0; k += RP) {
                const T l = L[(int64_t)k * r + row0 + ri];
                p0 += l * xs[0][k];
                p1 += l * xs[1][k];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, i = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][i];
            acc[q][i] = i < nb ? xs[q][row0 + i] - s : (T)0;
        }
        __syncthreads();
        const T* Ib = inv + (int64_t)b * TB * TB;           // row-major lower inverse of L_bb
        p0 = (T)0;
        p1 = (T)0;
        if (ri < nb)
            for (int t = kp; t <= ri; t += RP) {
                const T iv = Ib[ri * TB + t];
                p0 += iv * acc[0][t];
                p1 += iv * acc[1][t];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, i = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][i];
            if (i < nb) xs[q][row0 + i] = s;
        }
        __syncthreads();
    }
    // 3. D solve (ldl.py:101-102)
    for (int e = tid; e < 2 * w; e += RT) {
        const int q = e / w, j = e - q * w;
        xs[q][j] = xs[q][j] / dvec[a.c0 + j];
    }
    __syncthreads();
    // 4. backward, last block first
    for (int b = a.nbd - 1; b >= 0; --b) {
        const int col0 = b * TB, nb = min(TB, w - col0), i0 = col0 + nb;
        T p0 = (T)0, p1 = (T)0;
        if (ri < nb) {
            const T* Lc = L + (int64_t)(col0 + ri) * r;
            for (int i = i0 + kp; i < w; i += RP) {
                const T l = Lc[i];
                p0 += l * xs[0][i];
                p1 += l * xs[1][i];
            }
        }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, j = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][j];
            acc[q][j] = j < nb ? xs[q][col0 + j] - s : (T)0;
        }
        __syncthreads();
        const T* Ib = inv + (int64_t)b * TB * TB;
        p0 = (T)0;
        p1 = (T)0;
        if (ri < nb)
            for (int t = ri + kp; t < nb; t += RP) {          // x_j = sum_{t >= j} inv[t][j] acc_t
                const T iv = Ib[t * TB + ri];
                p0 += iv * acc[0][t];
                p1 += iv * acc[1][t];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, j = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][j];
            if (j < nb) xs[q][col0 + j] = s;
        }
        __syncthreads();
    }
    for (int e = tid; e < 2 * w; e += RT) {
        const int q = e / w, j = e - q * w;
        if (act[q]) x[q * a.dim + a.c0 + j] = xs[q][j];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(a.done, 1);
}

// root_solve with the root's factor and block inverses staged in shared memory
// first (cp.async, all in flight at once): every block GEMV of the substitution
// then reads shared memory instead of a chain of dependent L2 loads.
constexpr int RIB = TB * (TB + 1) / 2;      // packed lower triangle of one 64 x 64 inverse block
__device__ __forceinline__ int root_pk(int j, int w) { return j * w - ((j * (j - 1)) >> 1); }
template <typename T>
constexpr int root_solve_smem(int w) {
    return (int)sizeof(T) * (((w * (w + 1) / 2 + 3) & ~3) + ((w + TB - 1) / TB) * RIB);
}

template <typename T>
__global__ void __launch_bounds__(RT) root_solve_s(TailSolveArgs a0, const T* __restrict__ L, const T* __restrict__ inv,
                                                 const T* __restrict__ dvec, T* x, const T* __restrict__ vin) {
    TailSolveArgs a = a0;
    if (a.rstate) {
        a.act0 = a.act0 && a.rstate[4] == 0.0;
        a.act1 = a.act1 && a.rstate[12] == 0.0;
    }
    const int tid = threadIdx.x;
    const int w = a.w, r = a.r;
    __shared__ T xs[2][256];
    __shared__ T acc[2][TB];
    __shared__ T part[RP][2][TB];
    if (!a.act0 && !a.act1) {
        if (tid == 0) st_release(a.done, 1);
        return;
    }
    const bool act[2] = {a.act0 != 0, a.act1 != 0};
    // stage the root's factor (packed lower, Ls[cs[k] + i - k] = L(i, k)) and the
    // lower triangles of its 64 x 64 diagonal-block inverses (Is, row-major packed)
    // in shared memory with cp.async; the right-hand side is assembled meanwhile
    extern __shared__ __align__(16) unsigned char rss_raw[];
    T* Ls = reinterpret_cast<T*>(rss_raw);
    T* Is = Ls + ((w * (w + 1) / 2 + 3) & ~3);
    __shared__ int cs[257];
    {
        const int lane = tid & 31, wid = tid >> 5;
        for (int k = wid; k < w; k += RT / 32) {
            const int ck = root_pk(k, w) - k;
            for (int i = k + lane; i < w; i += 32) cp_async_elem(Ls + ck + i, L + (int64_t)k * r + i, true);
        }
        for (int row = wid; row < a.nbd * TB; row += RT / 32) {
            const int bb = row / TB, ri = row - bb * TB;
            if (bb * TB + ri >= w) continue;
            T* dst = Is + bb * RIB + ri * (ri + 1) / 2;
            const T* src = inv + (int64_t)bb * TB * TB + ri * TB;
            for (int t = lane; t <= ri; t += 32) cp_async_elem(dst + t, src + t, true);
        }
        cp_async_commit();
        for (int j = tid; j <= w; j += RT) cs[j] = root_pk(j, w);
    }
    // 1. right-hand side of the root columns minus the non-tiny vector inbox
    for (int e = tid; e < 2 * w; e += RT) {
        const int q = e / w, j = e - q * w;
        T v = (T)0;
        if (act[q]) {
            const int col = a.c0 + j;
            v = x[q * a.dim + col];
            const T* vq = vin + q * a.nv;
            for (int64_t p = a.vn_lo[col]; p < a.vn_hi[col]; ++p) v -= __ldcg(vq + p);
        }
        xs[q][j] = v;
    }
    __syncthreads();
    cp_async_wait<0>();
    __syncthreads();
    const int ri = tid & (TB - 1), kp = tid >> 6;       // row / column within the block, partial index
    // 2. forward, block by block
    for (int b = 0; b < a.nbd; ++b) {
        const int row0 = b * TB, nb = min(TB, w - row0);
        T p0 = (T)0, p1 = (T)0;
        if (ri < nb)
            for (int k = kp; k < row0; k += RP) {
                const T l = Ls[cs[k] + row0 + ri - k];
                p0 += l * xs[0][k];
                p1 += l * xs[1][k];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, i = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][i];
            acc[q][i] = i < nb ? xs[q][row0 + i] - s : (T)0;
        }
        __syncthreads();
        const T* Ib = Is + b * RIB + ri * (ri + 1) / 2;     // row ri of the lower inverse of L_bb
        p0 = (T)0;
        p1 = (T)0;
        if (ri < nb)
            for (int t = kp; t <= ri; t += RP) {
                const T iv = Ib[t];
                p0 += iv * acc[0][t];
                p1 += iv * acc[1][t];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, i = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][i];
            if (i < nb) xs[q][row0 + i] = s;
        }
        __syncthreads();
    }
    // 3. D solve (ldl.py:101-102)
    for (int e = tid; e < 2 * w; e += RT) {
        const int q = e / w, j = e - q * w;
        xs[q][j] = xs[q][j] / dvec[a.c0 + j];
    }
    __syncthreads();
    // 4. backward, last block first
    for (int b = a.nbd - 1; b >= 0; --b) {
        const int col0 = b * TB, nb = min(TB, w - col0), i0 = col0 + nb;
        T p0 = (T)0, p1 = (T)0;
        if (ri < nb) {
            const T* Lc = Ls + cs[col0 + ri] - (col0 + ri);
            for (int i = i0 + kp; i < w; i += RP) {
                const T l = Lc[i];
                p0 += l * xs[0][i];
                p1 += l * xs[1][i];
            }
        }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, j = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][j];
            acc[q][j] = j < nb ? xs[q][col0 + j] - s : (T)0;
        }
        __syncthreads();
        const T* Ib = Is + b * RIB;
        p0 = (T)0;
        p1 = (T)0;
        if (ri < nb)
            for (int t = ri + kp; t < nb; t += RP) {          // x_j = sum_{t >= j} inv[t][j] acc_t
                const T iv = Ib[t * (t + 1) / 2 + ri];
                p0 += iv * acc[0][t];
                p1 += iv * acc[1][t];
            }
        part[kp][0][ri] = p0;
        part[kp][1][ri] = p1;
        __syncthreads();
        if (tid < 2 * TB) {
            const int q = tid >> 6, j = tid & (TB - 1);
            T s = (T)0;
            for (int k = 0; k < RP; ++k) s += part[k][q][j];
            if (j < nb) xs[q][col0 + j] = s;
        }
        __syncthreads();
    }
    for (int e = tid; e < 2 * w; e += RT) {
        const int q = e / w, j = e - q * w;
        if (act[q]) x[q * a.dim + a.c0 + j] = xs[q][j];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(a.done, 1);
}

template <typename T>
void tail_factor_t(Ctx& c) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tail_diag<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem<T>());
        cudaFuncSetAttribute(tail_gemm<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem<T>());
        cudaFuncSetAttribute(tail_gemm<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem<T>());
        cudaFuncSetAttribute(tail_gemm<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem<T>());
        attr = true;
    }
    T* L = (T*)c.lval;
    T* D = (T*)c.dvec;
    T* inbox = (T*)c.inbox;
    T* inv = (T*)c.tinv;
    const Symbolic& S = c.host_sym;
    auto run_node = [&](const TailNode& t, cudaStream_t ms, cudaStream_t ss, cudaEvent_t* ev) {
        T* P = L + t.loff;
        const int r = t.r, w = t.w, o = r - w;
        tail_gather<T><<<(r + 7) / 8, 256, 0, ms>>>(P, r, c.sym.irow_ptr + t.r0, c.sym.inbox_tgt, inbox);
        c.launches++;
        // right-looking by 64-column panels with look-ahead: panel k's trailing update
        // is split into "next" (the columns of panel k+1, main stream: they gate
        // panel k+1's diagonal block), "rest1" (panel k+2's columns) and "rest2" (the
        // remainder), both on tail_side, so the diagonal block and TRSM of panel k+1
        // overlap the bulk of panel k's update.  Events: T = panel k's TRSM done
        // (side may start), E1 = rest1(k) done (next(k+1) writes the same columns;
        // side-stream order also puts rest2(k-1) before it).
        static const bool lookahead_env = !getenv("CIPM_TAIL_NO_LOOKAHEAD");
        const bool la = lookahead_env && w > 2 * TB;
        bool e1_pending = false, side_used = false;
        for (int kb = 0; kb < w; kb += TB) {
            const int nb = std::min(TB, w - kb);
            const int b = kb / TB;
            T* inv_rm = inv + t.inv_off + (int64_t)b * TB * TB;
            T* inv_cm = inv + t.inv_off + (int64_t)(t.nbd + b) * TB * TB;
            tail_diag<T><<<1, 256, diag_smem<T>(), ms>>>(P, r, kb, nb, t.c0, D, c.sym.sign, c.sn_maxd + t.J,
                                                              c.bumps, c.err, c.delta_s, c.delta_d, inv_rm, inv_cm);
            c.launches++;
            const int below = r - kb - nb;
            if (below > 0) {
                // L21 = A21 L11^-T D^-1 as a GEMM with the column-major inverse (DMMA in FP64)
                T* A21 = P + (int64_t)kb * r + kb + nb;
                dim3 g((below + GB - 1) / GB, 1);
                tail_gemm<T, 2><<<g, 128, gemm_smem<T>(), ms>>>(A21, r, inv_cm, TB, nullptr, below, nb, nb, 1 << 30, A21, r,
                                                         nullptr, nullptr, D + t.c0 + kb);
                c.launches++;
            }
            const int Mr = r - kb - nb, Nc = w - kb - nb;
            if (Nc <= 0) continue;
            const T* A = P + (int64_t)kb * r + kb + nb;
            const T* Dk = D + t.c0 + kb;
            T* C0 = P + (int64_t)(kb + nb) * r + kb + nb;
            // trailing update of the columns [j0, j1) of the trailing block (rows j0.. of A)
            auto update = [&](cudaStream_t st, int j0, int j1) {
                const int M = Mr - j0, N = j1 - j0;
                if (M <= 0 || N <= 0) return;
                dim3 g((M + GB - 1) / GB, (N + GB - 1) / GB);
                tail_gemm<T, 0><<<g, 128, gemm_smem<T>(), st>>>(A + j0, r, A + j0, r, Dk, M, N, nb, 0,
                                                               C0 + (int64_t)j0 * r + j0, r, nullptr, nullptr, nullptr);
                c.launches++;
            };
            if (!la) {
                update(ms, 0, Nc);
                continue;
            }
            // side: rest1 / rest2 of this panel, after its TRSM
            if (Nc > TB) {
                cudaEventRecord(ev[0], ms);
                cudaStreamWaitEvent(ss, ev[0], 0);
            }
            // main: next (panel k+1's columns), after rest1 of panel k-1
            if (e1_pending) cudaStreamWaitEvent(ms, ev[1], 0);
            update(ms, 0, std::min(TB, Nc));
            if (Nc > TB) {
                update(ss, TB, std::min(2 * TB, Nc));
                cudaEventRecord(ev[1], ss);
                e1_pending = true;
                update(ss, 2 * TB, Nc);
                side_used = true;
            } else {
                e1_pending = false;
            }
        }
        if (side_used) {
            cudaEventRecord(ev[2], ss);
            cudaStreamWaitEvent(ms, ev[2], 0);
        }
        if (o > 0) {
            const T* A = P + w;
            dim3 g((o + GB - 1) / GB, (o + GB - 1) / GB);
            tail_gemm<T, 1><<<g, 128, gemm_smem<T>(), ms>>>(A, r, A, r, D + t.c0, o, o, w, 0, nullptr, 0,
                                                     c.sym.push_pos + S.cb_off[t.J], inbox, nullptr);
            c.launches++;
        }
        tail_finish<<<1, 1, 0, ms>>>(c.sn_maxd, c.fac_count, t.J, t.parent);
        c.launches++;
    };
    static const bool par_env = !getenv("CIPM_TAIL_SERIAL_LEVELS");
    for (const auto& level : c.tail_levels) {
        if (level.size() == 1 || !par_env || c.tail_pool.empty()) {
            for (int i : level) run_node(c.tail[i], c.stream, c.tail_side, c.tail_ev);
            continue;
        }
        // independent nodes: parallel branches (fork / join through events)
        const int P = (int)c.tail_pool.size();
        cudaEventRecord(c.tail_fork, c.stream);
        const int used = std::min<int>(P, (int)level.size());
        for (int k = 0; k < used; ++k) cudaStreamWaitEvent(c.tail_pool[k], c.tail_fork, 0);
        for (size_t q = 0; q < level.size(); ++q) {
            const int k = (int)(q % P);
            run_node(c.tail[level[q]], c.tail_pool[k], c.tail_pool_side[k], &c.tail_pool_ev[4 * k]);
        }
        for (int k = 0; k < used; ++k) {
            cudaEventRecord(c.tail_pool_ev[4 * k + 3], c.tail_pool[k]);
            cudaStreamWaitEvent(c.stream, c.tail_pool_ev[4 * k + 3], 0);
        }
    }
}

TailSolveArgs tail_args(Ctx& c, const TailNode& t, int which, int act0, int act1) {
    TailSolveArgs a;
    a.c0 = t.c0;
    a.w = t.w;
    a.r = t.r;
    a.nbd = t.nbd;
    a.dim = c.dim;
    a.nv = c.sym.nv;
    a.cvo = c.host_sym.cv_off[t.J];
    a.rows = c.sym.sn_rows + t.r0;
    a.vn_lo = c.sym.vn_lo;
    a.vn_hi = c.sym.vn_hi;
    a.vpush_pos = c.sym.vpush_pos;
    a.flags = c.tflags + t.flag_off + (which ? t.nbd : 0);
    a.ticket = c.tflags + t.flag_off + 2 * t.nbd + which;
    a.done = c.bwd_done + t.J;
    a.act0 = act0;
    a.act1 = act1;
    a.rstate = c.rstate;
    return a;
}

// the nodes of one tail level (mutually independent): one node on the main
// stream, several as parallel branches over the stream pool (fork / join)
template <typename F>
void tail_level_run(Ctx& c, const std::vector<int>& level, F&& one) {
    static const bool par_env = !getenv("CIPM_TAIL_SERIAL_LEVELS");
    if (level.size() == 1 || !par_env || c.tail_pool.empty()) {
        for (int i : level) one(c.tail[i], c.stream);
        return;
    }
    const int P = (int)c.tail_pool.size();
    cudaEventRecord(c.tail_fork, c.stream);
    const int used = std::min<int>(P, (int)level.size());
    for (int k = 0; k < used; ++k) cudaStreamWaitEvent(c.tail_pool[k], c.tail_fork, 0);
    for (size_t q = 0; q < level.size(); ++q) one(c.tail[level[q]], c.tail_pool[q % P]);
    for (int k = 0; k < used; ++k) {
        cudaEventRecord(c.tail_pool_ev[4 * k + 3], c.tail_pool[k]);
        cudaStreamWaitEvent(c.stream, c.tail_pool_ev[4 * k + 3], 0);
    }
}

template <typename T>
void tail_forward_t(Ctx& c, T* x, int act0, int act1) {
    auto one = [&](const TailNode& t, cudaStream_t st) {
        const int blocks = t.nbd + (t.r - t.w + TB - 1) / TB;
        tail_fwd<T><<<blocks, 256, 0, st>>>(tail_args(c, t, 0, act0, act1), (const T*)c.lval + t.loff,
                                            (const T*)c.tinv + t.inv_off, x, (T*)c.vin);
        c.launches++;
    };
    for (size_t l = 0; l < c.tail_levels.size(); ++l) tail_level_run(c, c.tail_levels[l], one);
}

template <typename T>
void root_solve_t(Ctx& c, T* x, int act0, int act1) {
    const TailNode& t = c.tail[0];
    const int sm = root_solve_smem<T>(t.w);
    static const bool staged_env = !getenv("CIPM_ROOT_UNSTAGED");
    if (staged_env && sm <= 200 * 1024) {
        static int attr = 0;
        if (attr < sm) {
            cudaFuncSetAttribute(root_solve_s<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            attr = 200 * 1024;
        }
        root_solve_s<T><<<1, RT, sm, c.stream>>>(tail_args(c, t, 1, act0, act1), (const T*)c.lval + t.loff,
                                                 (const T*)c.tinv + t.inv_off, (const T*)c.dvec, x, (const T*)c.vin);
    } else {
        root_solve<T><<<1, RT, 0, c.stream>>>(tail_args(c, t, 1, act0, act1), (const T*)c.lval + t.loff,
                                              (const T*)c.tinv + t.inv_off, (const T*)c.dvec, x, (const T*)c.vin);
    }
    c.launches++;
}

template <typename T>
void tail_backward_t(Ctx& c, T* x, int act0, int act1) {
    auto one = [&](const TailNode& t, cudaStream_t st) {
        tail_bwd<T><<<t.nbd, 256, 0, st>>>(tail_args(c, t, 1, act0, act1), (const T*)c.lval + t.loff,
                                           (const T*)c.tinv + t.inv_off, (const T*)c.dvec, x);
        c.launches++;
    };
    for (size_t l = c.tail_levels.size(); l-- > 0;) tail_level_run(c, c.tail_levels[l], one);
}

}  // namespace

void tail_setup(Ctx& c, int64_t* inv_total, int64_t* flag_total) {
    const Symbolic& S = c.host_sym;
    c.tail.clear();
    int64_t io = 0, fo = 0;
    for (int32_t k = S.n_main; k < S.nsuper; ++k) {
        const int32_t J = S.order[k];
        TailNode t;
        t.J = J;
        t.c0 = S.sn_col[J];
        t.w = S.sn_col[J + 1] - S.sn_col[J];
        t.r0 = S.sn_rptr[J];
        t.r = (int)(S.sn_rptr[J + 1] - S.sn_rptr[J]);
        t.loff = S.sn_loff[J];
        t.parent = S.sn_parent[J];
        t.nbd = (t.w + TB - 1) / TB;
        t.inv_off = io;
        t.flag_off = fo;
        io += 2 * (int64_t)t.nbd * TB * TB;     // row-major (solves) + column-major (TRSM GEMM) inverses
        fo += 2 * t.nbd + 2;
        c.tail.push_back(t);
    }
    c.tflag_total = fo;
    *inv_total = io;
    *flag_total = fo;
    // levels of the tail forest (children first): nodes of one level are independent
    std::vector<int> lev(c.tail.size(), 0);
    std::vector<int> idx_of(S.nsuper, -1);
    for (size_t i = 0; i < c.tail.size(); ++i) idx_of[c.tail[i].J] = (int)i;
    int nlev = 0;
    for (size_t i = 0; i < c.tail.size(); ++i) {
        const int p = c.tail[i].parent >= 0 ? idx_of[c.tail[i].parent] : -1;
        if (p >= 0) lev[p] = std::max(lev[p], lev[i] + 1);
        nlev = std::max(nlev, lev[i] + 1);
    }
    c.tail_levels.assign(nlev, {});
    for (size_t i = 0; i < c.tail.size(); ++i) c.tail_levels[lev[i]].push_back((int)i);
}

void k_tail_factor(Ctx& c) {
    if (c.tail.empty()) return;
    if (c.precision == CIPM_FULL) tail_factor_t<double>(c);
    else tail_factor_t<float>(c);
}

void k_tail_forward(Ctx& c, void* x, int act0, int act1) {
    if (c.tail.empty()) return;
    if (c.precision == CIPM_FULL) tail_forward_t<double>(c, (double*)x, act0, act1);
    else tail_forward_t<float>(c, (float*)x, act0, act1);
}

bool tail_is_single_root(const Ctx& c) {
    return c.tail.size() == 1 && c.tail[0].r == c.tail[0].w && c.tail[0].w <= 256 && !getenv("CIPM_NO_ROOT_SOLVE");
}

void k_root_solve(Ctx& c, void* x, int act0, int act1) {
    if (c.precision == CIPM_FULL) root_solve_t<double>(c, (double*)x, act0, act1);
    else root_solve_t<float>(c, (float*)x, act0, act1);
}

void k_tail_backward(Ctx& c, void* x, int act0, int act1) {
    if (c.tail.empty()) return;
    if (c.precision == CIPM_FULL) tail_backward_t<double>(c, (double*)x, act0, act1);
    else tail_backward_t<float>(c, (float*)x, act0, act1);
}

}  // namespace cipm
