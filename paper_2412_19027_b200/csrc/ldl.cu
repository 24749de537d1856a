// Supernodal quasi-definite LDL' on sm_100a: numeric refactorisation and
// triangular solves (replaces kkt/ldl.py:37-104 and kkt/system.py:246-271).
//
// Scheduling — continuation, not polling.  Every persistent launch starts from
// a list of seed supernodes (those without children in its tier).  A task
// (warp or CTA) processes its supernode, publishes its outputs, fences, and
// increments its parent's same-tier child counter; the task whose increment
// completes the count continues directly with the parent.  Nothing spins,
// every supernode is processed exactly once, and the critical path of the
// elimination tree is walked by one task without hand-offs.  The backward
// sweep (root first) hands supernodes out by ticket in reverse topological
// order and waits on the parent's done flag.
//
// Numerics: push/pull inboxes.  A finished supernode K computes its
// contribution block C_K = L_off D L_off' and scatters it to the inbox slots
// of its ancestors; supernode J sums its inbox with fixed-order segmented
// scans.  No atomics touch floating-point data, so factors and solutions are
// bitwise reproducible run to run (SPEC kkt-solver "Determinism").
// Dynamic regularisation (ldl.py:79-87): a pivot with |d| < δs + δd·runmax is
// replaced by ±bound with the sign of its block; runmax is the largest |D| in
// the supernode's subtree computed so far (the sequential reference uses all
// earlier pivots; δd = eps² makes the term negligible — DESIGN.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

// tiny-leaf kernels: threads per block and minimum resident blocks (launch bounds)
#ifndef TINY_T
#define TINY_T 128
#endif
#ifndef TINY_MINB
#define TINY_MINB 1
#endif
#include "ctx.hpp"

namespace cipm {

namespace {

__device__ __forceinline__ int64_t gtimer() {
    int64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// device-side refinement state: a right-hand side is active while its done flag is 0
__device__ __forceinline__ void resolve_act(const double* rstate, int& act0, int& act1) {
    if (rstate) {
        act0 = act0 && rstate[4] == 0.0;
        act1 = act1 && rstate[12] == 0.0;
    }
}

// ---------------------------------------------------------------------------
// base image / assembly
// ---------------------------------------------------------------------------

template <typename T>
__global__ void scatter_vals(T* base, const int64_t* map, const double* vals, int64_t cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    int64_t p = map[i];
    if (p >= 0) base[p] = (T)vals[i];
}

template <typename T>
__global__ void add_static_reg(T* base, const int64_t* map_diag, int64_t n, int64_t dim, double delta_s) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= dim) return;
    T reg = (T)delta_s;
    T sgn = i < n ? (T)1 : (T)-1;
    base[map_diag[i]] = base[map_diag[i]] + sgn * reg;
}

// ---------------------------------------------------------------------------
// shared pieces
// ---------------------------------------------------------------------------

// per-supernode descriptor (symbolic.hpp desc32 / desc64), loaded by lanes 0..15 in one round trip
struct Desc {
    int c0, w, r, parent, tier;
    int64_t loff, cvo, vlo, vhi, ilo, ihi, cb, rptr;
};

__device__ __forceinline__ Desc desc_from_regs(int v32, int64_t v64) {
    Desc d;
    d.c0 = __shfl_sync(0xffffffffu, v32, 0);
    d.w = __shfl_sync(0xffffffffu, v32, 1);
    d.r = __shfl_sync(0xffffffffu, v32, 2);
    d.parent = __shfl_sync(0xffffffffu, v32, 3);
    d.tier = __shfl_sync(0xffffffffu, v32, 6);
    d.loff = __shfl_sync(0xffffffffu, v64, 8);
    d.cvo = __shfl_sync(0xffffffffu, v64, 9);
    d.vlo = __shfl_sync(0xffffffffu, v64, 10);
    d.vhi = __shfl_sync(0xffffffffu, v64, 11);
    d.ilo = __shfl_sync(0xffffffffu, v64, 12);
    d.ihi = __shfl_sync(0xffffffffu, v64, 13);
    d.cb = __shfl_sync(0xffffffffu, v64, 14);
    d.rptr = __shfl_sync(0xffffffffu, v64, 15);
    return d;
}

__device__ __forceinline__ Desc load_desc(const int32_t* __restrict__ d32, const int64_t* __restrict__ d64, int J) {
    const int lane = threadIdx.x & 31;
    const int v32 = lane < 8 ? __ldg(d32 + (int64_t)J * 8 + lane) : 0;
    const int64_t v64 = (lane >= 8 && lane < 16) ? __ldg(d64 + (int64_t)J * 8 + (lane - 8)) : 0;
    return desc_from_regs(v32, v64);
}

__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// Warp-cooperative segmented gather: entries [lo, hi) sorted so that equal
// targets are contiguous; P[tgt] -= sum of their values (fixed order: a warp
// Hillis-Steele scan per 32-entry chunk, carries across chunks).  Four chunks
// are loaded before they are reduced.
template <typename T>
__device__ __forceinline__ void warp_gather_sub(T* P, const int32_t* __restrict__ tgt, const T* vals, int64_t lo,
                                                int64_t hi) {
    const int lane = threadIdx.x & 31;
    int carry_t = -1;
    T carry = (T)0;
    for (int64_t base0 = lo; base0 < hi; base0 += 128) {
        T vv[4];
        int tt[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t e = base0 + 32 * u + lane;
            const bool valid = e < hi;
            tt[u] = valid ? tgt[e] : -(lane + 2);
            vv[u] = valid ? __ldcg(vals + e) : (T)0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t base = base0 + 32 * u;
            if (base >= hi) break;
            const int tg = tt[u];
            T v = vv[u];
            const bool valid = base + lane < hi;
            const int t0 = __shfl_sync(0xffffffffu, tg, 0);
            if (carry_t >= 0 && t0 != carry_t) {
                if (lane == 0) P[carry_t] -= carry;
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
            if (valid && is_end && !(lane == 31 && more)) P[tg] -= tot;
            const int t31 = __shfl_sync(0xffffffffu, tg, 31);
            const T v31 = __shfl_sync(0xffffffffu, tot, 31);
            if (more) {
                carry_t = t31;
                carry = v31;
            }
            __syncwarp();
        }
    }
    __syncwarp();
}

// stage a panel (r*w elements, 16-byte aligned in HBM) in the warp's shared-memory
// slice with one TMA bulk copy when it fits; otherwise read it in place
template <typename T>
__device__ __forceinline__ T* stage_panel(T* L, int psize, T* slice, int cap, uint64_t* bar, uint32_t& phase) {
    const uint32_t bytes = ((uint32_t)psize * (uint32_t)sizeof(T) + 15u) & ~15u;
    if (bytes > (uint32_t)cap * (uint32_t)sizeof(T)) return L;
    fence_proxy_async_smem();     // every lane's earlier generic reads of the slice precede the async write
    __syncwarp();
    if ((threadIdx.x & 31) == 0) bulk_g2s(slice, L, bytes, bar);
    mbar_wait(bar, phase);
    phase ^= 1u;
    return slice;
}

// ---------------------------------------------------------------------------
// numeric factorisation
// ---------------------------------------------------------------------------

struct FactorArgs {
    int32_t nstart;      // seeds of this tier
    const int32_t* start;
    int32_t ntiny;       // tiny leaves (warp tier only; one lane each)
    const int32_t* tiny;
    int32_t* ticket_tiny;
    int tier;
    const int32_t* desc32;
    const int64_t* desc64;
    const int32_t* need;
    const int64_t* push_pos;
    const int32_t* inbox_tgt;
    const int64_t* irow_ptr;
    const int8_t* sign;
    int32_t* count;
    int32_t* ticket;
    double* maxd;        // max |D| over the subtree, accumulated by the children (atomic max)
    int32_t* bumps;
    int* err;
    double delta_s, delta_d;
    int64_t smem_cap;    // panel elements per warp slice (warp tier) / per CTA (CTA tier)
    int64_t* trace;      // optional per-task timeline (cipm_trace)
};


// packed column-major lower index e of an o x o block -> (column bb, row aa >= bb);
// column bb starts at tb(bb) = bb*o - bb*(bb-1)/2
__device__ __forceinline__ void unpack_lower(int e, int o, int& bb, int& aa) {
    const double t = 2.0 * o + 1.0;
    int b = (int)((t - sqrt(t * t - 8.0 * (double)e)) * 0.5);
    b = max(0, min(b, o - 1));
    while (b > 0 && b * o - b * (b - 1) / 2 > e) --b;
    while (b + 1 < o && (b + 1) * o - (b + 1) * b / 2 <= e) ++b;
    bb = b;
    aa = b + (e - (b * o - b * (b - 1) / 2));
}

// warp-tier task body: gather, panel LDL', write-back, contribution push.
// Forced inline so P keeps its address space at each call site.
constexpr bool kWarpPanelSmem = false;   // true: the original shared-memory right-looking loop

// warp-tier panel LDL' with the panel in registers: lane l owns rows l and l + 32
// (r <= 64), all w <= 16 columns; column j's top entries a_cj are broadcast through
// shared memory (the short pivot chain of tools/micro/diag16.cu), l_ij = a_ij / d_j
// as a multiply by the reciprocal, then a_ic -= l_ij a_cj for c in (j, w).
template <typename T, int NW>
__device__ __forceinline__ void warp_panel_regs(T* P, int c0, int w, int r, double& runmax, T* sDw,
                                                const int8_t* sSgw, const FactorArgs& a, T* __restrict__ dvec,
                                                T* sCol) {
    const int lane = threadIdx.x & 31;
    const bool h0 = lane < r, h1 = lane + 32 < r;
    T x0[NW], x1[NW];
#pragma unroll
    for (int c = 0; c < NW; ++c) {
        x0[c] = (c < w && h0) ? P[c * r + lane] : (T)0;
        x1[c] = (c < w && h1) ? P[c * r + lane + 32] : (T)0;
    }
    double ds_r = a.delta_s, dd_r = a.delta_d;
    asm volatile("" : "+d"(ds_r), "+d"(dd_r));
    const unsigned pos = __ballot_sync(0xffffffffu, lane < w && sSgw[lane] > 0);
    T d_mine = (T)0;
    int nbump = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        if (j < w) {
            T* col = sCol + (j & 1) * 32;
            col[lane] = x0[j];                         // a_lj for lanes l < w (top rows)
            __syncwarp();
            double dd = (double)col[j];
            const double bound = ds_r + dd_r * runmax;
            const bool bump = fabs(dd) < bound;
            dd = bump ? (((pos >> j) & 1u) ? bound : -bound) : dd;
            const T dt = (T)dd;
            runmax = fmax(runmax, fabs(dd));
            nbump += bump ? 1 : 0;
            const T inv = (T)1 / dt;
            if (lane == j) d_mine = dt;
            const T l0 = x0[j] * inv, l1 = x1[j] * inv;
#pragma unroll
            for (int c = j + 1; c < NW; ++c) {
                if (c < w) {
                    const T acj = col[c];
                    if (lane >= c) x0[c] -= l0 * acj;
                    x1[c] -= l1 * acj;                  // rows 32.. are below every top row
                }
            }
            x0[j] = lane > j ? l0 : (lane == j ? (T)1 : x0[j]);
            x1[j] = l1;
        }
    }
    if (lane < w) {
        sDw[lane] = d_mine;
        dvec[c0 + lane] = d_mine;
        if (d_mine == (T)0) set_error(a.err, CIPM_E_FACTOR);
    }
    if (lane == 0 && nbump) atomicAdd(a.bumps, nbump);
    int row = lane;
    asm volatile("" : "+r"(row));
#pragma unroll
    for (int c = 0; c < NW; ++c) {
        if (c < w && h0 && c <= row) P[c * r + row] = x0[c];
        if (c < w && h1) P[c * r + row + 32] = x1[c];
    }
    __syncwarp();
}

template <typename T>
__device__ __forceinline__ void warp_task_body(T* P, T* L, bool in_smem, const Desc& d, int c0, int w, int r, int o,
                                               double& runmax, T* sDw, const int8_t* sSgw, const FactorArgs& a,
                                               T* __restrict__ dvec, T* __restrict__ inbox, int J, T* sCol) {
    const int lane = threadIdx.x & 31;
    const int psize = r * w;
    // 1. gather the inbox of all r rows (one contiguous, target-sorted range)
    warp_gather_sub(P, a.inbox_tgt, inbox, d.ilo, d.ihi);
    if (a.trace && lane == 0) a.trace[6 * J + 3] = gtimer();
    // 2. dense LDL' of the panel (right-looking, lanes over rows)
    static_assert(true, "");
    // (2 x NW values per lane within the 64-register budget: FP64 up to 8 columns)
    if (r <= 64 && w <= 8 && !kWarpPanelSmem) {
        warp_panel_regs<T, 8>(P, c0, w, r, runmax, sDw, sSgw, a, dvec, sCol);
    } else if (sizeof(T) == 4 && r <= 64 && w <= 16 && !kWarpPanelSmem) {
        warp_panel_regs<T, 16>(P, c0, w, r, runmax, sDw, sSgw, a, dvec, sCol);
    } else {
    int nbump = 0;
    for (int j = 0; j < w; ++j) {
        T* Pj = P + j * r;
        double dd = (double)Pj[j];
        const double bound = a.delta_s + a.delta_d * runmax;
        const bool bump = fabs(dd) < bound;
        if (bump) dd = sSgw[j] > 0 ? bound : -bound;
        const T dt = (T)dd;
        runmax = fmax(runmax, fabs(dd));
        __syncwarp();
        nbump += bump ? 1 : 0;
        if (lane == 0) {
            if (dt == (T)0) set_error(a.err, CIPM_E_FACTOR);
            dvec[c0 + j] = dt;
            sDw[j] = dt;
            Pj[j] = (T)1;
        }
        for (int i = j + 1 + lane; i < r; i += 32) Pj[i] = Pj[i] / dt;
        __syncwarp();
        for (int c = j + 1; c < w; ++c) {
            const T pjc = Pj[c];
            T* Pc = P + c * r;
            for (int i = c + lane; i < r; i += 32) Pc[i] -= Pj[i] * dt * pjc;
        }
        __syncwarp();
    }
    if (lane == 0 && nbump) atomicAdd(a.bumps, nbump);
    }
    if (a.trace && lane == 0) a.trace[6 * J + 4] = gtimer();
    // 3. push C_J = L_off D L_off' into the ancestors' inboxes, then write the factor back
    if (o > 0) {
        // C_J entries flattened over the lanes (packed column-major lower), push
        // positions loaded coalesced
        const int ne = o * (o + 1) / 2;
        for (int e = lane; e < ne; e += 32) {
            const int64_t pos = __ldg(a.push_pos + d.cb + e);
            int bb, aa;
            unpack_lower(e, o, bb, aa);
            T acc = (T)0;
            for (int k = 0; k < w; ++k) acc += P[k * r + w + aa] * (sDw[k] * P[k * r + w + bb]);
            inbox[pos] = acc;
        }
    }
    __syncwarp();
    (void)in_smem;
    (void)psize;
    (void)L;
}

constexpr int FW = 8;   // warps per factor CTA (warp tier)

// Warp tier: one warp per supernode.  Stage the panel in the warp's shared
// slice (in place in HBM when it does not fit); gather its inbox; factor the
// dense panel (right-looking, lanes over rows); write L and D; compute and
// scatter C_J = L_off D L_off'; signal the parent and continue with it if
// this was its last child.
// tiny leaf (w <= 4, r <= 16, no inbox): the whole task in one lane's registers,
// specialised on the width W so the register arrays are statically indexed.
// Returns the parent if this leaf completed its parent's child count.
template <typename T, int W>
__device__ __forceinline__ int factor_tiny_w(int J, int c0, int r, int parent, int64_t loff, int64_t cb,
                                             const FactorArgs& a, T* __restrict__ lval, T* __restrict__ dvec,
                                             T* __restrict__ inbox, double* runmax_out) {
    T* L = lval + loff;
    T p[W][16];
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
        for (int i = 0; i < 16; ++i) p[j][i] = i < r ? L[j * r + i] : (T)0;
    double runmax = 0.0;        // a leaf has no subtree below it
    T dv[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        double dd = (double)p[j][j];
        const double bound = a.delta_s + a.delta_d * runmax;
        if (fabs(dd) < bound) {
            dd = a.sign[c0 + j] > 0 ? bound : -bound;
            atomicAdd(a.bumps, 1);
        }
        const T dt = (T)dd;
        if (dt == (T)0) set_error(a.err, CIPM_E_FACTOR);
        runmax = fmax(runmax, fabs(dd));
        dv[j] = dt;
        dvec[c0 + j] = dt;
#pragma unroll
        for (int i = j + 1; i < 16; ++i) p[j][i] = p[j][i] / dt;
#pragma unroll
        for (int c = j + 1; c < W; ++c)
#pragma unroll
            for (int i = c; i < 16; ++i) p[c][i] -= p[j][i] * dt * p[j][c];
        p[j][j] = (T)1;
    }
    // contribution block: packed column-major lower over the off rows W..r-1
    const int o = r - W;
    int64_t tb = 0;
#pragma unroll
    for (int b = 0; b < 16 - W; ++b) {
        if (b >= o) break;
#pragma unroll
        for (int aa = b; aa < 16 - W; ++aa) {
            if (aa >= o) break;
            T acc = (T)0;
#pragma unroll
            for (int k = 0; k < W; ++k) acc += p[k][W + aa] * dv[k] * p[k][W + b];
            inbox[a.push_pos[cb + tb + (aa - b)]] = acc;
        }
        tb += o - b;
    }
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (i < r) L[j * r + i] = p[j][i];
    *runmax_out = runmax;       // the caller folds it into the parent's running max
    return -1;     // tiny leaves are excluded from the child counts (separate launch)
}

template <typename T>
__device__ __forceinline__ int factor_tiny_lane(int J, const FactorArgs& a, T* __restrict__ lval, T* __restrict__ dvec,
                                                T* __restrict__ inbox, int* parent_out, double* runmax_out) {
    const int32_t* d32 = a.desc32 + (int64_t)J * 8;
    const int c0 = d32[0], w = d32[1], r = d32[2], parent = d32[3];
    const int64_t loff = a.desc64[(int64_t)J * 8], cb = a.desc64[(int64_t)J * 8 + 6];
    *parent_out = parent;
    switch (w) {
        case 1: return factor_tiny_w<T, 1>(J, c0, r, parent, loff, cb, a, lval, dvec, inbox, runmax_out);
        case 2: return factor_tiny_w<T, 2>(J, c0, r, parent, loff, cb, a, lval, dvec, inbox, runmax_out);
        case 3: return factor_tiny_w<T, 3>(J, c0, r, parent, loff, cb, a, lval, dvec, inbox, runmax_out);
        default: return factor_tiny_w<T, 4>(J, c0, r, parent, loff, cb, a, lval, dvec, inbox, runmax_out);
    }
}

// one warp-tier supernode task and its continuation chain up the tree
template <typename T>
__device__ __forceinline__ void factor_warp_chain(int J, const FactorArgs& a, T* __restrict__ lval,
                                                  T* __restrict__ dvec, T* __restrict__ inbox, T* sp, T* sDw,
                                                  int8_t* sSgw, uint64_t* bar, uint32_t& phase, T* sCol) {
    const int lane = threadIdx.x & 31;
    double carry_max = 0.0;      // the child's runmax when continuing (its atomic max may still be in flight)
    while (J >= 0) {
        if (a.trace && lane == 0) a.trace[6 * J] = a.trace[6 * J + 1] = gtimer();
        const Desc d = load_desc(a.desc32, a.desc64, J);
        const int c0 = d.c0, w = d.w, r = d.r, o = r - w;
        int needP = 0, tierP = -1;
        if (lane == 0 && d.parent >= 0) {
            needP = a.need[2 * d.parent + 1];
            tierP = a.desc32[(int64_t)d.parent * 8 + 6];
        }
        double runmax = lane == 0 ? fmax(__ldcg(a.maxd + J), carry_max) : 0.0;
        runmax = __shfl_sync(0xffffffffu, runmax, 0);
        if (lane < w) sSgw[lane] = a.sign[c0 + lane];
        if (lane + 32 < w) sSgw[lane + 32] = a.sign[c0 + lane + 32];
        T* L = lval + d.loff;
        const int psize = r * w;
        T* P = stage_panel(L, psize, sp, (int)a.smem_cap, bar, phase);
        if (a.trace && lane == 0) a.trace[6 * J + 2] = gtimer();
        if (P != L) warp_task_body(sp, L, true, d, c0, w, r, o, runmax, sDw, sSgw, a, dvec, inbox, J, sCol);
        else warp_task_body(L, L, false, d, c0, w, r, o, runmax, sDw, sSgw, a, dvec, inbox, J, sCol);
        __syncwarp();
        int cont = -1;
        if (lane == 0) {
            if (d.parent >= 0) {
                atomic_max_pos(a.maxd + d.parent, runmax);
                if (tierP == a.tier) {
                    if (needP == 1) cont = d.parent;        // sole same-tier child: no counter round trip
                    else if (atomic_add_acq_rel(a.count + d.parent, 1) == needP - 1) cont = d.parent;
                }
            }
            if (a.trace) a.trace[6 * J + 5] = gtimer();
        }
        // the factor is written back after the signal (the ancestors only read the inbox)
        if (P != L)
            for (int i = lane; i < psize; i += 32) L[i] = sp[i];
        J = __shfl_sync(0xffffffffu, cont, 0);
        carry_max = runmax;
        __syncwarp();
    }
}

// tiny leaves: one thread each (launched before the warp tier)
template <typename T>
__global__ void __launch_bounds__(TINY_T, TINY_MINB) factor_tiny_kernel(FactorArgs a, T* __restrict__ lval, T* __restrict__ dvec,
                                                          T* __restrict__ inbox) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int parent = -1;
    double runmax = 0.0;
    if (k < a.ntiny) factor_tiny_lane(a.tiny[k], a, lval, dvec, inbox, &parent, &runmax);
    // the parents' running max |d|: siblings are adjacent in the leaf list, so fold
    // each run of equal parents in the warp first (max is idempotent: overlapping
    // windows are harmless) and let the run's first lane issue the one atomic
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_down_sync(0xffffffffu, runmax, off);
        const int po = __shfl_down_sync(0xffffffffu, parent, off);
        if (lane + off < 32 && po == parent) runmax = fmax(runmax, o);
    }
    const int pprev = __shfl_up_sync(0xffffffffu, parent, 1);
    if (parent >= 0 && (lane == 0 || pprev != parent)) atomic_max_pos(a.maxd + parent, runmax);
}

template <typename T>
__global__ void __launch_bounds__(FW * 32) factor_kernel(FactorArgs a, T* __restrict__ lval, T* __restrict__ dvec,
                                                         T* __restrict__ inbox) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ T sD[FW][64];
    __shared__ __align__(16) T sColw[FW][64];
    __shared__ int8_t sSg[FW][64];
    __shared__ uint64_t bars[FW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T* sp = reinterpret_cast<T*>(smem_raw) + (int64_t)wid * a.smem_cap;
    if (lane == 0) mbar_init(&bars[wid], 1);
    __syncwarp();
    uint32_t phase = 0;
    // phase 2: the other seeds of the tier, by ticket
    for (;;) {
        int J = -1;
        if (lane == 0) {
            const int t = atomicAdd(a.ticket, 1);
            J = t < a.nstart ? a.start[t] : -1;
        }
        J = __shfl_sync(0xffffffffu, J, 0);
        if (J < 0) return;
        factor_warp_chain(J, a, lval, dvec, inbox, sp, sD[wid], sSg[wid], &bars[wid], phase, sColw[wid]);
    }
}

// CTA-tier dense panel LDL' (see factor_cta_kernel); forced inline so the
// panel pointer keeps its address space (shared -> LDS/STS) at each call site
//
// Blocked by 32 columns.  Per block k0: (a) warp 0 factors the nbk x nbk
// diagonal block with lane i holding row i in registers (warp-synchronous
// right-looking, shuffles, no barriers), publishing L11' and 1/d; (b) one thread
// per row below holds its nbk entries in registers and applies the same
// right-looking elimination against L11 (broadcast shared-memory reads);
// (c) rank-nbk update of the trailing columns.  Two or three barriers per block
// instead of one per column.
template <typename T, int NB>
__device__ __forceinline__ void cta_diag_block(T* Pk, int r, int k0, int nbk, const int8_t* sSg, T* sD,
                                               double& s_runmax, const FactorArgs& a, T* sLt, T* sInv, T* sCol) {
    const int lane = threadIdx.x & 31;
    double runmax = s_runmax;
    double ds_r = a.delta_s, dd_r = a.delta_d;
    asm volatile("" : "+d"(ds_r), "+d"(dd_r));
    T x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c)
        x[c] = (lane < nbk && c < nbk && c <= lane) ? Pk[c * r + k0 + lane] : (T)0;
    const unsigned pos = __ballot_sync(0xffffffffu, lane < nbk && sSg[k0 + lane] > 0);
    T d_mine = (T)0, inv_mine = (T)0;
    bool bump_mine = false;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        if (j < nbk) {
            // column j through shared memory (one store + broadcast loads instead of
            // NB - 1 shuffles: the shorter pivot chain of tools/micro/diag16.cu)
            T* col = sCol + (j & 1) * 32;
            col[lane] = x[j];
            __syncwarp();
            T cc[NB];
            load_col<T, NB>(cc, col);                  // one burst (common.cuh)
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
            const T lj = x[j] * inv;                 // l_ij (lanes i > j)
#pragma unroll
            for (int c = j + 1; c < NB; ++c) {
                const T acj = cc[c];                  // unscaled a_cj
                if (lane >= c) x[c] -= lj * acj;
            }
            x[j] = lane > j ? lj : (lane == j ? (T)1 : x[j]);
        }
    }
    if (lane < NB) {
        sInv[lane] = lane < nbk ? inv_mine : (T)0;
        if (lane < nbk) {
            sD[k0 + lane] = d_mine;
            if (d_mine == (T)0) set_error(a.err, CIPM_E_FACTOR);
        }
    }
    const unsigned nb_bumps = __popc(__ballot_sync(0xffffffffu, bump_mine));
    if (lane == 0 && nb_bumps) atomicAdd(a.bumps, (int)nb_bumps);
    int row = k0 + lane;
    asm volatile("" : "+r"(row));            // recompute the store addresses (no 32 live pointers)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
        if (lane < nbk && c < nbk && c <= lane) Pk[c * r + row] = x[c];
        if (lane < NB) sLt[c * NB + lane] = (c < lane && lane < nbk) ? x[c] : (T)0;   // Lt[j][i] = l_ij
    }
    __syncwarp();                           // every lane read s_runmax before lane 0 updates it
    if (lane == 0) s_runmax = runmax;
}

template <typename T, int NB>
__device__ __forceinline__ void cta_below_rows(T* Pk, int r, int i0, int nbk, const T* sLt, const T* sInv) {
#pragma unroll 1
    for (int i = i0 + threadIdx.x; i < r; i += blockDim.x) {
        T x[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) x[c] = c < nbk ? Pk[c * r + i] : (T)0;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const T xj = x[j];
#pragma unroll
            for (int c = j + 1; c < NB; ++c) x[c] -= xj * sLt[j * NB + c];
            x[j] = xj * sInv[j];
            asm volatile("" ::: "memory");      // L11 row loads per step (register budget)
        }
        int is = i;
        asm volatile("" : "+r"(is));         // recompute the store addresses (no 32 live pointers)
#pragma unroll
        for (int c = 0; c < NB; ++c)
            if (c < nbk) Pk[c * r + is] = x[c];
    }
}

//
// Blocked by 16 columns.  Per block k0: (a) warp 0 factors the nbk x nbk
// diagonal block with lane i holding row i in registers (warp-synchronous
// right-looking, shuffles, no barriers), publishing L11' and 1/d; (b) one thread
// per row below holds its nbk entries in registers and applies the same
// right-looking elimination against L11 (broadcast shared-memory reads);
// (c) rank-nbk update of the trailing columns.  Two or three barriers per block
// instead of one per column.
template <typename T>
__device__ __forceinline__ void cta_panel_ldl(T* P, int r, int w, int c0, const int8_t* sSg, T* sD, double& s_runmax,
                                              const FactorArgs& a, T* __restrict__ dvec, T* sLt, T* sInv, T* sCol) {
    // block width 16: a row of the block in registers, 2 CTAs / SM without spills
    constexpr int KB = 16;
    const int tid = threadIdx.x, wid = tid >> 5, nw = blockDim.x >> 5;
    for (int k0 = 0; k0 < w; k0 += KB) {
        const int nbk = min(KB, w - k0);
        T* Pk = P + k0 * r;               // column k0 of the panel
        if (wid == 0) {
            if (nbk <= 8) cta_diag_block<T, 8>(Pk, r, k0, nbk, sSg, sD, s_runmax, a, sLt, sInv, sCol);
            else cta_diag_block<T, KB>(Pk, r, k0, nbk, sSg, sD, s_runmax, a, sLt, sInv, sCol);
        }
        __syncthreads();
        // (b) rows below the diagonal block
        if (nbk <= 8) cta_below_rows<T, 8>(Pk, r, k0 + nbk, nbk, sLt, sInv);
        else cta_below_rows<T, KB>(Pk, r, k0 + nbk, nbk, sLt, sInv);
        __syncthreads();
        // (c) trailing columns c >= k0 + nbk, rows i >= c: A(i,c) -= sum_k l_ik d_k l_ck
        //     (only reached with a full block, nbk == KB)
        const int c1 = k0 + nbk;
        if (c1 < w) {
            // d_k l_ck for the trailing columns, into the (now free) L11' buffer
            for (int idx = tid; idx < (w - c1) * KB; idx += blockDim.x) {
                const int cc = idx / KB, k = idx - cc * KB;
                sLt[idx] = sD[k0 + k] * Pk[k * r + c1 + cc];
            }
            __syncthreads();
            for (int c = c1 + wid; c < w; c += nw) {
                const T* dl = sLt + (c - c1) * KB;
                T* Pc = P + c * r;
#pragma unroll 1
                for (int i = c + (tid & 31); i < r; i += 32) {
                    T acc = (T)0;
#pragma unroll 8
                    for (int k = 0; k < KB; ++k) acc += Pk[k * r + i] * dl[k];
                    Pc[i] -= acc;
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < w; j += blockDim.x) dvec[c0 + j] = sD[j];
}


// CTA-tier contribution block C = L_off D L_off' scattered to the ancestors'
// inboxes: entries (packed column-major lower) flattened over all threads, push
// positions loaded coalesced
template <typename T>
__device__ __forceinline__ void cta_push(const T* P, int r, int w, int o, int64_t base, const T* sD,
                                         const FactorArgs& a, T* __restrict__ inbox) {
    const int ne = o * (o + 1) / 2;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        const int64_t pos = __ldg(a.push_pos + base + e);
        int bb, aa;
        unpack_lower(e, o, bb, aa);
        const T* Pa = P + w + aa;
        const T* Pb = P + w + bb;
        T acc0 = (T)0, acc1 = (T)0;
        int k = 0;
        for (; k + 1 < w; k += 2) {
            acc0 += Pa[(int64_t)k * r] * (sD[k] * Pb[(int64_t)k * r]);
            acc1 += Pa[(int64_t)(k + 1) * r] * (sD[k + 1] * Pb[(int64_t)(k + 1) * r]);
        }
        if (k < w) acc0 += Pa[(int64_t)k * r] * (sD[k] * Pb[(int64_t)k * r]);
        inbox[pos] = acc0 + acc1;
    }
}

// CTA tier (one CTA per supernode): panels too large for one warp — the inbox
// gather is split by rows over the CTA's warps, the dense panel LDL' and the
// contribution block use all threads.  Same continuation protocol.
template <typename T>
__global__ void __launch_bounds__(256, 2) factor_cta_kernel(FactorArgs a, T* __restrict__ lval, T* __restrict__ dvec,
                                                         T* __restrict__ inbox) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sp = reinterpret_cast<T*>(smem_raw);
    __shared__ int s_J, s_needP, s_tierP, s_next;
    __shared__ double s_runmax, s_carry;
    __shared__ T sD[64];
    __shared__ __align__(16) T sLt[64 * 16];    // blocked LDL: L11' of a 16-column block / d_k l_ck
    __shared__ T sInv[16];
    __shared__ __align__(16) T sCol[64];
    __shared__ int8_t sSg[64];
    __shared__ int32_t s_d32[8];
    __shared__ int64_t s_d64[8];
    const int tid = threadIdx.x, nt = blockDim.x, wid = tid >> 5, nw = nt >> 5;
    if (tid == 0) s_next = -1;
    __syncthreads();
    for (;;) {
        if (tid == 0) {
            int J = s_next;
            if (J < 0) {
                const int t = atomicAdd(a.ticket, 1);
                J = t < a.nstart ? a.start[t] : -1;
                s_carry = 0.0;
            }
            s_J = J;
        }
        __syncthreads();
        const int J = s_J;
        if (J < 0) return;
        if (tid < 8) s_d32[tid] = a.desc32[(int64_t)J * 8 + tid];
        else if (tid < 16) s_d64[tid - 8] = a.desc64[(int64_t)J * 8 + tid - 8];
        if (tid == 0) {
            if (a.trace) a.trace[6 * J] = a.trace[6 * J + 1] = gtimer();
            s_runmax = fmax(__ldcg(a.maxd + J), s_carry);
        }
        __syncthreads();
        const int c0 = s_d32[0], w = s_d32[1], r = s_d32[2], parent = s_d32[3];
        const int o = r - w;
        const int64_t r0 = s_d64[7];
        if (tid == 0) {
            s_needP = parent >= 0 ? a.need[2 * parent + 1] : 0;
            s_tierP = parent >= 0 ? a.desc32[(int64_t)parent * 8 + 6] : -1;
        }
        T* L = lval + s_d64[0];
        const int64_t psize = (int64_t)r * w;
        const bool in_smem = psize <= a.smem_cap;
        if (in_smem)
            for (int64_t i0 = tid; i0 < psize; i0 += (int64_t)nt * 8) {   // 8 loads per thread in flight
                T v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = i0 + nt * u < psize ? L[i0 + nt * u] : (T)0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (i0 + nt * u < psize) sp[i0 + nt * u] = v[u];
            }
        if (tid < w) sSg[tid] = a.sign[c0 + tid];
        __syncthreads();
        if (a.trace && tid == 0) a.trace[6 * J + 2] = gtimer();
        // 1. inbox gather, rows split over the warps (targets are unique per row)
        {
            const int rs = (int)((int64_t)r * wid / nw), re = (int)((int64_t)r * (wid + 1) / nw);
            if (re > rs) {
                if (in_smem) warp_gather_sub(sp, a.inbox_tgt, inbox, a.irow_ptr[r0 + rs], a.irow_ptr[r0 + re]);
                else warp_gather_sub(L, a.inbox_tgt, inbox, a.irow_ptr[r0 + rs], a.irow_ptr[r0 + re]);
            }
        }
        __syncthreads();
        if (a.trace && tid == 0) a.trace[6 * J + 3] = gtimer();
        // 2. dense LDL' of the panel: blocked by 16 columns (cta_panel_ldl)
        if (in_smem) cta_panel_ldl(sp, r, w, c0, sSg, sD, s_runmax, a, dvec, sLt, sInv, sCol);
        else cta_panel_ldl(L, r, w, c0, sSg, sD, s_runmax, a, dvec, sLt, sInv, sCol);
        if (a.trace && tid == 0) a.trace[6 * J + 4] = gtimer();
        // 3. push C_J = L_off D L_off' (the factor is written back after the signal:
        //    the ancestors only read the inbox, so the release does not wait for it)
        if (o > 0) {
            if (in_smem) cta_push(sp, r, w, o, s_d64[6], sD, a, inbox);
            else cta_push(L, r, w, o, s_d64[6], sD, a, inbox);
        }
        __syncthreads();
        if (tid == 0) {
            int cont = -1;
            if (parent >= 0) {
                atomic_max_pos(a.maxd + parent, s_runmax);
                if (s_tierP == a.tier) {
                    if (s_needP == 1) cont = parent;        // sole same-tier child: no counter round trip
                    else if (atomic_add_acq_rel(a.count + parent, 1) == s_needP - 1) cont = parent;
                }
            }
            if (a.trace) a.trace[6 * J + 5] = gtimer();
            s_next = cont;
            s_carry = s_runmax;
        }
        if (in_smem)
            for (int64_t i = tid; i < psize; i += nt) L[i] = sp[i];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// solve form: after the factorisation, every warp / CTA-tier panel
// P = [L11; L21] (r x w, column-major, unit lower L11) is rewritten in place as
// M = [L11^-1; L21 L11^-1] (strict upper triangle of the top block zeroed), so
// each supernode of the triangular sweeps is one dense GEMV with independent
// dot products: forward [y_J; push] = M b_J, backward x_J = M' [y_J / D; -x_off]
// (the same L, D solves as ldl.py:91-104).  One warp per supernode, all
// supernodes in parallel, off the factorisation's critical path (tiny leaves do
// the same in registers inside factor_tiny_kernel; the dense tail keeps its own
// blocked inverses).
//   (i)  Linv, lanes over columns j (j + 32): x_i = -sum_{k<i} L[i][k] x_k with
//        x_j = 1 and x_k = 0 for k < j — the same trip count on every lane;
//   (ii) rows below, lanes over rows: m_i[j] = sum_{k>=j} l_i[k] Linv[k][j],
//        j ascending, in place.
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ bool solve_form_body(T* P, int r, int w, T* inv, double tau) {
    const int lane = threadIdx.x & 31;
    // (i) Linv row-major in inv[i * w + j] (lane j writes column j: conflict-free)
    for (int i = 0; i < w; ++i) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            if (j < w) {
                T acc = (T)0;
                for (int k = j; k < i; ++k) acc += P[(int64_t)k * r + i] * inv[k * w + j];
                inv[i * w + j] = i == j ? (T)1 : (i < j ? (T)0 : -acc);
            }
        }
        __syncwarp();
    }
    // growth test: the explicit inverse is used only when max |Linv| <= tau (an
    // inverse-based solve loses at most that factor against substitution); larger
    // panels keep L and the sweeps use substitution for them
    double g = 0.0;
    for (int e = lane; e < w * w; e += 32) g = fmax(g, fabs((double)inv[e]));
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (!(g <= tau)) return false;
    // (ii) rows below
    for (int i = w + lane; i < r; i += 32)
        for (int j = 0; j < w; ++j) {
            T acc = P[(int64_t)j * r + i];
#pragma unroll 4
            for (int k = j + 1; k < w; ++k) acc += P[(int64_t)k * r + i] * inv[k * w + j];
            P[(int64_t)j * r + i] = acc;
        }
    // top block <- Linv (column-major, zeros above the diagonal)
    for (int e = lane; e < w * w; e += 32) {
        const int j = e / w, i = e - j * w;
        P[(int64_t)j * r + i] = inv[i * w + j];
    }
    __syncwarp();
    return true;
}

constexpr int SFW = 4;   // warps per solve-form CTA

template <typename T>
__global__ void __launch_bounds__(SFW * 32) solve_form_kernel(const int32_t* __restrict__ list, int32_t n,
                                                              const int32_t* __restrict__ d32,
                                                              const int64_t* __restrict__ d64, T* lval, int slice,
                                                              int inv_cap, double tau, int8_t* sf) {
    extern __shared__ __align__(16) unsigned char sraw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T* inv = reinterpret_cast<T*>(sraw) + (int64_t)wid * (inv_cap + slice);
    T* sp = inv + inv_cap;
    for (int64_t t = blockIdx.x * (int64_t)SFW + wid; t < n; t += (int64_t)gridDim.x * SFW) {
        const int J = list[t];
        const int w = __ldg(d32 + (int64_t)J * 8 + 1), r = __ldg(d32 + (int64_t)J * 8 + 2);
        T* L = lval + __ldg(d64 + (int64_t)J * 8);
        const int psize = r * w;
        if (w < 1) continue;
        bool ok;
        if (psize <= slice) {
            for (int e = lane; e < psize; e += 32) sp[e] = L[e];
            __syncwarp();
            ok = solve_form_body(sp, r, w, inv, tau);
            if (ok)
                for (int e = lane; e < psize; e += 32) L[e] = sp[e];
        } else {
            ok = solve_form_body(L, r, w, inv, tau);
        }
        if (lane == 0) sf[J] = ok ? 1 : 0;
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// triangular solves
// ---------------------------------------------------------------------------

struct SolveArgs {
    int32_t nstart;      // forward seeds
    const int32_t* start;
    int32_t n_main;      // backward: tickets over order[0 .. n_main) reversed
    const int32_t* order;
    int32_t ntiny;       // tiny leaves (one lane each)
    const int32_t* tiny;
    int32_t* ticket_tiny;
    const int32_t* bwd_done;   // forward tiny-leaf path: unused; backward: parents' done flags
    const int32_t* desc32;
    const int64_t* desc64;
    const int32_t* need;
    int64_t dim;
    int64_t nv;          // vector inbox length per right-hand side
    const int32_t* sn_rows;
    const int32_t* vpush_pos;
    const uint8_t* vin_col;
    int32_t* count;      // forward: children done; backward: done flags
    int32_t* ticket;
    int act0, act1;      // active right-hand sides
    int64_t* trace;      // optional per-task timeline (cipm_trace)
    int slice;           // per-warp shared-memory panel slice (elements)
    const double* rstate;   // refinement state: skip right-hand sides that have converged
    const int8_t* sf;       // per supernode: 1 = panel in solve form (M), 0 = plain L (solve_form_kernel)
    const int4* tdesc;      // tiny leaves, compact: {c0, loff, cvo, w | r << 8}
    const int32_t* trptr;   // tiny leaves: offset of the row list in sn_rows
};

// warp-cooperative sums of the vector inbox of one supernode's columns (entries
// [lo, hi), grouped by column, local column ids in vin_col), for NQ right-hand
// sides at once: cs[q][j] = sum of column j's entries of RHS q.  The entries of
// every RHS (32 * CH per round trip) are loaded before any is reduced, and the
// segmented scan shares its column-id shuffles across the RHS.
template <typename T, int NQ>
__device__ __forceinline__ void vgather_q(T* const (&vq)[NQ], const uint8_t* __restrict__ vin_col, int64_t lo,
                                          int64_t hi, int w, T (*cs)[64]) {
    constexpr int CH = 8 / NQ;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
        for (int j = lane; j < w; j += 32) cs[q][j] = (T)0;
    __syncwarp();
    for (int64_t base = lo; base < hi; base += 32 * CH) {
        T v[NQ][CH];
        int col[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u) {             // one round trip for every RHS
            const int64_t e = base + 32 * u + lane;
            const bool ok = e < hi;
#pragma unroll
            for (int q = 0; q < NQ; ++q) v[q][u] = ok ? __ldcg(vq[q] + e) : (T)0;
            col[u] = ok ? (int)__ldg(vin_col + e) : -(lane + 2);
        }
#pragma unroll
        for (int u = 0; u < CH; ++u) {
            if (base + 32 * u >= hi) break;
            const int cu = col[u];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int cp = __shfl_up_sync(0xffffffffu, cu, off);
                const bool take = lane >= off && cp == cu;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const T vp = __shfl_up_sync(0xffffffffu, v[q][u], off);
                    if (take) v[q][u] += vp;
                }
            }
            const int cn = __shfl_down_sync(0xffffffffu, cu, 1);
            if (cu >= 0 && (lane == 31 || cn != cu)) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) cs[q][cu] += v[q][u];
            }
            __syncwarp();
        }
    }
    __syncwarp();
}

// forward task, compute part: triangle and off-row push for NQ right-hand sides
// together (each L element is read once for all of them).  Forced inline so L
// keeps its address space (staged panel -> LDS).
template <typename T, int NQ>
__device__ __forceinline__ void fwd_compute_tri(const T* L, const SolveArgs& a, const Desc& d, T* const (&xq)[NQ],
                                            T* const (&vq)[NQ], const T (&xa)[NQ], const T (&xb)[NQ],
                                            T (*cs)[64], int J, const int64_t (&pos_pf)[2]) {
    const int lane = threadIdx.x & 31;
    const int c0 = d.c0, w = d.w, r = d.r;
    T x0[NQ], x1[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        x0[q] = lane < w ? xa[q] - cs[q][lane] : (T)0;
        x1[q] = lane + 32 < w ? xb[q] - cs[q][lane + 32] : (T)0;
    }
    constexpr int KB = 8 / NQ;                  // columns whose loads are issued together
    for (int j0 = 0; j0 < w; j0 += KB) {
        T l0[KB], l1[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {          // issue the block's loads before the dependent chain
            const int j = j0 + k;
            l0[k] = (j < w && lane > j && lane < w) ? L[j * r + lane] : (T)0;
            l1[k] = (j < w && lane + 32 > j && lane + 32 < w) ? L[j * r + lane + 32] : (T)0;
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int j = j0 + k;
            if (j >= w) break;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const T xj = __shfl_sync(0xffffffffu, j < 32 ? x0[q] : x1[q], j & 31);
                x0[q] -= l0[k] * xj;
                x1[q] -= l1[k] * xj;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        if (lane < w) xq[q][c0 + lane] = x0[q];
        if (lane + 32 < w) xq[q][c0 + lane + 32] = x1[q];
    }
    if (a.trace && lane == 0) a.trace[6 * J + 3] = gtimer();
    for (int i0 = w; i0 < r; i0 += 32) {
        const int i = i0 + lane;
        const bool ok = i < r;
        const int ii = ok ? i : r - 1;
        const int pass = (i0 - w) >> 5;
        const int64_t pos = pass < 2 ? pos_pf[pass] : (ok ? a.vpush_pos[d.cvo + i - w] : 0);
        T acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = (T)0;
#pragma unroll 8
        for (int k = 0; k < w; ++k) {
            const T lk = L[k * r + ii];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] += lk * __shfl_sync(0xffffffffu, k < 32 ? x0[q] : x1[q], k & 31);
        }
        if (ok) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) vq[q][pos] = acc[q];
        }
    }
    if (a.trace && lane == 0) a.trace[6 * J + 4] = gtimer();
}

// forward task, compute part, for NQ right-hand sides together: the panel is in
// solve form (M = [L11^-1; L21 L11^-1]), so y_J = M_top b_J and the off-row push
// M_off b_J are one GEMV with independent row dot products (lanes over rows; b_J
// broadcast from shared memory).  Forced inline so L keeps its address space
// (staged panel -> LDS).
template <typename T, int NQ>
__device__ __forceinline__ void fwd_compute_sf(const T* L, const SolveArgs& a, const Desc& d, T* const (&xq)[NQ],
                                            T* const (&vq)[NQ], const T (&xa)[NQ], const T (&xb)[NQ],
                                            T (*cs)[64], int J, const int64_t (&pos_pf)[2]) {
    const int lane = threadIdx.x & 31;
    const int c0 = d.c0, w = d.w, r = d.r;
    // b_J = own values - inbox sums, into the shared column buffer
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        if (lane < w) cs[q][lane] = xa[q] - cs[q][lane];
        if (lane + 32 < w) cs[q][lane + 32] = xb[q] - cs[q][lane + 32];
    }
    __syncwarp();
    // top rows: y_J (M_top is unit lower: the diagonal term is b_i itself)
    for (int i0 = 0; i0 < w; i0 += 32) {
        const int i = i0 + lane;
        const int ii = i < w ? i : w - 1;
        T acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = cs[q][ii];
#pragma unroll 8
        for (int k = 0; k < ii; ++k) {
            const T mk = L[k * r + ii];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] += mk * cs[q][k];
        }
        if (i < w) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) xq[q][c0 + i] = acc[q];
        }
    }
    if (a.trace && lane == 0) a.trace[6 * J + 3] = gtimer();
    // off rows: push M_off b_J into the ancestors' vector inboxes
    for (int i0 = w; i0 < r; i0 += 32) {
        const int i = i0 + lane;
        const bool ok = i < r;
        const int ii = ok ? i : r - 1;
        const int pass = (i0 - w) >> 5;
        const int64_t pos = pass < 2 ? pos_pf[pass] : (ok ? a.vpush_pos[d.cvo + i - w] : 0);
        T acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = (T)0;
#pragma unroll 8
        for (int k = 0; k < w; ++k) {
            const T mk = L[k * r + ii];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] += mk * cs[q][k];
        }
        if (ok) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) vq[q][pos] = acc[q];
        }
    }
    if (a.trace && lane == 0) a.trace[6 * J + 4] = gtimer();
}

// backward task body for NQ right-hand sides: own values (xa/xb, loaded before
// the parent wait) D-solved, the ancestors' values at the off rows gathered for
// every RHS in one round trip (64 rows at a time), then the transposed triangle.
template <typename T, int NQ>
__device__ __forceinline__ void bwd_body_tri(const T* L, const SolveArgs& a, int c0, int w, int r, int o,
                                         const int32_t* rowsJ, T* const (&xq)[NQ], T (*xo)[64],
                                         const int (&rows_pf)[2], const T (&d_pf)[2], const T (&xa)[NQ],
                                         const T (&xb)[NQ]) {
    const int lane = threadIdx.x & 31;
    const T* L0 = L + lane * r;
    const T* L1 = L + (lane + 32) * r;
    const bool o0 = lane < w, o1 = lane + 32 < w;
    T x0[NQ], x1[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        x0[q] = o0 ? xa[q] / d_pf[0] : (T)0;      // D solve (ldl.py:101-102)
        x1[q] = o1 ? xb[q] / d_pf[1] : (T)0;
    }
    for (int i0 = 0; i0 < o; i0 += 64) {
        const int n = min(64, o - i0);
        const int ra = i0 == 0 ? rows_pf[0] : (lane < n ? rowsJ[i0 + lane] : 0);
        const int rb = i0 == 0 ? rows_pf[1] : (lane + 32 < n ? rowsJ[i0 + lane + 32] : 0);
        T va[NQ], vb[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            va[q] = lane < n ? __ldcg(xq[q] + ra) : (T)0;
            vb[q] = lane + 32 < n ? __ldcg(xq[q] + rb) : (T)0;
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            xo[q][lane] = va[q];
            xo[q][lane + 32] = vb[q];
        }
        __syncwarp();
#pragma unroll 8
        for (int k = 0; k < n; ++k) {
            const T la = o0 ? L0[w + i0 + k] : (T)0;
            const T lb = o1 ? L1[w + i0 + k] : (T)0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const T xi = xo[q][k];
                x0[q] -= la * xi;
                x1[q] -= lb * xi;
            }
        }
        __syncwarp();
    }
    constexpr int KB = 8 / NQ;
    for (int j1 = w - 1; j1 >= 0; j1 -= KB) {
        T l0[KB], l1[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {          // loads first, then the dependent chain
            const int j = j1 - k;
            l0[k] = (j >= 0 && lane < j) ? L0[j] : (T)0;
            l1[k] = (j >= 0 && lane + 32 < j) ? L1[j] : (T)0;
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int j = j1 - k;
            if (j < 0) break;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const T xj = __shfl_sync(0xffffffffu, j < 32 ? x0[q] : x1[q], j & 31);
                x0[q] -= l0[k] * xj;
                x1[q] -= l1[k] * xj;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        if (o0) xq[q][c0 + lane] = x0[q];
        if (o1) xq[q][c0 + lane + 32] = x1[q];
    }
}

// backward task body for NQ right-hand sides, panel in solve form:
// x_J = M' v with v = [y_J / D; -x_off] — lane j owns columns j and j + 32 and
// accumulates independent products over the rows (no dependent chain).  Own
// values (xa / xb) were loaded before the parent wait; the ancestors' values at
// the off rows are gathered for every RHS in one round trip (64 rows at a time).
template <typename T, int NQ>
__device__ __forceinline__ void bwd_body_sf(const T* L, const SolveArgs& a, int c0, int w, int r, int o,
                                         const int32_t* rowsJ, T* const (&xq)[NQ], T (*xo)[64],
                                         const int (&rows_pf)[2], const T (&d_pf)[2], const T (&xa)[NQ],
                                         const T (&xb)[NQ]) {
    const int lane = threadIdx.x & 31;
    const T* L0 = L + lane * r;
    const T* L1 = L + (lane + 32) * r;
    const bool o0 = lane < w, o1 = lane + 32 < w;
    T x0[NQ], x1[NQ];
    // top rows: v = y_J / D (ldl.py:101-102) through the shared buffer; M_top' is unit upper
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const T v0 = o0 ? xa[q] / d_pf[0] : (T)0;
        const T v1 = o1 ? xb[q] / d_pf[1] : (T)0;
        x0[q] = v0;
        x1[q] = v1;
        xo[q][lane] = v0;
        xo[q][lane + 32] = v1;
    }
    __syncwarp();
    {
        const int j0 = o0 ? lane : w, j1 = o1 ? lane + 32 : w;
#pragma unroll 4
        for (int i = j0 + 1; i < w; ++i) {
            const T m = L0[i];
#pragma unroll
            for (int q = 0; q < NQ; ++q) x0[q] += m * xo[q][i];
        }
#pragma unroll 4
        for (int i = j1 + 1; i < w; ++i) {
            const T m = L1[i];
#pragma unroll
            for (int q = 0; q < NQ; ++q) x1[q] += m * xo[q][i];
        }
    }
    __syncwarp();
    for (int i0 = 0; i0 < o; i0 += 64) {
        const int n = min(64, o - i0);
        const int ra = i0 == 0 ? rows_pf[0] : (lane < n ? rowsJ[i0 + lane] : 0);
        const int rb = i0 == 0 ? rows_pf[1] : (lane + 32 < n ? rowsJ[i0 + lane + 32] : 0);
        T va[NQ], vb[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            va[q] = lane < n ? __ldcg(xq[q] + ra) : (T)0;
            vb[q] = lane + 32 < n ? __ldcg(xq[q] + rb) : (T)0;
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            xo[q][lane] = va[q];
            xo[q][lane + 32] = vb[q];
        }
        __syncwarp();
#pragma unroll 8
        for (int k = 0; k < n; ++k) {
            const T la = o0 ? L0[w + i0 + k] : (T)0;
            const T lb = o1 ? L1[w + i0 + k] : (T)0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const T xi = xo[q][k];
                x0[q] -= la * xi;
                x1[q] -= lb * xi;
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        if (o0) xq[q][c0 + lane] = x0[q];
        if (o1) xq[q][c0 + lane + 32] = x1[q];
    }
}

constexpr int SW = 8;   // warps per solve CTA

// forward sweep L y = b: warp per supernode, columns in registers (lane owns
// columns lane and lane+32; non-tail supernodes are narrower than 64), panel
// staged in shared memory by one bulk copy, continuation to the parent
// tiny leaf, forward: x_J = L11^-1 b_J (no inbox below a leaf), push L_off x_J
template <typename T, int W>
__device__ __forceinline__ int fwd_tiny_w(const int4 td, const SolveArgs& a, const T* __restrict__ lval,
                                          T* x, T* vin) {
    // compact tiny-leaf descriptor {c0, loff, cvo, w | r << 8} (16 bytes instead of 96)
    const int c0 = td.x, r = (td.w >> 8) & 0xff, parent = -1;
    const int64_t loff = (uint32_t)td.y, cvo = (uint32_t)td.z;
    const T* L = lval + loff;
    T p[W][16];
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
        for (int i = 0; i < 16; ++i) p[j][i] = (i < r && i > j) ? L[j * r + i] : (T)0;
    const int needP = 0;
    (void)parent;
    T xv2[2][W];                  // both right-hand sides loaded before any store
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const bool act = q == 0 ? a.act0 : a.act1;
#pragma unroll
        for (int j = 0; j < W; ++j) xv2[q][j] = act ? x[(int64_t)q * a.dim + c0 + j] : (T)0;
    }
    int pp[16];
#pragma unroll
    for (int i = W; i < 16; ++i) pp[i] = i < r ? a.vpush_pos[cvo + i - W] : 0;
    for (int q = 0; q < 2; ++q) {
        if (!(q == 0 ? a.act0 : a.act1)) continue;
        T* xJ = x + (int64_t)q * a.dim + c0;
        T (&xv)[W] = xv2[q];
#pragma unroll
        for (int j = 0; j < W; ++j)
#pragma unroll
            for (int i = j + 1; i < W; ++i) xv[i] -= p[j][i] * xv[j];
#pragma unroll
        for (int j = 0; j < W; ++j) xJ[j] = xv[j];
        T* vq = vin + (int64_t)q * a.nv;
#pragma unroll
        for (int i = W; i < 16; ++i) {
            if (i >= r) break;
            T acc = (T)0;
#pragma unroll
            for (int k = 0; k < W; ++k) acc += p[k][i] * xv[k];
            vq[pp[i]] = acc;
        }
    }
    (void)needP;
    return -1;     // tiny leaves are excluded from the child counts (separate launch)
}

template <typename T>
__device__ __forceinline__ int fwd_tiny_lane(int64_t k, const SolveArgs& a, const T* __restrict__ lval, T* x, T* vin) {
    const int4 td = __ldg(a.tdesc + k);
    switch (td.w & 0xff) {
        case 1: return fwd_tiny_w<T, 1>(td, a, lval, x, vin);
        case 2: return fwd_tiny_w<T, 2>(td, a, lval, x, vin);
        case 3: return fwd_tiny_w<T, 3>(td, a, lval, x, vin);
        default: return fwd_tiny_w<T, 4>(td, a, lval, x, vin);
    }
}

// one forward task and its continuation chain
template <typename T, int NQ>
__device__ __forceinline__ void fwd_chain(int J, const SolveArgs& a, const T* __restrict__ lval, T* const (&xq)[NQ],
                                          T* const (&vq)[NQ], T* slice, T (*cs)[64], uint64_t* bar,
                                          uint32_t& phase) {
    const int lane = threadIdx.x & 31;
    bool have_dn = false;
    Desc dn;                       // descriptor of the parent, prefetched for a continuation
    while (J >= 0) {
        if (a.trace && lane == 0) a.trace[6 * J] = a.trace[6 * J + 1] = gtimer();
        const Desc d = have_dn ? dn : load_desc(a.desc32, a.desc64, J);
        const int w = d.w, r = d.r;
        const T* Lg = lval + d.loff;
        // 1. issue the panel's TMA bulk copy; it lands while the inputs are gathered
        const uint32_t bytes = ((uint32_t)(r * w) * (uint32_t)sizeof(T) + 15u) & ~15u;
        const bool staged = bytes <= (uint32_t)a.slice * (uint32_t)sizeof(T);
        if (staged) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) bulk_g2s(slice, Lg, bytes, bar);
        }
        const int needP = (lane == 0 && d.parent >= 0) ? a.need[2 * d.parent] : 0;
        const bool sfJ = __ldg(a.sf + J) != 0;
        // parent descriptor: raw loads now, shuffled after the compute (off the critical path)
        const int Jn = d.parent >= 0 ? d.parent : J;
        const int pv32 = lane < 8 ? __ldg(a.desc32 + (int64_t)Jn * 8 + lane) : 0;
        const int64_t pv64 = (lane >= 8 && lane < 16) ? __ldg(a.desc64 + (int64_t)Jn * 8 + (lane - 8)) : 0;
        // push positions of the first 64 off rows (static: prefetched with the inputs)
        int64_t pos_pf[2];
        pos_pf[0] = lane < r - w ? __ldg(a.vpush_pos + d.cvo + lane) : 0;
        pos_pf[1] = lane + 32 < r - w ? __ldg(a.vpush_pos + d.cvo + 32 + lane) : 0;
        // 2. own right-hand-side values and the vector inbox of the supernode's columns
        T xa[NQ], xb[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            xa[q] = lane < w ? xq[q][d.c0 + lane] : (T)0;
            xb[q] = lane + 32 < w ? xq[q][d.c0 + lane + 32] : (T)0;
        }
        vgather_q<T, NQ>(vq, a.vin_col, d.vlo, d.vhi, w, cs);
        if (a.trace && lane == 0) a.trace[6 * J + 2] = gtimer();
        // 3. GEMV (solve form) or triangle + push, from shared memory when staged
        if (staged) {
            mbar_wait(bar, phase);
            phase ^= 1u;
            if (sfJ) fwd_compute_sf<T, NQ>(slice, a, d, xq, vq, xa, xb, cs, J, pos_pf);
            else fwd_compute_tri<T, NQ>(slice, a, d, xq, vq, xa, xb, cs, J, pos_pf);
        } else {
            if (sfJ) fwd_compute_sf<T, NQ>(Lg, a, d, xq, vq, xa, xb, cs, J, pos_pf);
            else fwd_compute_tri<T, NQ>(Lg, a, d, xq, vq, xa, xb, cs, J, pos_pf);
        }
        dn = desc_from_regs(pv32, pv64);
        __syncwarp();
        int cont = -1;
        if (lane == 0) {
            if (d.parent >= 0) {
                // a sole (non-tiny) child continues without the counter round trip: this
                // warp's writes are ordered before its own later reads, and before other
                // tasks' reads by the release of the chain's next counted increment
                if (needP == 1) cont = d.parent;
                else if (atomic_add_acq_rel(a.count + d.parent, 1) == needP - 1) cont = d.parent;
            }
            if (a.trace) a.trace[6 * J + 5] = gtimer();
        }
        J = __shfl_sync(0xffffffffu, cont, 0);
        have_dn = true;
        __syncwarp();
    }
}

// after the tiny leaves: fold their vector-inbox entries into the right-hand side,
// one thread per receiving column, entries in ascending order (deterministic);
// the persistent sweep then gathers only the entries of non-tiny children
template <typename T>
__global__ void __launch_bounds__(256) tiny_fold_kernel(SolveArgs a0, const int32_t* __restrict__ cols, int64_t ncols,
                                                        const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                                                        T* x, const T* __restrict__ vin) {
    SolveArgs a = a0;
    resolve_act(a.rstate, a.act0, a.act1);
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ncols) return;
    const int32_t j = cols[k];
    const int64_t e0 = lo[j], e1 = hi[j];
    for (int q = 0; q < 2; ++q) {
        if (!(q == 0 ? a.act0 : a.act1)) continue;
        const T* vq = vin + (int64_t)q * a.nv;
        T s = (T)0;
        for (int64_t e = e0; e < e1; ++e) s += vq[e];
        x[(int64_t)q * a.dim + j] -= s;
    }
}

// tiny leaves, forward: one thread each (launched before the persistent sweep)
template <typename T>
__global__ void __launch_bounds__(TINY_T, TINY_MINB) fwd_tiny_kernel(SolveArgs a0, const T* __restrict__ lval, T* x, T* vin) {
    SolveArgs a = a0;
    resolve_act(a.rstate, a.act0, a.act1);
    if (!a.act0 && !a.act1) return;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < a.ntiny) fwd_tiny_lane(k, a, lval, x, vin);
}

template <typename T>
__global__ void __launch_bounds__(SW * 32, 3) forward_kernel(SolveArgs a0, const T* __restrict__ lval, T* x, T* vin) {
    SolveArgs a = a0;
    resolve_act(a.rstate, a.act0, a.act1);
    if (!a.act0 && !a.act1) return;
    extern __shared__ __align__(16) unsigned char sraw[];
    __shared__ T colsum[SW][2][64];
    __shared__ uint64_t bars[SW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T* slice = reinterpret_cast<T*>(sraw) + (int64_t)wid * a.slice;
    if (lane == 0) mbar_init(&bars[wid], 1);
    __syncwarp();
    uint32_t phase = 0;
    // phase 2: remaining seeds by ticket
    for (;;) {
        int J = -1;
        if (lane == 0) {
            const int t = atomicAdd(a.ticket, 1);
            J = t < a.nstart ? a.start[t] : -1;
        }
        J = __shfl_sync(0xffffffffu, J, 0);
        if (J < 0) return;
        if (a.act0 && a.act1) {
            T* const xq[2] = {x, x + a.dim};
            T* const vq[2] = {vin, vin + a.nv};
            fwd_chain<T, 2>(J, a, lval, xq, vq, slice, colsum[wid], &bars[wid], phase);
        } else {
            const int64_t q = a.act0 ? 0 : 1;
            T* const xq[1] = {x + q * a.dim};
            T* const vq[1] = {vin + q * a.nv};
            fwd_chain<T, 1>(J, a, lval, xq, vq, slice, colsum[wid], &bars[wid], phase);
        }
    }
}

// backward sweep L' x = D^-1 y: warp per supernode, reverse topological order
// tiny leaves, backward: one thread each, launched after the persistent sweep
template <typename T, int W>
__device__ __forceinline__ void bwd_tiny_w(const int4 td, int64_t rptr, const SolveArgs& a, const T* __restrict__ lval,
                                           const T* __restrict__ dvec, T* x);

template <typename T>
__global__ void __launch_bounds__(TINY_T, TINY_MINB) bwd_tiny_kernel(SolveArgs a0, const T* __restrict__ lval,
                                                       const T* __restrict__ dvec, T* x) {
    SolveArgs a = a0;
    resolve_act(a.rstate, a.act0, a.act1);
    if (!a.act0 && !a.act1) return;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= a.ntiny) return;
    const int4 td = __ldg(a.tdesc + k);
    const int64_t rptr = (uint32_t)__ldg(a.trptr + k);
    switch (td.w & 0xff) {
        case 1: bwd_tiny_w<T, 1>(td, rptr, a, lval, dvec, x); break;
        case 2: bwd_tiny_w<T, 2>(td, rptr, a, lval, dvec, x); break;
        case 3: bwd_tiny_w<T, 3>(td, rptr, a, lval, dvec, x); break;
        default: bwd_tiny_w<T, 4>(td, rptr, a, lval, dvec, x); break;
    }
}

// tiny leaf, backward: x_J = L11^-T (D^-1 x_J - L_off' x_off) once the parent is final
template <typename T, int W>
__device__ __forceinline__ void bwd_tiny_w(const int4 td, int64_t rptr, const SolveArgs& a, const T* __restrict__ lval,
                                           const T* __restrict__ dvec, T* x) {
    const int c0 = td.x, r = (td.w >> 8) & 0xff, parent = -1;
    const int64_t loff = (uint32_t)td.y;
    const T* L = lval + loff;
    T p[W][16];
#pragma unroll
    for (int j = 0; j < W; ++j)
#pragma unroll
        for (int i = 0; i < 16; ++i) p[j][i] = (i < r && i > j) ? L[j * r + i] : (T)0;
    int rows[16];
#pragma unroll
    for (int i = W; i < 16; ++i) rows[i] = i < r ? a.sn_rows[rptr + i] : 0;
    T dinv[W];
#pragma unroll
    for (int j = 0; j < W; ++j) dinv[j] = dvec[c0 + j];
    (void)parent;      // the persistent backward sweep finished before this launch
    // both right-hand sides' loads are issued before any store (the stores of one
    // RHS would otherwise order the other's gathers behind them)
    T xr[2][W], xo[2][16];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const bool act = q == 0 ? a.act0 : a.act1;
        const T* xv = x + (int64_t)q * a.dim;
#pragma unroll
        for (int j = 0; j < W; ++j) xr[q][j] = act ? xv[c0 + j] : (T)0;
#pragma unroll
        for (int i = W; i < 16; ++i) xo[q][i] = (act && i < r) ? __ldcg(xv + rows[i]) : (T)0;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (!(q == 0 ? a.act0 : a.act1)) continue;
#pragma unroll
        for (int j = 0; j < W; ++j) xr[q][j] = xr[q][j] / dinv[j];      // D solve (ldl.py:101-102)
#pragma unroll
        for (int i = W; i < 16; ++i) {
            if (i >= r) break;
#pragma unroll
            for (int j = 0; j < W; ++j) xr[q][j] -= p[j][i] * xo[q][i];
        }
#pragma unroll
        for (int j = W - 1; j >= 0; --j)
#pragma unroll
            for (int i = j + 1; i < W; ++i) xr[q][j] -= p[j][i] * xr[q][i];
        T* xv = x + (int64_t)q * a.dim;
#pragma unroll
        for (int j = 0; j < W; ++j) xv[c0 + j] = xr[q][j];
    }
}

template <typename T>
__global__ void __launch_bounds__(SW * 32, 3) backward_kernel(SolveArgs a0, const T* __restrict__ lval,
                                                           const T* __restrict__ dvec, T* x) {
    SolveArgs a = a0;
    resolve_act(a.rstate, a.act0, a.act1);
    if (!a.act0 && !a.act1) return;
    extern __shared__ __align__(16) unsigned char sraw[];
    __shared__ T xs[SW][2][64];
    __shared__ uint64_t bars[SW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T* slice = reinterpret_cast<T*>(sraw) + (int64_t)wid * a.slice;
    if (lane == 0) mbar_init(&bars[wid], 1);
    __syncwarp();
    uint32_t phase = 0;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(a.ticket, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= a.n_main) return;
        const int J = a.order[a.n_main - 1 - t];     // a.order = bwd_order here
        const Desc d = load_desc(a.desc32, a.desc64, J);
        const int c0 = d.c0, w = d.w, r = d.r;
        const int o = r - w;
        const int32_t* rowsJ = a.sn_rows + d.rptr + w;
        const T* Lg = lval + d.loff;
        // the panel is static: start its bulk copy before waiting for the parent
        const uint32_t bytes = ((uint32_t)(r * w) * (uint32_t)sizeof(T) + 15u) & ~15u;
        const bool staged = bytes <= (uint32_t)a.slice * (uint32_t)sizeof(T);
        if (staged) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) bulk_g2s(slice, Lg, bytes, &bars[wid]);
        }
        // static inputs fetched before waiting for the parent
        const bool sfJ = __ldg(a.sf + J) != 0;
        const int rows_pf[2] = {lane < o ? __ldg(rowsJ + lane) : 0, lane + 32 < o ? __ldg(rowsJ + 32 + lane) : 0};
        const T d_pf[2] = {lane < w ? dvec[c0 + lane] : (T)1, lane + 32 < w ? dvec[c0 + lane + 32] : (T)1};
        // own values: final since the forward sweep, loaded before the wait too
        if (a.act0 && a.act1) {
            T* const xq[2] = {x, x + a.dim};
            const T xa[2] = {lane < w ? xq[0][c0 + lane] : (T)0, lane < w ? xq[1][c0 + lane] : (T)0};
            const T xb[2] = {lane + 32 < w ? xq[0][c0 + lane + 32] : (T)0,
                             lane + 32 < w ? xq[1][c0 + lane + 32] : (T)0};
            if (lane == 0 && d.parent >= 0) wait_ge(a.count + d.parent, 1);
            __syncwarp();
            if (staged) {
                mbar_wait(&bars[wid], phase);
                phase ^= 1u;
                { if (sfJ) bwd_body_sf<T, 2>(slice, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb);
                  else bwd_body_tri<T, 2>(slice, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb); }
            } else {
                { if (sfJ) bwd_body_sf<T, 2>(Lg, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb);
                  else bwd_body_tri<T, 2>(Lg, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb); }
            }
        } else {
            T* const xq[1] = {x + (a.act0 ? 0 : a.dim)};
            const T xa[1] = {lane < w ? xq[0][c0 + lane] : (T)0};
            const T xb[1] = {lane + 32 < w ? xq[0][c0 + lane + 32] : (T)0};
            if (lane == 0 && d.parent >= 0) wait_ge(a.count + d.parent, 1);
            __syncwarp();
            if (staged) {
                mbar_wait(&bars[wid], phase);
                phase ^= 1u;
                { if (sfJ) bwd_body_sf<T, 1>(slice, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb);
                  else bwd_body_tri<T, 1>(slice, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb); }
            } else {
                { if (sfJ) bwd_body_sf<T, 1>(Lg, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb);
                  else bwd_body_tri<T, 1>(Lg, a, c0, w, r, o, rowsJ, xq, xs[wid], rows_pf, d_pf, xa, xb); }
            }
        }
        __syncwarp();
        if (lane == 0) st_release(a.count + J, 1);
    }
}

// ---------------------------------------------------------------------------
// refinement glue: permute / accumulate
// ---------------------------------------------------------------------------

template <typename T>
__global__ void gather_perm(const double* __restrict__ r, T* __restrict__ t, const int32_t* __restrict__ perm,
                            int64_t dim, int act0, int act1, const double* rstate, int32_t* __restrict__ z0,
                            int64_t n0, int32_t* __restrict__ z1, int64_t n1, int32_t* __restrict__ z2, int64_t n2) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // the sweeps' dependency counters / done flags / tail flags, reset in the same pass
    for (int64_t i = k; i < n0; i += (int64_t)gridDim.x * blockDim.x) z0[i] = 0;
    for (int64_t i = k; i < n1; i += (int64_t)gridDim.x * blockDim.x) z1[i] = 0;
    for (int64_t i = k; i < n2; i += (int64_t)gridDim.x * blockDim.x) z2[i] = 0;
    resolve_act(rstate, act0, act1);
    if (k >= dim) return;
    const int32_t p = perm[k];
    if (act0) t[k] = (T)r[p];
    if (act1) t[dim + k] = (T)r[dim + p];
}

template <typename T>
__global__ void scatter_add_perm(double* __restrict__ x, const T* __restrict__ t, const int32_t* __restrict__ perm,
                                 int64_t dim, int act0, int act1, const double* rstate, double* __restrict__ best) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // the previous step's iterate becomes the best one if its residual improved
    // (rstate[5], set by the controller; system.py:301-302) — before it is updated
    const bool imp0 = rstate && rstate[5] != 0.0, imp1 = rstate && act1 && rstate[13] != 0.0;
    resolve_act(rstate, act0, act1);
    if (k >= dim) return;
    const int32_t p = perm[k];
    if (imp0) best[p] = x[p];
    if (imp1) best[dim + p] = x[dim + p];
    if (act0) x[p] = x[p] + (double)t[k];
    if (act1) x[dim + p] = x[dim + p] + (double)t[dim + k];
}

SolveArgs solve_args(Ctx& c, int32_t* count, int32_t* ticket, int act0, int act1) {
    SolveArgs a;
    a.nstart = (int32_t)c.host_sym.start_solve.size();
    a.start = c.sym.start_solve;
    a.n_main = (int32_t)c.host_sym.bwd_order.size();
    a.order = c.sym.bwd_order;
    a.ntiny = (int32_t)c.host_sym.tiny.size();
    a.tiny = c.sym.tiny;
    a.ticket_tiny = nullptr;
    a.bwd_done = nullptr;
    a.desc32 = c.sym.desc32;
    a.desc64 = c.sym.desc64;
    a.need = c.sym.need;
    a.dim = c.dim;
    a.nv = c.sym.nv;
    a.sn_rows = c.sym.sn_rows;
    a.vpush_pos = c.sym.vpush_pos;
    a.vin_col = c.sym.vin_col;
    a.count = count;
    a.ticket = ticket;
    a.act0 = act0;
    a.act1 = act1;
    a.trace = nullptr;
    a.slice = (int)c.solve_slice;
    a.rstate = c.rstate;
    a.sf = c.sf_flag;
    a.tdesc = c.sym.tdesc;
    a.trptr = c.sym.trptr;
    return a;
}

// the factor storage's base image (zeros, P and A values, the static +-delta on the
// diagonal), written straight into the factor storage at every assembly: a
// write-only memset plus three small scatters instead of a read + write copy of a
// kept image (the graph's memcpy node ran at ~2 TB/s: C3 170 us per factorisation)
template <typename T>
void build_base_t(Ctx& c, T* base) {
    cudaMemsetAsync(base, 0, sizeof(T) * c.sym.nnz_storage, c.stream);
    if (c.p_nnz) {
        scatter_vals<T><<<grid_for(c.p_nnz), kThreads, 0, c.stream>>>(base, c.sym.map_p, c.p_v, c.p_nnz);
        c.launches++;
    }
    if (c.a_nnz) {
        scatter_vals<T><<<grid_for(c.a_nnz), kThreads, 0, c.stream>>>(base, c.sym.map_a, c.a_v, c.a_nnz);
        c.launches++;
    }
    add_static_reg<T><<<grid_for(c.dim), kThreads, 0, c.stream>>>(base, c.sym.map_diag, c.n, c.dim, c.delta_s);
    c.launches++;
}

template <typename T>
int factor_t(Ctx& c) {
    FactorArgs a;
    a.desc32 = c.sym.desc32;
    a.desc64 = c.sym.desc64;
    a.need = c.sym.need;
    a.push_pos = c.sym.push_pos;
    a.inbox_tgt = c.sym.inbox_tgt;
    a.irow_ptr = c.sym.irow_ptr;
    a.sign = c.sym.sign;
    a.count = c.fac_count;
    a.maxd = c.sn_maxd;
    a.bumps = c.bumps;
    a.err = c.err;
    a.delta_s = c.delta_s;
    a.delta_d = c.delta_d;
    a.trace = c.trace ? c.trace + 6 * (int64_t)c.sym.nsuper : nullptr;
    cudaMemsetAsync(c.fac_count, 0, sizeof(int32_t) * c.sym.nsuper, c.stream);
    cudaMemsetAsync(c.sn_maxd, 0, sizeof(double) * c.sym.nsuper, c.stream);
    cudaMemsetAsync(c.tickets, 0, sizeof(int32_t) * 8, c.stream);
    cudaMemsetAsync(c.bumps, 0, sizeof(int32_t), c.stream);
    int e0 = 0;
    if (c.profile) {
        e0 = (int)(2 * (c.ev_factor.size() + c.ev_solve.size()));
        cudaEventRecord(pooled_event(c, e0), c.stream);
    }
    const int ns_warp = (int)c.host_sym.start_fac_warp.size(), ns_cta = (int)c.host_sym.start_fac_cta.size();
    const int ntiny = (int)c.host_sym.tiny.size();
    if (ntiny > 0) {
        a.ntiny = ntiny;
        a.tiny = c.sym.tiny;
        factor_tiny_kernel<T><<<grid_for(ntiny, TINY_T), TINY_T, 0, c.stream>>>(a, (T*)c.lval, (T*)c.dvec, (T*)c.inbox);
        c.launches++;
    }
    if (ns_warp > 0) {
        a.tier = 0;
        a.nstart = ns_warp;
        a.start = c.sym.start_fac_warp;
        a.ntiny = 0;
        a.ticket_tiny = c.tickets + 4;
        a.ticket = c.tickets;
        a.smem_cap = c.factor_slice;
        factor_kernel<T><<<c.factor_blocks, FW * 32, c.factor_smem, c.stream>>>(a, (T*)c.lval, (T*)c.dvec,
                                                                                (T*)c.inbox);
        c.launches++;
    }
    if (ns_cta > 0) {
        a.ntiny = 0;
        a.tier = 1;
        a.nstart = ns_cta;
        a.start = c.sym.start_fac_cta;
        a.ticket = c.tickets + 3;
        a.smem_cap = c.factor_cta_smem / (int64_t)sizeof(T);
        factor_cta_kernel<T><<<c.factor_cta_blocks, 256, c.factor_cta_smem, c.stream>>>(a, (T*)c.lval, (T*)c.dvec,
                                                                                       (T*)c.inbox);
        c.launches++;
    }
    // the solve-form pass only touches warp / CTA-tier panels, which the dense
    // tail never reads (it consumes their inbox contributions): run it on the
    // side stream while the tail factorises (fork / join; captured into the
    // factor graph as two parallel branches)
    const int nsf = (int)c.host_sym.bwd_order.size();
    const bool sf = nsf > 0 && c.solve_form;
    static const bool overlap = !getenv("CIPM_SF_SERIAL");
    cudaStream_t sfs = c.stream;
    if (sf && overlap) {
        cudaEventRecord(c.fork_ev, c.stream);
        cudaStreamWaitEvent(c.side, c.fork_ev, 0);
        sfs = c.side;
    }
    if (sf) {
        const int slice = (int)c.solve_form_slice;
        const size_t smem = sizeof(T) * (size_t)(c.solve_form_inv + slice) * SFW;
        solve_form_kernel<T><<<c.solve_form_blocks, SFW * 32, smem, sfs>>>(c.sym.bwd_order, nsf, c.sym.desc32,
                                                                           c.sym.desc64, (T*)c.lval, slice,
                                                                           c.solve_form_inv, c.sf_tau, c.sf_flag);
        c.launches++;
    }
    k_tail_factor(c);
    if (sf && overlap) {
        cudaEventRecord(c.join_ev, c.side);
        cudaStreamWaitEvent(c.stream, c.join_ev, 0);
    }
    if (c.profile) {
        cudaEventRecord(pooled_event(c, e0 + 1), c.stream);
        c.ev_factor.emplace_back(e0, e0 + 1);
    }
    return CIPM_OK;
}

// CIPM_PHASES=1 (probes only): per-launch warm timings of one sweep pair, on stderr
struct PhaseTimer {
    Ctx& c;
    bool on;
    std::vector<std::pair<const char*, cudaEvent_t>> ev;
    explicit PhaseTimer(Ctx& cc) : c(cc), on(false) {
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(c.stream, &st);
        on = getenv("CIPM_PHASES") != nullptr && st == cudaStreamCaptureStatusNone;
        mark("start");
    }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, c.stream);
        ev.emplace_back(name, e);
    }
    ~PhaseTimer() {
        if (!on) return;
        cudaEventSynchronize(ev.back().second);
        fprintf(stderr, "[phases]");
        for (size_t k = 1; k < ev.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[k - 1].second, ev[k].second);
            fprintf(stderr, " %s=%.1f", ev[k].first, ms * 1000.f);
        }
        fprintf(stderr, " us\n");
        for (auto& p : ev) cudaEventDestroy(p.second);
    }
};

template <typename T>
void refine_solve_t(Ctx& c, int act0, int act1, bool gather) {
    PhaseTimer pt(c);
    T* t = (T*)c.rt;
    cudaMemsetAsync(c.tickets, 0, sizeof(int32_t) * 8, c.stream);
    if (gather) gather_perm<T><<<grid_for(c.dim), kThreads, 0, c.stream>>>(c.rr, t, c.sym.perm, c.dim, act0, act1, c.rstate,
                                                               c.fac_count, c.sym.nsuper, c.bwd_done, c.sym.nsuper,
                                                               c.tflags, c.tflag_total);
    int e0 = 0;
    if (c.profile) {
        e0 = (int)(2 * (c.ev_factor.size() + c.ev_solve.size()));
        cudaEventRecord(pooled_event(c, e0), c.stream);
    }
    SolveArgs f = solve_args(c, c.fac_count, c.tickets + 1, act0, act1);
    f.ticket_tiny = c.tickets + 5;
    f.trace = c.trace;
    const size_t ssm = sizeof(T) * (size_t)c.solve_slice * SW;
    if (f.ntiny > 0) {
        fwd_tiny_kernel<T><<<grid_for(f.ntiny, TINY_T), TINY_T, 0, c.stream>>>(f, (const T*)c.lval, t, (T*)c.vin);
        c.launches++;
    }
    pt.mark("gather+fwd_tiny");
    f.ntiny = 0;
    if (c.sym.ntfold > 0) {
        tiny_fold_kernel<T><<<grid_for(c.sym.ntfold, 256), 256, 0, c.stream>>>(f, c.sym.tfold_cols, c.sym.ntfold,
                                                                               c.sym.vt_lo, c.sym.vt_hi, t,
                                                                               (const T*)c.vin);
        c.launches++;
    }
    pt.mark("fold");
    if (f.nstart > 0) forward_kernel<T><<<c.solve_blocks, SW * 32, ssm, c.stream>>>(f, (const T*)c.lval, t, (T*)c.vin);
    pt.mark("forward");
    if (tail_is_single_root(c)) {
        k_root_solve(c, t, act0, act1);
        pt.mark("root_solve");
    } else {
        k_tail_forward(c, t, act0, act1);
        pt.mark("tail_fwd");
        k_tail_backward(c, t, act0, act1);
        pt.mark("tail_bwd");
    }
    SolveArgs b = solve_args(c, c.bwd_done, c.tickets + 2, act0, act1);
    b.ticket_tiny = c.tickets + 6;
    if (b.n_main > 0)
        backward_kernel<T><<<c.solve_blocks, SW * 32, ssm, c.stream>>>(b, (const T*)c.lval, (const T*)c.dvec, t);
    pt.mark("backward");
    if (b.ntiny > 0) {
        bwd_tiny_kernel<T><<<grid_for(b.ntiny, TINY_T), TINY_T, 0, c.stream>>>(b, (const T*)c.lval, (const T*)c.dvec, t);
        c.launches++;
    }
    if (c.profile) {
        cudaEventRecord(pooled_event(c, e0 + 1), c.stream);
        c.ev_solve.emplace_back(e0, e0 + 1);
    }
    pt.mark("bwd_tiny");
    scatter_add_perm<T><<<grid_for(c.dim), kThreads, 0, c.stream>>>(c.rx, t, c.sym.perm, c.dim, act0, act1,
                                                                    c.rstate, c.rbest);
    pt.mark("scatter");
    c.launches += 4;
}

}  // namespace

void k_build_base(Ctx&) {
    // nothing to precompute: k_assemble rebuilds the base image from the current P / A
    // values (p_v, a_v) in place at every factorisation
}

void k_assemble(Ctx& c) {
    if (c.precision == CIPM_FULL) build_base_t<double>(c, (double*)c.lval);
    else build_base_t<float>(c, (float*)c.lval);
    k_scatter_h(c);
}

int k_factor(Ctx& c) {
    return c.precision == CIPM_FULL ? factor_t<double>(c) : factor_t<float>(c);
}

// one refinement correction: x += solve(r) for the active right-hand sides
void k_refine_step(Ctx& c, int nrhs, const int* active, bool gather) {
    const int a0 = active[0], a1 = nrhs > 1 ? active[1] : 0;
    if (c.profile) c.solve_rhs += a0 + a1;
    if (c.precision == CIPM_FULL) refine_solve_t<double>(c, a0, a1, gather);
    else refine_solve_t<float>(c, a0, a1, gather);
}

// the first step's permuted right-hand side (and the sweep counters' reset) when the
// fused residual gathers for the later steps
void k_refine_gather(Ctx& c, int nrhs) {
    const int a1 = nrhs > 1 ? 1 : 0;
    if (c.precision == CIPM_FULL)
        gather_perm<double><<<grid_for(c.dim), kThreads, 0, c.stream>>>(
            c.rr, (double*)c.rt, c.sym.perm, c.dim, 1, a1, c.rstate, c.fac_count, c.sym.nsuper, c.bwd_done,
            c.sym.nsuper, c.tflags, c.tflag_total);
    else
        gather_perm<float><<<grid_for(c.dim), kThreads, 0, c.stream>>>(
            c.rr, (float*)c.rt, c.sym.perm, c.dim, 1, a1, c.rstate, c.fac_count, c.sym.nsuper, c.bwd_done,
            c.sym.nsuper, c.tflags, c.tflag_total);
    c.launches++;
}

}  // namespace cipm

namespace cipm {

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

int factor_grid(Ctx& c) {
    // per-warp shared-memory panel slice: the largest non-tail panel, capped at
    // 6 KiB so four 8-warp CTAs fit per SM; bigger panels are factored in place
    const int64_t es = c.precision == CIPM_FULL ? 8 : 4;
    int64_t slice = std::min<int64_t>((c.host_sym.max_panel_warp + 3) & ~int64_t(3), 6144 / es);   // 16-byte multiple (TMA)
    if (slice < 64) slice = 64;
    c.factor_slice = slice;
    c.factor_smem = (int)(slice * es * FW);
    int per = 0;
    if (c.precision == CIPM_FULL) {
        cudaFuncSetAttribute(factor_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, c.factor_smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, factor_kernel<double>, FW * 32, c.factor_smem);
    } else {
        cudaFuncSetAttribute(factor_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, c.factor_smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, factor_kernel<float>, FW * 32, c.factor_smem);
    }
    if (per < 1) per = 1;
    int64_t g = (int64_t)sm_count() * per;
    const int64_t need = (c.host_sym.n_warp + FW - 1) / FW;
    if (g > need) g = need;
    if (const char* e = getenv("CIPM_FACTOR_BLOCKS")) g = std::min<int64_t>(g, atoll(e));   // experiments
    // mid tier: one CTA per supernode, panel in dynamic shared memory up to 96 KiB
    {
        int64_t cap = std::min<int64_t>(c.host_sym.max_panel_main * es, 96 * 1024);
        if (cap < 1024) cap = 1024;
        c.factor_cta_smem = (int)cap;
        int pc = 0;
        if (c.precision == CIPM_FULL) {
            cudaFuncSetAttribute(factor_cta_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pc, factor_cta_kernel<double>, 256, (int)cap);
        } else {
            cudaFuncSetAttribute(factor_cta_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pc, factor_cta_kernel<float>, 256, (int)cap);
        }
        if (pc < 1) pc = 1;
        int64_t gc = (int64_t)sm_count() * pc;
        const int64_t nmid = c.host_sym.n_main - c.host_sym.n_warp;
        if (gc > nmid) gc = nmid;
        c.factor_cta_blocks = (int)(gc < 1 ? 1 : gc);
    }
    return (int)(g < 1 ? 1 : g);
}

int solve_grid(Ctx& c) {
    // per-warp panel slice: up to 8 KiB (three 8-warp CTAs per SM); larger panels are read from L2/HBM
    const int64_t es = c.precision == CIPM_FULL ? 8 : 4;
    // Staging every panel (slice = the largest non-tail panel) pays when a level
    // holds fewer tasks than the GPU has warps; wide levels want occupancy instead
    // (smaller slices, more CTAs per SM).  Measured on the B200: C2 / C5a stage
    // everything (pair -10 % / -15 %), C3 (65k leaf-level warp tasks) wants 6 KB.
    {
        const Symbolic& S = c.host_sym;
        std::vector<int64_t> per_level(S.height + 1, 0);
        std::vector<char> tiny(S.nsuper, 0);
        for (int32_t J : S.tiny) tiny[J] = 1;
        for (int32_t J = 0; J < S.nsuper; ++J)
            if (!S.is_tail[J] && !tiny[J]) per_level[S.level[J]]++;
        const int64_t widest = *std::max_element(per_level.begin(), per_level.end());
        const int64_t warps_1cta = (int64_t)sm_count() * SW;          // one 8-warp CTA per SM
        const int64_t full = (c.host_sym.max_panel_main + 3) & ~int64_t(3);
        const int64_t cap = (200 * 1024 / SW) / es;                     // one CTA per SM at most
        if (widest <= 8 * warps_1cta) c.solve_slice = std::max<int64_t>(64, std::min<int64_t>(full, cap));
        else c.solve_slice = std::max<int64_t>(64, std::min<int64_t>(full, 6144 / es));
    }
    if (const char* e = getenv("CIPM_SOLVE_SLICE")) c.solve_slice = std::max<int64_t>(4, atoll(e) & ~int64_t(3));   // experiments
    const int ssm = (int)(es * c.solve_slice * SW);
    int per = 0, per2 = 0;
    if (c.precision == CIPM_FULL) {
        cudaFuncSetAttribute(forward_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm);
        cudaFuncSetAttribute(backward_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, forward_kernel<double>, SW * 32, ssm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, backward_kernel<double>, SW * 32, ssm);
    } else {
        cudaFuncSetAttribute(forward_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm);
        cudaFuncSetAttribute(backward_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, forward_kernel<float>, SW * 32, ssm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, backward_kernel<float>, SW * 32, ssm);
    }
    per = std::min(per, per2);
    if (per < 1) per = 1;
    {
        // solve-form pass: one warp per supernode, Linv (64 x 64) + a panel slice of up to 16 KiB per warp
        c.solve_form_slice = std::max<int64_t>(64, std::min<int64_t>((c.host_sym.max_panel_main + 3) & ~int64_t(3),
                                                                     16384 / es));
        int64_t maxw = 1;
        for (int32_t J : c.host_sym.bwd_order)
            maxw = std::max<int64_t>(maxw, c.host_sym.sn_col[J + 1] - c.host_sym.sn_col[J]);
        c.solve_form_inv = (int)((maxw * maxw + 3) & ~int64_t(3));
        const int sfm = (int)(es * (c.solve_form_inv + c.solve_form_slice) * SFW);
        int pf = 0;
        if (c.precision == CIPM_FULL) {
            cudaFuncSetAttribute(solve_form_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, sfm);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pf, solve_form_kernel<double>, SFW * 32, sfm);
        } else {
            cudaFuncSetAttribute(solve_form_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, sfm);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pf, solve_form_kernel<float>, SFW * 32, sfm);
        }
        if (pf < 1) pf = 1;
        const int64_t nsf = (int64_t)c.host_sym.bwd_order.size();
        c.solve_form_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count() * pf, (nsf + SFW - 1) / SFW));
    }
    int64_t g = (int64_t)sm_count() * per;
    int64_t need = (c.host_sym.n_main + SW - 1) / SW;
    if (g > need) g = need;
    if (const char* e = getenv("CIPM_SOLVE_BLOCKS")) g = std::min<int64_t>(g, atoll(e));     // experiments
    return (int)(g < 1 ? 1 : g);
}

}  // namespace cipm
