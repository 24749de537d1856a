// Supernodal quasi-definite LDL' on sm_100a: numeric refactorisation and
// triangular solves (replaces kkt/ldl.py:37-104 and kkt/system.py:246-271).
//
// Scheduling: one persistent launch per phase.  Tasks (supernodes) are handed
// out by an atomic ticket in a fixed topological order (leaves first), and a
// task spins on per-supernode dependency counters until its inputs are final.
// A task only ever waits on tasks with smaller tickets, which are already held
// by running CTAs/warps, so the scheme cannot deadlock; there is one launch per
// factorisation / solve instead of one per elimination-tree level.
//
// Numerics: left-looking (fan-in).  Supernode J gathers the updates of every
// descendant K listed in its update list in a fixed order, then factors its
// dense panel.  No atomics touch floating-point data, so factors and solutions
// are bitwise reproducible run to run (SPEC kkt-solver "Determinism").
// Dynamic regularisation (ldl.py:79-87): a pivot with |d| < δs + δd·runmax is
// replaced by ±bound with the sign of its block; runmax is the largest |D| in
// the supernode's subtree computed so far (the sequential reference uses all
// earlier pivots; δd = eps² makes the term negligible — DESIGN.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ctx.hpp"

namespace cipm {

namespace {

__device__ __forceinline__ int64_t gtimer() {
    int64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
    return __ldcg(p);
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
// numeric factorisation (push/pull inbox scheme)
//
// Task J (one CTA): wait until its children are done; copy its panel to shared
// memory; gather its inbox — every contribution block entry of every descendant
// that lands in J, pre-sorted by (row, column, source) so each thread owns one
// panel row and accumulates runs in registers (no atomics, no barriers, fixed
// order); factor the dense panel; write L and D; then compute its own packed
// contribution block C_J = L_off D L_off' and scatter it into the ancestors'
// inboxes.  The expensive dot products therefore run in the producer, spread
// over many CTAs, instead of serially in the consumer.
// ---------------------------------------------------------------------------

struct FactorArgs {
    int32_t nsuper;      // tickets t in [t_begin, nsuper) of `order`
    int32_t t_begin;
    const int32_t* order;
    const int32_t* sn_col;
    const int64_t* sn_rptr;
    const int64_t* sn_loff;
    const int32_t* sn_parent;
    const int32_t* sn_nchild;
    const int64_t* cb_off;
    const int64_t* push_pos;
    const int64_t* irow_ptr;
    const int32_t* inbox_tgt;
    const int8_t* sign;
    int32_t* count;
    int32_t* ticket;
    double* maxd;        // max |D| over the subtree, accumulated by the children (atomic max)
    int32_t* bumps;
    int* err;
    double delta_s, delta_d;
    int64_t smem_cap;    // panel elements that fit the dynamic shared memory
    int64_t* trace;      // optional per-task timeline (cipm_trace)
};

__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// Warp-cooperative segmented gather: entries [lo, hi) sorted so that equal
// targets are contiguous; P[tgt] -= sum of their values (fixed order: a warp
// Hillis-Steele scan per 32-entry chunk, carries across chunks).
template <typename T>
__device__ __forceinline__ void warp_gather_sub(T* P, const int32_t* __restrict__ tgt, const T* vals, int64_t lo,
                                                int64_t hi) {
    const int lane = threadIdx.x & 31;
    int carry_t = -1;
    T carry = (T)0;
    for (int64_t base = lo; base < hi; base += 32) {
        const int64_t e = base + lane;
        const bool valid = e < hi;
        const int tg = valid ? tgt[e] : -(lane + 2);
        T v = valid ? __ldcg(vals + e) : (T)0;
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
    __syncwarp();
}

constexpr int FW = 8;   // warps per factor CTA

// Task J (one warp): wait until its children are done; stage its panel in the
// warp's shared-memory slice (in place in HBM when it does not fit); gather its
// inbox (every contribution entry of every descendant that lands in J, sorted
// by target, fixed-order segmented sums); factor the dense panel; write L and
// D; then compute its packed contribution block C_J = L_off D L_off' and
// scatter it into the ancestors' inboxes.  No floating-point atomics.
template <typename T>
__global__ void __launch_bounds__(FW * 32) factor_kernel(FactorArgs a, T* __restrict__ lval, T* __restrict__ dvec,
                                                         T* __restrict__ inbox) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ T sD[FW][64];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T* sp = reinterpret_cast<T*>(smem_raw) + (int64_t)wid * a.smem_cap;
    for (;;) {
        int t = 0;
        if (lane == 0) t = a.t_begin + atomicAdd(a.ticket, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= a.nsuper) return;
        const int J = a.order[t];
        double runmax = 0.0;
        if (lane == 0) {
            if (a.trace) a.trace[3 * t] = gtimer();
            wait_ge(a.count + J, a.sn_nchild[J]);
            runmax = __ldcg(a.maxd + J);
            if (a.trace) a.trace[3 * t + 1] = gtimer();
        }
        runmax = __shfl_sync(0xffffffffu, runmax, 0);
        const int c0 = a.sn_col[J];
        const int w = a.sn_col[J + 1] - c0;
        const int64_t r0 = a.sn_rptr[J];
        const int r = (int)(a.sn_rptr[J + 1] - r0);
        const int o = r - w;
        T* L = lval + a.sn_loff[J];
        const int psize = r * w;
        const bool in_smem = psize <= a.smem_cap;
        T* P = in_smem ? sp : L;
        if (in_smem)
            for (int i = lane; i < psize; i += 32) sp[i] = L[i];
        __syncwarp();

        // 1. gather the inbox of all r rows (one contiguous, target-sorted range)
        warp_gather_sub(P, a.inbox_tgt, inbox, a.irow_ptr[r0], a.irow_ptr[r0 + r]);

        // 2. dense LDL' of the panel (right-looking, lanes over rows)
        for (int j = 0; j < w; ++j) {
            T* Pj = P + j * r;
            double d = (double)Pj[j];
            const double bound = a.delta_s + a.delta_d * runmax;
            const bool bump = fabs(d) < bound;
            if (bump) d = a.sign[c0 + j] > 0 ? bound : -bound;
            const T dt = (T)d;
            runmax = fmax(runmax, fabs(d));
            __syncwarp();
            if (lane == 0) {
                if (bump) atomicAdd(a.bumps, 1);
                if (dt == (T)0) set_error(a.err, CIPM_E_FACTOR);
                dvec[c0 + j] = dt;
                sD[wid][j] = dt;
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

        // 3. write the factor back, then push C_J = L_off D L_off' into the ancestors' inboxes
        if (in_smem)
            for (int i = lane; i < psize; i += 32) L[i] = sp[i];
        if (o > 0) {
            const int64_t base = a.cb_off[J];
            const T* Dj = sD[wid];
            int64_t tb = 0;   // packed offset of column bb
            for (int bb = 0; bb < o; ++bb) {
                const T* Pb = P + w + bb;
                for (int aa = bb + lane; aa < o; aa += 32) {
                    T acc = (T)0;
                    for (int k = 0; k < w; ++k) acc += P[k * r + w + aa] * Dj[k] * Pb[k * r];
                    inbox[a.push_pos[base + tb + (aa - bb)]] = acc;
                }
                tb += o - bb;
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            const int Pn = a.sn_parent[J];
            if (Pn >= 0) {
                atomic_max_pos(a.maxd + Pn, runmax);
                __threadfence();
                atomicAdd(a.count + Pn, 1);
            }
            if (a.trace) a.trace[3 * t + 2] = gtimer();
        }
    }
}


// Mid tier (one CTA per supernode): the same task for panels too large for one
// warp — the inbox gather is split by rows over the CTA's warps, the dense
// panel LDL' uses all threads, the contribution block is computed by all
// threads.  Launched after the warp tier, before the dense tail.
template <typename T>
__global__ void __launch_bounds__(256) factor_cta_kernel(FactorArgs a, T* __restrict__ lval, T* __restrict__ dvec,
                                                         T* __restrict__ inbox) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sp = reinterpret_cast<T*>(smem_raw);
    __shared__ int s_task;
    __shared__ double s_piv;
    __shared__ double s_runmax;
    __shared__ T sD[64];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    for (;;) {
        if (tid == 0) s_task = a.t_begin + atomicAdd(a.ticket, 1);
        __syncthreads();
        const int t = s_task;
        if (t >= a.nsuper) return;
        const int J = a.order[t];
        if (tid == 0) {
            if (a.trace) a.trace[3 * t] = gtimer();
            wait_ge(a.count + J, a.sn_nchild[J]);
            s_runmax = __ldcg(a.maxd + J);
            if (a.trace) a.trace[3 * t + 1] = gtimer();
        }
        __syncthreads();
        const int c0 = a.sn_col[J];
        const int w = a.sn_col[J + 1] - c0;
        const int64_t r0 = a.sn_rptr[J];
        const int r = (int)(a.sn_rptr[J + 1] - r0);
        const int o = r - w;
        T* L = lval + a.sn_loff[J];
        const int64_t psize = (int64_t)r * w;
        const bool in_smem = psize <= a.smem_cap;
        T* P = in_smem ? sp : L;
        if (in_smem)
            for (int64_t i = tid; i < psize; i += nt) sp[i] = L[i];
        __syncthreads();
        // 1. inbox gather, rows split over the warps (targets are unique per row)
        {
            const int rs = (int)((int64_t)r * wid / nw), re = (int)((int64_t)r * (wid + 1) / nw);
            if (re > rs) warp_gather_sub(P, a.inbox_tgt, inbox, a.irow_ptr[r0 + rs], a.irow_ptr[r0 + re]);
            (void)lane;
        }
        __syncthreads();
        // 2. dense LDL' of the panel (right-looking inside the panel)
        for (int j = 0; j < w; ++j) {
            if (tid == 0) {
                double d = (double)P[(int64_t)j * r + j];
                const double bound = a.delta_s + a.delta_d * s_runmax;
                if (fabs(d) < bound) {
                    d = a.sign[c0 + j] > 0 ? bound : -bound;
                    atomicAdd(a.bumps, 1);
                }
                const T dt = (T)d;
                if (dt == (T)0) set_error(a.err, CIPM_E_FACTOR);
                dvec[c0 + j] = dt;
                sD[j] = dt;
                P[(int64_t)j * r + j] = (T)1;
                s_piv = (double)dt;
                s_runmax = fmax(s_runmax, fabs(d));
            }
            __syncthreads();
            const T d = (T)s_piv;
            T* Pj = P + (int64_t)j * r;
            for (int i = j + 1 + tid; i < r; i += nt) Pj[i] = Pj[i] / d;
            __syncthreads();
            const int rem_c = w - j - 1;
            if (rem_c > 0) {
                const int rows = r - j - 1;
                const int64_t total = (int64_t)rem_c * rows;
                for (int64_t idx = tid; idx < total; idx += nt) {
                    const int i = j + 1 + (int)(idx % rows);
                    const int c = j + 1 + (int)(idx / rows);
                    if (i < c) continue;
                    P[(int64_t)c * r + i] -= Pj[i] * d * Pj[c];
                }
            }
            __syncthreads();
        }
        // 3. write back, push C_J = L_off D L_off'
        if (in_smem)
            for (int64_t i = tid; i < psize; i += nt) L[i] = sp[i];
        if (o > 0) {
            const int64_t base = a.cb_off[J];
            const int64_t tot = (int64_t)o * o;
            for (int64_t idx = tid; idx < tot; idx += nt) {
                const int aa = (int)(idx % o), bb = (int)(idx / o);
                if (aa < bb) continue;
                T acc = (T)0;
                for (int k = 0; k < w; ++k) acc += P[(int64_t)k * r + w + aa] * sD[k] * P[(int64_t)k * r + w + bb];
                const int64_t tpk = (int64_t)bb * o - (int64_t)bb * (bb - 1) / 2 + (aa - bb);
                inbox[a.push_pos[base + tpk]] = acc;
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const int Pn = a.sn_parent[J];
            if (Pn >= 0) {
                atomic_max_pos(a.maxd + Pn, s_runmax);
                __threadfence();
                atomicAdd(a.count + Pn, 1);
            }
            if (a.trace) a.trace[3 * t + 2] = gtimer();
        }
    }
}

// ---------------------------------------------------------------------------
// triangular solves, one warp per supernode task (push/pull for the forward sweep)
// ---------------------------------------------------------------------------

struct SolveArgs {
    int32_t nsuper;
    int64_t dim;
    int64_t nv;          // vector inbox length per right-hand side
    const int32_t* order;
    const int32_t* sn_col;
    const int64_t* sn_rptr;
    const int32_t* sn_rows;
    const int64_t* sn_loff;
    const int32_t* sn_parent;
    const int32_t* sn_nchild;
    const int64_t* cv_off;
    const int64_t* vpush_pos;
    const int64_t* vcol_ptr;
    int32_t* count;      // forward: children done; backward: done flags
    int32_t* ticket;
    int act0, act1;      // active right-hand sides
    int64_t* trace;      // optional per-task timeline (cipm_trace): ticket / ready / done (ns)
    int slice;           // per-warp shared-memory panel slice (elements)
};


// warp-cooperative sums of the vector inbox of columns c0 .. c0+w-1 (one
// contiguous range grouped by column): colsum[j] = sum of column c0+j's entries.
// Four 32-entry chunks are loaded before they are reduced (memory parallelism).
template <typename T>
__device__ __forceinline__ void vgather_warp(const T* vq, const int64_t* __restrict__ gptr, int c0, int w,
                                             T* colsum, int64_t* win) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < w; j += 32) colsum[j] = (T)0;
    for (int j = lane; j <= w; j += 32) win[j] = gptr[c0 + j];   // column-pointer window
    __syncwarp();
    const int64_t lo = win[0], hi = win[w];
    for (int64_t base = lo; base < hi; base += 128) {
        T v[4];
        int col[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t e = base + 32 * u + lane;
            v[u] = e < hi ? __ldcg(vq + e) : (T)0;
            col[u] = -(lane + 2);
            if (e < hi) {
                int lc = 0, hc = w - 1;
                while (lc < hc) {
                    const int mid = (lc + hc + 1) >> 1;
                    if (win[mid] <= e) lc = mid; else hc = mid - 1;
                }
                col[u] = lc;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            T x = v[u];
            const int cu = col[u];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int cp = __shfl_up_sync(0xffffffffu, cu, off);
                const T vp = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off && cp == cu) x += vp;
            }
            const int cn = __shfl_down_sync(0xffffffffu, cu, 1);
            if (cu >= 0 && (lane == 31 || cn != cu)) colsum[cu] += x;
            __syncwarp();
        }
    }
    __syncwarp();
}

// stage a panel (r*w elements, 16-byte aligned in HBM) in the warp's shared-memory
// slice with one TMA bulk copy when it fits; otherwise read it in place
template <typename T>
__device__ __forceinline__ const T* stage_panel(const T* L, int psize, T* slice, int cap, uint64_t* bar,
                                                uint32_t& phase) {
    const uint32_t bytes = ((uint32_t)psize * (uint32_t)sizeof(T) + 15u) & ~15u;
    if (bytes > (uint32_t)cap * (uint32_t)sizeof(T)) return L;
    fence_proxy_async_smem();     // every lane's earlier generic reads of the slice precede the async write
    __syncwarp();
    if ((threadIdx.x & 31) == 0) bulk_g2s(slice, L, bytes, bar);
    mbar_wait(bar, phase);
    phase ^= 1u;
    return slice;
}

constexpr int SW = 8;   // warps per solve CTA

// forward sweep L y = b: warp per supernode, columns in registers (lane owns
// columns lane and lane+32; non-tail supernodes are narrower than 64), panel
// staged in shared memory
template <typename T>
__global__ void __launch_bounds__(SW * 32) forward_kernel(SolveArgs a, const T* __restrict__ lval, T* x, T* vin) {
    extern __shared__ __align__(16) unsigned char sraw[];
    __shared__ T colsum[SW][64];
    __shared__ int64_t vwin[SW][65];
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
        if (t >= a.nsuper) return;
        const int J = a.order[t];
        if (a.trace && lane == 0) a.trace[6 * t] = gtimer();
        if (lane == 0) {
            const int need = a.sn_nchild[J];
            if (need > 0) wait_ge(a.count + J, need);
        }
        __syncwarp();
        if (a.trace && lane == 0) a.trace[6 * t + 1] = gtimer();
        const int c0 = a.sn_col[J];
        const int w = a.sn_col[J + 1] - c0;
        const int64_t r0 = a.sn_rptr[J];
        const int r = (int)(a.sn_rptr[J + 1] - r0);
        const int64_t cvo = a.cv_off[J];
        const T* L = stage_panel(lval + a.sn_loff[J], r * w, slice, a.slice, &bars[wid], phase);
        for (int q = 0; q < 2; ++q) {
            if (!(q == 0 ? a.act0 : a.act1)) continue;
            T* xJ = x + (int64_t)q * a.dim + c0;
            T* vq = vin + (int64_t)q * a.nv;
            T* cs = colsum[wid];
            vgather_warp(vq, a.vcol_ptr, c0, w, cs, vwin[wid]);
            if (a.trace && lane == 0) a.trace[6 * t + 2] = gtimer();
            T x0 = (T)0, x1 = (T)0;
            if (lane < w) x0 = xJ[lane] - cs[lane];
            if (lane + 32 < w) x1 = xJ[lane + 32] - cs[lane + 32];
            for (int j = 0; j < w; ++j) {
                const T l0 = (lane > j && lane < w) ? L[j * r + lane] : (T)0;
                const T l1 = (lane + 32 > j && lane + 32 < w) ? L[j * r + lane + 32] : (T)0;
                const T xj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
                x0 -= l0 * xj;
                x1 -= l1 * xj;
            }
            if (lane < w) xJ[lane] = x0;
            if (lane + 32 < w) xJ[lane + 32] = x1;
            if (a.trace && lane == 0) a.trace[6 * t + 3] = gtimer();
            for (int i0 = w; i0 < r; i0 += 32) {
                const int i = i0 + lane;
                const bool ok = i < r;
                const int ii = ok ? i : r - 1;
                T acc = (T)0;
                for (int k = 0; k < w; ++k) {
                    const T xk = __shfl_sync(0xffffffffu, k < 32 ? x0 : x1, k & 31);
                    acc += L[k * r + ii] * xk;
                }
                if (ok) vq[a.vpush_pos[cvo + i - w]] = acc;
            }
            if (a.trace && lane == 0) a.trace[6 * t + 4] = gtimer();
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            const int P = a.sn_parent[J];
            if (P >= 0) atomicAdd(a.count + P, 1);
            if (a.trace) a.trace[6 * t + 5] = gtimer();
        }
    }
}

// backward sweep L' x = D^-1 y: warp per supernode, reverse topological order
template <typename T>
__global__ void __launch_bounds__(SW * 32) backward_kernel(SolveArgs a, const T* __restrict__ lval,
                                                           const T* __restrict__ dvec, T* x) {
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
        if (t >= a.nsuper) return;
        const int J = a.order[a.nsuper - 1 - t];
        const int P = a.sn_parent[J];
        if (lane == 0 && P >= 0) wait_ge(a.count + P, 1);
        __syncwarp();
        const int c0 = a.sn_col[J];
        const int w = a.sn_col[J + 1] - c0;
        const int64_t r0 = a.sn_rptr[J];
        const int r = (int)(a.sn_rptr[J + 1] - r0);
        const int o = r - w;
        const int32_t* rowsJ = a.sn_rows + r0 + w;
        const T* L = stage_panel(lval + a.sn_loff[J], r * w, slice, a.slice, &bars[wid], phase);
        const T* L0 = L + lane * r;
        const T* L1 = L + (lane + 32) * r;
        const bool o0 = lane < w, o1 = lane + 32 < w;
        for (int q = 0; q < 2; ++q) {
            if (!(q == 0 ? a.act0 : a.act1)) continue;
            T* xv = x + (int64_t)q * a.dim;
            T* xJ = xv + c0;
            T x0 = o0 ? xJ[lane] / dvec[c0 + lane] : (T)0;      // D solve (ldl.py:101-102)
            T x1 = o1 ? xJ[lane + 32] / dvec[c0 + lane + 32] : (T)0;
            // ancestors' values at the off rows: gathered once (coalesced over lanes)
            for (int i0 = 0; i0 < o; i0 += 64) {
                T* xo = xs[wid][0];
                const int n = min(64, o - i0);
                if (lane < n) xo[lane] = __ldcg(xv + rowsJ[i0 + lane]);
                if (lane + 32 < n) xo[lane + 32] = __ldcg(xv + rowsJ[i0 + lane + 32]);
                __syncwarp();
                for (int k = 0; k < n; ++k) {
                    const T xi = xo[k];
                    if (o0) x0 -= L0[w + i0 + k] * xi;
                    if (o1) x1 -= L1[w + i0 + k] * xi;
                }
                __syncwarp();
            }
            for (int j = w - 1; j >= 0; --j) {
                const T xj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
                if (lane < j) x0 -= L0[j] * xj;
                if (lane + 32 < j) x1 -= L1[j] * xj;
            }
            if (o0) xJ[lane] = x0;
            if (o1) xJ[lane + 32] = x1;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.count + J, 1);
    }
}

// ---------------------------------------------------------------------------
// refinement glue: permute / accumulate
// ---------------------------------------------------------------------------

template <typename T>
__global__ void gather_perm(const double* __restrict__ r, T* __restrict__ t, const int32_t* __restrict__ perm,
                            int64_t dim, int act0, int act1) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= dim) return;
    const int32_t p = perm[k];
    if (act0) t[k] = (T)r[p];
    if (act1) t[dim + k] = (T)r[dim + p];
}

template <typename T>
__global__ void scatter_add_perm(double* __restrict__ x, const T* __restrict__ t, const int32_t* __restrict__ perm,
                                 int64_t dim, int act0, int act1) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= dim) return;
    const int32_t p = perm[k];
    if (act0) x[p] = x[p] + (double)t[k];
    if (act1) x[dim + p] = x[dim + p] + (double)t[dim + k];
}

SolveArgs solve_args(Ctx& c, int32_t* count, int32_t* ticket, int act0, int act1) {
    SolveArgs a;
    a.nsuper = c.host_sym.n_main;
    a.dim = c.dim;
    a.nv = c.sym.nv;
    a.order = c.sym.order;
    a.sn_col = c.sym.sn_col;
    a.sn_rptr = c.sym.sn_rptr;
    a.sn_rows = c.sym.sn_rows;
    a.sn_loff = c.sym.sn_loff;
    a.sn_parent = c.sym.sn_parent;
    a.sn_nchild = c.sym.sn_nchild;
    a.cv_off = c.sym.cv_off;
    a.vpush_pos = c.sym.vpush_pos;
    a.vcol_ptr = c.sym.vcol_ptr;
    a.count = count;
    a.ticket = ticket;
    a.act0 = act0;
    a.act1 = act1;
    a.trace = nullptr;
    a.slice = (int)c.solve_slice;
    return a;
}

template <typename T>
void build_base_t(Ctx& c) {
    T* base = (T*)c.lbase;
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
    a.nsuper = c.host_sym.n_main;
    a.order = c.sym.order;
    a.sn_col = c.sym.sn_col;
    a.sn_rptr = c.sym.sn_rptr;
    a.sn_loff = c.sym.sn_loff;
    a.sn_parent = c.sym.sn_parent;
    a.sn_nchild = c.sym.sn_nchild;
    a.cb_off = c.sym.cb_off;
    a.push_pos = c.sym.push_pos;
    a.irow_ptr = c.sym.irow_ptr;
    a.inbox_tgt = c.sym.inbox_tgt;
    a.sign = c.sym.sign;
    a.count = c.fac_count;
    a.ticket = c.tickets;
    a.maxd = c.sn_maxd;
    a.bumps = c.bumps;
    a.err = c.err;
    a.delta_s = c.delta_s;
    a.delta_d = c.delta_d;
    a.smem_cap = c.factor_slice;
    a.trace = c.trace ? c.trace + 6 * (int64_t)c.sym.nsuper : nullptr;
    cudaMemsetAsync(c.fac_count, 0, sizeof(int32_t) * c.sym.nsuper, c.stream);
    cudaMemsetAsync(c.sn_maxd, 0, sizeof(double) * c.sym.nsuper, c.stream);
    cudaMemsetAsync(c.tickets, 0, sizeof(int32_t) * 4, c.stream);
    cudaMemsetAsync(c.bumps, 0, sizeof(int32_t), c.stream);
    int e0 = 0;
    if (c.profile) {
        e0 = (int)(2 * (c.ev_factor.size() + c.ev_solve.size()));
        cudaEventRecord(pooled_event(c, e0), c.stream);
    }
    const int n_warp = c.host_sym.n_warp, n_main = c.host_sym.n_main;
    if (n_warp > 0) {
        a.t_begin = 0;
        a.nsuper = n_warp;
        a.ticket = c.tickets;
        a.smem_cap = c.factor_slice;
        factor_kernel<T><<<c.factor_blocks, FW * 32, c.factor_smem, c.stream>>>(a, (T*)c.lval, (T*)c.dvec,
                                                                                (T*)c.inbox);
        c.launches++;
    }
    if (n_main > n_warp) {
        a.t_begin = n_warp;
        a.nsuper = n_main;
        a.ticket = c.tickets + 3;
        a.smem_cap = c.factor_cta_smem / (int64_t)sizeof(T);
        factor_cta_kernel<T><<<c.factor_cta_blocks, 256, c.factor_cta_smem, c.stream>>>(a, (T*)c.lval, (T*)c.dvec,
                                                                                       (T*)c.inbox);
        c.launches++;
    }
    k_tail_factor(c);
    if (c.profile) {
        cudaEventRecord(pooled_event(c, e0 + 1), c.stream);
        c.ev_factor.emplace_back(e0, e0 + 1);
    }
    return CIPM_OK;
}

template <typename T>
void refine_solve_t(Ctx& c, int act0, int act1) {
    T* t = (T*)c.rt;
    gather_perm<T><<<grid_for(c.dim), kThreads, 0, c.stream>>>(c.rr, t, c.sym.perm, c.dim, act0, act1);
    cudaMemsetAsync(c.fac_count, 0, sizeof(int32_t) * c.sym.nsuper, c.stream);
    cudaMemsetAsync(c.bwd_done, 0, sizeof(int32_t) * c.sym.nsuper, c.stream);
    cudaMemsetAsync(c.tickets, 0, sizeof(int32_t) * 4, c.stream);
    if (c.tflag_total) cudaMemsetAsync(c.tflags, 0, sizeof(int32_t) * c.tflag_total, c.stream);
    int e0 = 0;
    if (c.profile) {
        e0 = (int)(2 * (c.ev_factor.size() + c.ev_solve.size()));
        cudaEventRecord(pooled_event(c, e0), c.stream);
    }
    SolveArgs f = solve_args(c, c.fac_count, c.tickets + 1, act0, act1);
    f.trace = c.trace;
    const size_t ssm = sizeof(T) * (size_t)c.solve_slice * SW;
    if (f.nsuper > 0) forward_kernel<T><<<c.solve_blocks, SW * 32, ssm, c.stream>>>(f, (const T*)c.lval, t, (T*)c.vin);
    k_tail_forward(c, t, act0, act1);
    k_tail_backward(c, t, act0, act1);
    SolveArgs b = solve_args(c, c.bwd_done, c.tickets + 2, act0, act1);
    if (b.nsuper > 0)
        backward_kernel<T><<<c.solve_blocks, SW * 32, ssm, c.stream>>>(b, (const T*)c.lval, (const T*)c.dvec, t);
    if (c.profile) {
        cudaEventRecord(pooled_event(c, e0 + 1), c.stream);
        c.ev_solve.emplace_back(e0, e0 + 1);
    }
    scatter_add_perm<T><<<grid_for(c.dim), kThreads, 0, c.stream>>>(c.rx, t, c.sym.perm, c.dim, act0, act1);
    c.launches += 4;
}

}  // namespace

void k_build_base(Ctx& c) {
    if (c.precision == CIPM_FULL) build_base_t<double>(c);
    else build_base_t<float>(c);
}

void k_assemble(Ctx& c) {
    const size_t es = c.precision == CIPM_FULL ? sizeof(double) : sizeof(float);
    cudaMemcpyAsync(c.lval, c.lbase, es * c.sym.nnz_storage, cudaMemcpyDeviceToDevice, c.stream);
    k_scatter_h(c);
}

int k_factor(Ctx& c) {
    return c.precision == CIPM_FULL ? factor_t<double>(c) : factor_t<float>(c);
}

// one refinement correction: x += solve(r) for the active right-hand sides
void k_refine_step(Ctx& c, int nrhs, const int* active) {
    const int a0 = active[0], a1 = nrhs > 1 ? active[1] : 0;
    if (c.profile) c.solve_rhs += a0 + a1;
    if (c.precision == CIPM_FULL) refine_solve_t<double>(c, a0, a1);
    else refine_solve_t<float>(c, a0, a1);
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
    int64_t slice = std::min<int64_t>(c.host_sym.max_panel_warp, 6144 / es);
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
    // per-warp panel slice: 6 KiB (four 8-warp CTAs per SM); larger panels are read from L2/HBM
    const int64_t es = c.precision == CIPM_FULL ? 8 : 4;
    c.solve_slice = std::max<int64_t>(64, std::min<int64_t>((c.host_sym.max_panel_main + 3) & ~int64_t(3), 6144 / es));
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
    int64_t g = (int64_t)sm_count() * per;
    int64_t need = (c.host_sym.n_main + SW - 1) / SW;
    if (g > need) g = need;
    if (const char* e = getenv("CIPM_SOLVE_BLOCKS")) g = std::min<int64_t>(g, atoll(e));     // experiments
    return (int)(g < 1 ? 1 : g);
}

}  // namespace cipm
