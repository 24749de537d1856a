// Shared device-side definitions for libcipm (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <type_traits>
#include <cstdint>
#include <cstdio>

#include <nvtx3/nvToolsExt.h>

#include "../../include/cipm.h"

namespace cipm {

// NVTX range around a C-ABI entry point (header-only NVTX v3: no library to
// link; a no-op unless a profiler injects itself).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define CIPM_NVTX(name) ::cipm::NvtxRange nvtx_range__(name)

constexpr int kThreads = 256;
constexpr int kMaxRedBlocks = 1184;     // 148 SMs x 8 — fixed grid => deterministic reductions
constexpr double kMinStep = 1e-11;

#define CIPM_CUDA(call)                                                              \
    do {                                                                             \
        cudaError_t e__ = (call);                                                    \
        if (e__ != cudaSuccess) {                                                    \
            fprintf(stderr, "[cipm] CUDA error %s at %s:%d: %s\n", #call, __FILE__, \
                    __LINE__, cudaGetErrorString(e__));                              \
            return CIPM_E_CUDA;                                                      \
        }                                                                            \
    } while (0)

// ---------------------------------------------------------------------------
// device scalar block: every per-iteration scalar lives here (no host round
// trip unless the host needs a decision).  Field order is part of the ABI of
// cipm_read_scalars() (see include/cipm.h CIPM_SC_*).
// ---------------------------------------------------------------------------
struct Scalars {
    double v[CIPM_SC_COUNT];
};

// ordered min on non-negative doubles (bit pattern is monotone)
__device__ __forceinline__ void atomic_min_pos(double* addr, double val) {
    if (!(val >= 0.0)) val = 0.0;   // NaN / negative -> 0 (forces StepTooSmall)
    atomicMin(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(val));
}

__device__ __forceinline__ void set_error(int* err, int code) { atomicCAS(err, 0, code); }

// a pivot column published in shared memory (16-byte aligned), read back as one
// burst of 16-byte broadcast loads (N a multiple of 16 / sizeof(T))
template <typename T, int N>
__device__ __forceinline__ void load_col(T (&cc)[N], const T* col) {
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    constexpr int VW = 16 / (int)sizeof(T);
    static_assert(N % VW == 0, "column length");
#pragma unroll
    for (int c = 0; c < N; c += VW) *reinterpret_cast<V*>(&cc[c]) = *reinterpret_cast<const V*>(col + c);
}

// Dependency flags between CTAs/warps of one persistent launch.  Poll with a
// relaxed load (no per-poll L1 invalidation — ld.acquire compiles to
// LDG.STRONG + CCTL.IVALL, which thrashes the SM's L1 for every other warp),
// then order the following reads with one fence.  Data produced by other CTAs
// is read with ld.cg (L2) anyway.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void wait_ge(const int* p, int need) {
    if (ld_relaxed(p) < need) {
        do {
            __nanosleep(32);
        } while (ld_relaxed(p) < need);
    }
    fence_acq_rel_gpu();
}

// counter increment that publishes this thread's (and, after a warp/CTA barrier,
// its group's) earlier writes and acquires the writes published by earlier
// increments — one RMW instead of fence + atomic + fence
__device__ __forceinline__ int atomic_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// ---------------------------------------------------------------------------
// TMA 1-D bulk copies (cp.async.bulk global -> shared, completion on an
// mbarrier): one instruction stages a whole supernode panel.  Addresses and
// sizes must be 16-byte aligned (panel offsets are padded in symbolic.cpp).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// elected lane: arm the barrier with the byte count and issue the bulk copy
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

// generic-proxy reads of a shared buffer must be ordered before the next async-proxy write to it
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// deterministic multi-value reduction: each block writes K partials, the last
// block to arrive combines them in block order (fixed grid => bitwise
// reproducible), then calls the finaliser.
// ---------------------------------------------------------------------------
enum RedOp { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

template <int K>
struct RedSpec {
    int op[K];
};

__device__ __forceinline__ double red_apply(int op, double a, double b) {
    if (op == RED_SUM) return a + b;
    if (op == RED_MAX) return fmax(a, b);
    return fmin(a, b);
}

__device__ __forceinline__ double red_identity(int op) {
    if (op == RED_SUM) return 0.0;
    if (op == RED_MAX) return -INFINITY;
    return INFINITY;
}

// block reduce K values held per thread into lane 0 of warp 0; returns true on thread 0
template <int K>
__device__ __forceinline__ void block_reduce(double (&vals)[K], const int (&ops)[K], double* smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double v = vals[k];
        for (int o = 16; o > 0; o >>= 1) v = red_apply(ops[k], v, __shfl_down_sync(0xffffffffu, v, o));
        if (lane == 0) smem[warp * K + k] = v;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double v = lane < nw ? smem[lane * K + k] : red_identity(ops[k]);
            for (int o = 16; o > 0; o >>= 1) v = red_apply(ops[k], v, __shfl_down_sync(0xffffffffu, v, o));
            vals[k] = v;
        }
    }
    __syncthreads();
}

// Write block partials; the last block combines.  Returns true (on thread 0 of
// the last block) with `out` holding the grid-wide result.
template <int K>
__device__ bool grid_reduce(double (&vals)[K], const int (&ops)[K], double* partials,
                            unsigned int* counter, double (&out)[K]) {
    __shared__ double smem[32 * K];
    __shared__ bool last;
    block_reduce<K>(vals, ops, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) partials[blockIdx.x * K + k] = vals[k];
        __threadfence();
        unsigned int t = atomicAdd(counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    // last block: thread t folds blocks t, t+nt, ... (fixed order), then a fixed tree
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double acc = red_identity(ops[k]);
        for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
            acc = red_apply(ops[k], acc, __ldcg(partials + b * K + k));
        vals[k] = acc;
    }
    block_reduce<K>(vals, ops, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = vals[k];
        *counter = 0u;
        return true;
    }
    return false;
}

inline int red_grid(int64_t n) {
    int64_t b = (n + kThreads - 1) / kThreads;
    if (b < 1) b = 1;
    if (b > kMaxRedBlocks) b = kMaxRedBlocks;
    return (int)b;
}

// grid of a grid-stride reduction kernel: at most ONE wave of the kernel's resident
// blocks (occupancy API, cached per kernel).  For the division-heavy neighbourhood
// candidates over nonneg rows (16 sums, 86 registers, 1184 blocks = 4 waves) fewer
// block reductions and partials win (C2: 42 -> 20 us); memory-bound passes — the
// thread-per-row SpMVs (kkt_resid2, resid_n), the same candidates over mostly
// cone rows (C5a: -7 % per solve) — measured slower with it and keep the plain grid.
// Fixed per kernel and device, so the reductions stay deterministic.
int occupancy_blocks(const void* kernel, int threads);   // blocks per SM x SMs (capi.cu)
template <typename K>
inline int red_grid(int64_t n, K* kernel) {
    int64_t b = (n + kThreads - 1) / kThreads;
    const int wave = occupancy_blocks(reinterpret_cast<const void*>(kernel), kThreads);
    if (b > wave) b = wave;
    if (b < 1) b = 1;
    if (b > kMaxRedBlocks) b = kMaxRedBlocks;
    return (int)b;
}

inline int grid_for(int64_t n, int threads = kThreads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > (1 << 30)) b = 1 << 30;
    return (int)b;
}

}  // namespace cipm
