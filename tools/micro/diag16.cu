// Microbenchmark: latency of the 16 x 16 diagonal sub-block LDL' (the serial
// pivot chain of tail_diag) in several formulations, clock64 inside one warp.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_19027_b200/csrc/dense.cu"

namespace mb {
constexpr int SB = 16, TB = 64;

// V0: registers, lane i owns row i, shuffles (tail_diag's formulation)
template <typename T>
__device__ void v0(T* Sk, int k0, int nbk, const int8_t* sSg, double delta_s, double delta_d, double& runmax, T* sD,
                   T* sInv) {
    const int lane = threadIdx.x & 31;
    T x[SB];
#pragma unroll
    for (int c = 0; c < SB; ++c) x[c] = (lane < nbk && c <= lane) ? Sk[c * TB + k0 + lane] : (T)0;
#pragma unroll
    for (int j = 0; j < SB; ++j) {
        if (j < nbk) {
            double dd = (double)__shfl_sync(0xffffffffu, x[j], j);
            const double bound = delta_s + delta_d * runmax;
            const bool bump = fabs(dd) < bound;
            if (bump) dd = sSg[k0 + j] > 0 ? bound : -bound;
            const T dt = (T)dd;
            runmax = fmax(runmax, fabs(dd));
            const T inv = (T)1 / dt;
            if (lane == 0) { sD[k0 + j] = dt; sInv[j] = inv; }
            const T xj = x[j];
#pragma unroll
            for (int c = j + 1; c < SB; ++c) {
                const T acj = __shfl_sync(0xffffffffu, xj, c);
                if (lane >= c) x[c] -= xj * (acj * inv);
            }
            x[j] = lane > j ? xj * inv : (lane == j ? (T)1 : x[j]);
        }
    }
#pragma unroll
    for (int c = 0; c < SB; ++c)
        if (lane < nbk && c <= lane) Sk[c * TB + k0 + lane] = x[c];
}

// V1: shared memory, rolled pivot loop, lane i updates row i (no big unrolled body)
template <typename T>
__device__ void v1(T* Sk, int k0, int nbk, const int8_t* sSg, double delta_s, double delta_d, double& runmax, T* sD,
                   T* sInv) {
    const int lane = threadIdx.x & 31;
    const int i = k0 + lane;
#pragma unroll 1
    for (int j = 0; j < nbk; ++j) {
        T* colj = Sk + j * TB;
        double dd = (double)colj[k0 + j];
        const double bound = delta_s + delta_d * runmax;
        const bool bump = fabs(dd) < bound;
        if (bump) dd = sSg[k0 + j] > 0 ? bound : -bound;
        const T dt = (T)dd;
        runmax = fmax(runmax, fabs(dd));
        const T inv = (T)1 / dt;
        const T lij = (lane > j && lane < nbk) ? colj[i] : (T)0;    // unscaled a_ij
        // a_ic -= a_ij a_cj / d  for c in (j, i]
#pragma unroll 4
        for (int c = j + 1; c < nbk; ++c) {
            const T acj = colj[k0 + c];
            if (lane >= c && lane < nbk) Sk[c * TB + i] -= lij * (acj * inv);
        }
        __syncwarp();
        if (lane > j && lane < nbk) colj[i] = lij * inv;
        if (lane == 0) { sD[k0 + j] = dt; sInv[j] = inv; colj[k0 + j] = (T)1; }
        __syncwarp();
    }
}

// V2: registers, but the pivot row broadcast from shared memory instead of 15 shuffles:
// lane j publishes its row after step j-1; lanes read a_cj for all c from smem
template <typename T>
__device__ void v2(T* Sk, int k0, int nbk, const int8_t* sSg, double delta_s, double delta_d, double& runmax, T* sD,
                   T* sInv, T* colbuf) {
    const int lane = threadIdx.x & 31;
    T x[SB];
#pragma unroll
    for (int c = 0; c < SB; ++c) x[c] = (lane < nbk && c <= lane) ? Sk[c * TB + k0 + lane] : (T)0;
#pragma unroll
    for (int j = 0; j < SB; ++j) {
        if (j < nbk) {
            // column j of every row into smem (lanes > j hold a_lane,j)
            colbuf[(j & 1) * 32 + lane] = x[j];
            __syncwarp();
            double dd = (double)colbuf[(j & 1) * 32 + j];
            const double bound = delta_s + delta_d * runmax;
            const bool bump = fabs(dd) < bound;
            if (bump) dd = sSg[k0 + j] > 0 ? bound : -bound;
            const T dt = (T)dd;
            runmax = fmax(runmax, fabs(dd));
            const T inv = (T)1 / dt;
            if (lane == 0) { sD[k0 + j] = dt; sInv[j] = inv; }
            const T xj = x[j] * inv;
#pragma unroll
            for (int c = j + 1; c < SB; ++c) {
                const T acj = colbuf[(j & 1) * 32 + c];
                if (lane >= c) x[c] -= xj * acj;
            }
            x[j] = lane > j ? xj : (lane == j ? (T)1 : x[j]);
        }
    }
#pragma unroll
    for (int c = 0; c < SB; ++c)
        if (lane < nbk && c <= lane) Sk[c * TB + k0 + lane] = x[c];
}

}  // namespace mb
using namespace mb;

__device__ double g_ds = 1e-8, g_dd = 0.0;
__device__ int g_err[1];
__device__ int32_t g_bumps[1];
__device__ double g_dvec_d[64];
template <typename T> __device__ T* dv();
template <> __device__ double* dv<double>() { return g_dvec_d; }
__device__ float g_dvec_f[64];
template <> __device__ float* dv<float>() { return g_dvec_f; }

template <typename T, int V>
__global__ void bench(const T* src, T* dst, long long* cyc) {
    T* g_dvec = dv<T>();
#ifdef DYN_S
    extern __shared__ __align__(16) unsigned char dyn_raw[];
    T* S = reinterpret_cast<T*>(dyn_raw);
#else
    __shared__ T S[TB * TB];
#endif
    __shared__ T sD[TB], sInv[SB], colbuf[64];
    __shared__ int8_t sSg[TB];
    __shared__ T sLt[SB * SB];
    __shared__ double s_rm;
    if (threadIdx.x == 0) s_rm = 0.0;
    for (int i = threadIdx.x; i < TB * TB; i += blockDim.x) S[i] = src[i];
    if (threadIdx.x < TB) sSg[threadIdx.x] = threadIdx.x % 3 ? 1 : -1;
    __syncthreads();
    if (V == 5) {
        // V4 + warp 0 runs an unrelated 4 KB+ unrolled code block between sub-blocks
        // (as tail_diag's (b)/(c) phases do): does the pivot chain slow down?
        long long acc = 0;
        double junk = threadIdx.x;
        for (int k0 = 0; k0 < TB; k0 += SB) {
            const long long ta = clock64();
            if ((threadIdx.x >> 5) == 0)
                cipm::diag_sub<T, true>(S + k0 * TB, k0, SB, sSg, colbuf, g_ds, g_dd, &s_rm, sD, sInv, g_dvec, 0, 0, g_err, g_bumps, sLt);
            __syncwarp();
            acc += clock64() - ta;
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 400; ++u) junk = junk * 1.0000001 + (double)(u & 7) * S[(u * 7 + threadIdx.x) & 4095];
            __syncthreads();
        }
        if (threadIdx.x == 0) cyc[0] = acc;            // the diagonal sub-blocks only
        if (junk == 12345.678) dst[0] = junk;
        for (int i = threadIdx.x; i < TB * TB; i += blockDim.x) dst[i] = S[i];
        return;
    }
    if (V == 4) {
        // tail_diag's context: warp 0 inside a divergent branch, the others at a barrier
        long long t0 = clock64();
        for (int k0 = 0; k0 < TB; k0 += SB) {
            if ((threadIdx.x >> 5) == 0)
                cipm::diag_sub<T, true>(S + k0 * TB, k0, SB, sSg, colbuf, g_ds, g_dd, &s_rm, sD, sInv, g_dvec, 0, 0, g_err, g_bumps, sLt);
            __syncthreads();
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[0] = t1 - t0;
        for (int i = threadIdx.x; i < TB * TB; i += blockDim.x) dst[i] = S[i];
        return;
    }
    if (threadIdx.x >= 32) return;
    double runmax = 0.0;
    long long t0 = clock64();
    for (int k0 = 0; k0 < TB; k0 += SB) {
        T* Sk = S + k0 * TB;
        if (V == 0) v0<T>(Sk, k0, SB, sSg, 1e-8, 0.0, runmax, sD, sInv);
        if (V == 1) v1<T>(Sk, k0, SB, sSg, 1e-8, 0.0, runmax, sD, sInv);
        if (V == 2) v2<T>(Sk, k0, SB, sSg, 1e-8, 0.0, runmax, sD, sInv, colbuf);
        if (V == 3) cipm::diag_sub<T, true>(Sk, k0, SB, sSg, colbuf, g_ds, g_dd, &s_rm, sD, sInv, g_dvec, 0, 0, g_err, g_bumps, sLt);
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    for (int i = threadIdx.x; i < TB * TB; i += 32) dst[i] = S[i];
}

template <typename T, int V>
void run(const char* tag, const T* src, T* dst, long long* cyc) {
    long long best = 1LL << 60;
    for (int rep = 0; rep < 5; ++rep) {
        #ifdef DYN_S
        cudaFuncSetAttribute(bench<T, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(T) * TB * TB));
        bench<T, V><<<1, V >= 4 ? 256 : 64, sizeof(T) * TB * TB>>>(src, dst, cyc);
#else
        bench<T, V><<<1, V >= 4 ? 256 : 64>>>(src, dst, cyc);
#endif
        long long h;
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (h < best) best = h;
    }
    T out[TB * TB];
    cudaMemcpy(out, dst, sizeof(out), cudaMemcpyDeviceToHost);
    double cs = 0;
    for (int i = 0; i < TB * TB; ++i) cs += (double)out[i] * ((i % 7) + 1);
    printf("%s V%d: %lld cycles for 4 sub-blocks (%.0f per column)  checksum %.12g  %s\n", tag, V, best, best / 64.0, cs,
           cudaGetErrorString(cudaGetLastError()));
}

template <typename T>
void all(const char* tag) {
    T h[TB * TB];
    for (int j = 0; j < TB; ++j)
        for (int i = 0; i < TB; ++i) h[j * TB + i] = (T)(i == j ? (j % 3 ? 8.0 : -8.0) : (i > j ? 0.01 * ((i * 7 + j * 3) % 11 - 5) : 0.0));
    T *src, *dst;
    long long* cyc;
    cudaMalloc(&src, sizeof(h));
    cudaMalloc(&dst, sizeof(h));
    cudaMalloc(&cyc, 8);
    cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
    run<T, 0>(tag, src, dst, cyc);
    run<T, 1>(tag, src, dst, cyc);
    run<T, 2>(tag, src, dst, cyc);
    run<T, 3>(tag, src, dst, cyc);
    run<T, 4>(tag, src, dst, cyc);
    run<T, 5>(tag, src, dst, cyc);
}

int main() {
    all<double>("fp64");
    all<float>("fp32");
    return 0;
}
