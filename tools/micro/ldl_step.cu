// Microbenchmark: latency of one CTA-tier panel LDL' (w=28, r=56, FP32) with
// several implementations, timed with clock64 inside a single CTA (no contention).
#include <cstdio>
#include <cuda_runtime.h>

template <int NB, int MODE>
__device__ __forceinline__ void ldl_regs(float* P, int r, int w, float* sD, float (*scol)[NB + 1], double ds, double dd_) {
    const int tid = threadIdx.x, lane = tid & 31;
    const bool have = tid < r;
    double runmax = 0.0;
    float x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = (c < w && have) ? P[c * r + tid] : 0.f;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        if (j < w) {
            float* col = scol[j & 1];
            if (tid < 32) {
                float inv;
                if (MODE == 0) {
                    double dd = (double)__shfl_sync(0xffffffffu, x[j], j);
                    const double bound = ds + dd_ * runmax;
                    if (fabs(dd) < bound) dd = bound;
                    const float dt = (float)dd;
                    runmax = fmax(runmax, fabs(dd));
                    inv = 1.f / dt;
                    if (lane == 0) { sD[j] = dt; col[NB] = inv; }
                } else {
                    const float dt = __shfl_sync(0xffffffffu, x[j], j);
                    inv = __frcp_rn(dt);
                    if (lane == 0) { sD[j] = dt; col[NB] = inv; }
                }
                if (lane > j && lane < w) col[lane] = x[j] * inv;
            }
            asm volatile("bar.sync 1, 64;" ::: "memory");
            const float inv = col[NB];
            const float aij = x[j];
#pragma unroll
            for (int c = j + 1; c < NB; ++c)
                if (c < w) x[c] -= aij * col[c];
            x[j] = tid > j ? aij * inv : (tid == j ? 1.f : aij);
        }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
        if (c < w && have && tid >= c) P[c * r + tid] = x[c];
}

template <int MODE>
__global__ void k(const float* src, float* dst, long long* cyc, int r, int w, int reps) {
    __shared__ float P[64 * 32];
    __shared__ float sD[32];
    __shared__ float scol[2][33];
    long long best = 1LL << 60;
    for (int rep = 0; rep < reps; ++rep) {
        for (int i = threadIdx.x; i < r * w; i += blockDim.x) P[i] = src[i];
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < 64) ldl_regs<32, MODE>(P, r, w, sD, scol, 1e-8, 1e-30);
        __syncthreads();
        long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    for (int i = threadIdx.x; i < r * w; i += blockDim.x) dst[i] = P[i];
    if (threadIdx.x == 0) *cyc = best;
}


template <int NB>
__device__ __forceinline__ void rot_ldl(float* P, int r, int w, float* sD, float (*scol)[2 * NB + 1], double ds, double dd_) {
    const int tid = threadIdx.x, lane = tid & 31;
    const bool two = r > 32;
    const bool have = tid < r;
    double runmax = 0.0;
    float x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = (c < w && have) ? P[c * r + tid] : 0.f;
    if (tid < 2 * NB + 1) { scol[0][tid] = 0.f; scol[1][tid] = 0.f; }
    asm volatile("bar.sync 1, 64;" ::: "memory");
#pragma unroll 1
    for (int j = 0; j < w; ++j) {
        float* col = scol[j & 1];
        if (tid < 32) {
            double dd = (double)__shfl_sync(0xffffffffu, x[0], j);
            const double bound = ds + dd_ * runmax;
            if (fabs(dd) < bound) dd = bound;
            const float dt = (float)dd;
            runmax = fmax(runmax, fabs(dd));
            const float inv = 1.f / dt;
            if (lane == 0) { sD[j] = dt; col[2 * NB] = inv; }
            if (lane > j && lane < w) col[lane - j] = x[0] * inv;
            if (lane >= w - j && lane < NB) col[lane] = 0.f;
        }
        asm volatile("bar.sync 1, 64;" ::: "memory");
        const float inv = col[2 * NB];
        const float aij = x[0];
        if (have && tid >= j) P[j * r + tid] = tid > j ? aij * inv : 1.f;
#pragma unroll
        for (int c = 1; c < NB; ++c) x[c - 1] = x[c] - aij * col[c];
        x[NB - 1] = 0.f;
    }
}

__global__ void krot(const float* src, float* dst, long long* cyc, int r, int w, int reps) {
    __shared__ float P[64 * 32];
    __shared__ float sD[32];
    __shared__ float scol[2][65];
    long long best = 1LL << 60;
    for (int rep = 0; rep < reps; ++rep) {
        for (int i = threadIdx.x; i < r * w; i += blockDim.x) P[i] = src[i];
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < 64) rot_ldl<32>(P, r, w, sD, scol, 1e-8, 1e-30);
        __syncthreads();
        long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
    }
    for (int i = threadIdx.x; i < r * w; i += blockDim.x) dst[i] = P[i];
    if (threadIdx.x == 0) *cyc = best;
}

int main() {
    const int r = 56, w = 28;
    float h[64 * 32];
    for (int c = 0; c < w; ++c)
        for (int i = 0; i < r; ++i) h[c * r + i] = (i == c) ? 10.f + i : 0.01f * ((i * 7 + c * 3) % 11 - 5);
    float *src, *dst;
    long long* cyc;
    cudaMalloc(&src, sizeof(h)); cudaMalloc(&dst, sizeof(h)); cudaMalloc(&cyc, 8);
    cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
    long long c0 = 0, c1 = 0;
    k<0><<<1, 256>>>(src, dst, cyc, r, w, 20); cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    k<1><<<1, 256>>>(src, dst, cyc, r, w, 20); cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
    long long c2 = 0;
    krot<<<1, 256>>>(src, dst, cyc, r, w, 20); cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
    printf("rotated: %lld cycles (%.2f per step)\n", c2, c2 / (double)w);
    printf("ldl w=%d r=%d: full %lld cycles (%.2f per step), no-fp64/rcp %lld cycles (%.2f per step) err=%s\n", w, r, c0,
           c0 / (double)w, c1, c1 / (double)w, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
