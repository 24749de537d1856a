// Microbenchmark: one tail_diag launch (64 x 64 diagonal block LDL' + inverse)
// on a synthetic quasi-definite block, with the kernel's phase timestamps
// (CIPM_DIAG_TS).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -DCIPM_DIAG_TS tools/micro/diag_bench.cu -o tools/micro/diag_bench
//   -Lpaper_2412_19027_b200/lib -lcipm   (links the other translation units)
#define CIPM_DIAG_TS 1
#include "../../paper_2412_19027_b200/csrc/dense.cu"
using namespace cipm;
#include <vector>
#include <random>

template <typename T>
void run(const char* tag, int nthr) {
    const int r = 64, nb = 64;
    std::vector<T> h(r * r, (T)0);
    std::mt19937 g(1);
    std::uniform_real_distribution<double> u(-1, 1);
    for (int j = 0; j < nb; ++j)
        for (int i = j; i < r; ++i) h[j * r + i] = (T)(i == j ? (j % 3 ? 8.0 : -8.0) : 0.1 * u(g));
    std::vector<int8_t> sg(nb);
    for (int j = 0; j < nb; ++j) sg[j] = j % 3 ? 1 : -1;
    T *L, *Lsrc, *D, *inv;
    int8_t* sign;
    double* maxd;
    int32_t* bumps;
    int* err;
    cudaMalloc(&L, sizeof(T) * r * r);
    cudaMalloc(&Lsrc, sizeof(T) * r * r);
    cudaMalloc(&D, sizeof(T) * nb);
    cudaMalloc(&inv, sizeof(T) * 2 * TB * TB);
    cudaMalloc(&sign, nb);
    cudaMalloc(&maxd, sizeof(double));
    cudaMalloc(&bumps, 4);
    cudaMalloc(&err, 4);
    cudaMemcpy(Lsrc, h.data(), sizeof(T) * r * r, cudaMemcpyHostToDevice);
    cudaMemcpy(sign, sg.data(), nb, cudaMemcpyHostToDevice);
    cudaMemset(maxd, 0, 8);
    cudaMemset(bumps, 0, 4);
    cudaMemset(err, 0, 4);
    cudaFuncSetAttribute(tail_diag<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, diag_smem<T>());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 20; ++rep) {
        cudaMemcpy(L, Lsrc, sizeof(T) * r * r, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        tail_diag<T><<<1, nthr, diag_smem<T>()>>>(L, r, 0, nb, 0, D, sign, maxd, bumps, err, 1e-8, 0.0, inv, inv + TB * TB);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    long long ts[64];
    cudaMemcpyFromSymbol(ts, g_diag_ts, sizeof(ts));
    printf("%s x%d: best %.1f us (event); phases (cycles from start):", tag, nthr, best * 1000.f);
    const int keys[] = {1, 2, 3, 4, 6, 7, 8, 10, 11, 12, 14, 15, 16, 18, 19, 20};
    for (int k : keys) printf(" %d:%lld", k, ts[k] - ts[0]);
    printf("  err %s\n", cudaGetErrorString(cudaGetLastError()));
}

int main() {
    for (int nt : {256, 128, 64}) run<double>("fp64", nt);
    run<float>("fp32", 256);
    return 0;
}
