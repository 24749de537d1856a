// Problem-value setup on the device: cone reordering of A/b and Ruiz
// equilibration (reference problem.py:177-284), so a parametric re-solve
// (Solver.update_data, ipm.py:187-221) ships only the user's raw arrays to the
// GPU.  Every operation is the reference's elementwise IEEE operation in the
// reference's order (max-abs norms are order independent; 1/sqrt, clip, the
// two-factor products (c_i * v) * c_j) and the file is built with FMA
// contraction off, so D_r, D_c, c and the scaled values are bitwise the host
// routine's (tests/test_gpu_kernels.py checks this).
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"

namespace cipm {

namespace {

constexpr double kScaleMin = 1e-4, kScaleMax = 1e4;   // problem.py:36-40
constexpr int kRuizIters = 10;                        // RUIZ_ITERS, problem.py:36

__global__ void gather_reorder(const double* __restrict__ a_user, const int64_t* __restrict__ a_src,
                               double* __restrict__ a_v, int64_t nnz, const double* __restrict__ b_user,
                               const int64_t* __restrict__ b_src, double* __restrict__ b, int64_t m) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nnz) a_v[i] = a_user[a_src[i]];
    if (i < m) b[i] = b_user[b_src[i]];
}

__global__ void set_ones(double* a, int64_t n, double* b, int64_t m) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = 1.0;
    if (i < m) b[i] = 1.0;
}

// column norms (P is symmetric: column j of P = row j; A columns via the A' CSR)
// and row norms of A
__global__ void ruiz_norms(int64_t n, int64_t m, const int64_t* __restrict__ prp, const double* __restrict__ pv,
                           const int64_t* __restrict__ atrp, const int64_t* __restrict__ at_src,
                           const int64_t* __restrict__ arp, const double* __restrict__ av, double* cnorm,
                           double* rnorm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double c = 0.0;
        for (int64_t p = prp[i]; p < prp[i + 1]; ++p) c = fmax(c, fabs(pv[p]));
        for (int64_t p = atrp[i]; p < atrp[i + 1]; ++p) c = fmax(c, fabs(av[at_src[p]]));
        cnorm[i] = c;
    } else if (i < n + m) {
        const int64_t r = i - n;
        double c = 0.0;
        for (int64_t p = arp[r]; p < arp[r + 1]; ++p) c = fmax(c, fabs(av[p]));
        rnorm[r] = c;
    }
}

// block-uniform row scaling over every SOC / exp / pow / PSD block
__global__ void ruiz_blocks(double* rnorm, const int32_t* __restrict__ boff, const int32_t* __restrict__ bdim,
                            int64_t nb) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nb) return;
    const int o = boff[k], d = bdim[k];
    double mx = 0.0;
    for (int i = 0; i < d; ++i) mx = fmax(mx, rnorm[o + i]);
    for (int i = 0; i < d; ++i) rnorm[o + i] = mx;
}

__device__ __forceinline__ double clipd(double v) { return fmin(fmax(v, kScaleMin), kScaleMax); }

__global__ void ruiz_steps(int64_t n, int64_t m, const double* __restrict__ cnorm, const double* __restrict__ rnorm,
                           double* dcol, double* drow, double* cstep, double* rstep) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const double c = cnorm[i];
        const double st = c > 0.0 ? 1.0 / sqrt(c) : 1.0;
        const double nd = clipd(dcol[i] * st);
        cstep[i] = nd / dcol[i];
        dcol[i] = nd;
    } else if (i < n + m) {
        const int64_t r = i - n;
        const double c = rnorm[r];
        const double st = c > 0.0 ? 1.0 / sqrt(c) : 1.0;
        const double nd = clipd(drow[r] * st);
        rstep[r] = nd / drow[r];
        drow[r] = nd;
    }
}

__global__ void ruiz_scale(int64_t n, int64_t m, const int64_t* __restrict__ prp, const int64_t* __restrict__ pci,
                           double* pv, const int64_t* __restrict__ arp, const int64_t* __restrict__ aci, double* av,
                           double* q, double* b, const double* __restrict__ cstep,
                           const double* __restrict__ rstep) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const double ci = cstep[i];
        for (int64_t p = prp[i]; p < prp[i + 1]; ++p) pv[p] = (ci * pv[p]) * cstep[pci[p]];
        q[i] *= ci;
    } else if (i < n + m) {
        const int64_t r = i - n;
        const double ri = rstep[r];
        for (int64_t p = arp[r]; p < arp[r + 1]; ++p) av[p] = (ri * av[p]) * cstep[aci[p]];
        b[r] *= ri;
    }
}

__global__ void qmax_kernel(const double* q, int64_t n, double* out, double* partials, unsigned int* counter) {
    double v[1] = {0.0};
    const int ops[1] = {RED_MAX};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[0] = fmax(v[0], fabs(q[i]));
    double res[1];
    if (grid_reduce<1>(v, ops, partials, counter, res)) {
        const double qmax = n ? res[0] : 0.0;
        *out = qmax == 0.0 ? 1.0 : clipd(1.0 / qmax);
    }
}

__global__ void cost_scale(double* pv, int64_t nnzp, double* q, int64_t n, const double* cobj) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double c = *cobj;
    if (i < nnzp) pv[i] = pv[i] * c;
    if (i < n) q[i] = q[i] * c;
}

// q / b through the recorded Ruiz passes: the same per-pass products q_i *= c_i^(k),
// b_r *= r_r^(k) in the same order as ruiz_scale, so bitwise the full run's q, b
__global__ void ruiz_replay(int64_t n, int64_t m, double* q, double* b, const double* __restrict__ csteps,
                            const double* __restrict__ rsteps, int iters) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double v = q[i];
        for (int k = 0; k < iters; ++k) v *= csteps[(int64_t)k * n + i];
        q[i] = v;
    } else if (i < n + m) {
        const int64_t r = i - n;
        double v = b[r];
        for (int k = 0; k < iters; ++k) v *= rsteps[(int64_t)k * m + r];
        b[r] = v;
    }
}

__global__ void transpose_vals(const double* __restrict__ av, const int64_t* __restrict__ at_src,
                               double* __restrict__ at_v, int64_t nnz) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nnz) at_v[t] = av[at_src[t]];
}

}  // namespace

// raw user-order values -> reordered, equilibrated device problem (+ factor base image)
int k_set_problem(Ctx& c, bool equilibrate, bool replay) {
    const int64_t n = c.n, m = c.m, nb = std::max<int64_t>(c.a_nnz, m);
    if (replay) {
        // q / b changed, P / A raw values did not: D_r, D_c, the Ruiz-scaled P, A and A'
        // are the previous run's (the passes depend on P and A only, problem.py:232-260);
        // replay the recorded per-pass steps on the fresh q / b, then the cost scaling
        gather_reorder<<<grid_for(std::max<int64_t>(m, 1)), kThreads, 0, c.stream>>>(c.a_user, c.a_src, c.a_v, 0,
                                                                                     c.b_user, c.b_src, c.b, m);
        ruiz_replay<<<grid_for(n + m), kThreads, 0, c.stream>>>(n, m, c.q, c.b, c.eq_cstep, c.eq_rstep, kRuizIters);
        if (c.p_nnz)
            cudaMemcpyAsync(c.p_v, c.eq_p_ruiz, sizeof(double) * c.p_nnz, cudaMemcpyDeviceToDevice, c.stream);
        qmax_kernel<<<red_grid(n), kThreads, 0, c.stream>>>(c.q, n, c.eq_cobj, c.partials, c.counter);
        cost_scale<<<grid_for(std::max(c.p_nnz, n)), kThreads, 0, c.stream>>>(c.p_v, c.p_nnz, c.q, n, c.eq_cobj);
        c.launches += 4;
        k_build_base(c);
        return CIPM_OK;
    }
    gather_reorder<<<grid_for(nb), kThreads, 0, c.stream>>>(c.a_user, c.a_src, c.a_v, c.a_nnz, c.b_user, c.b_src,
                                                            c.b, m);
    set_ones<<<grid_for(std::max(n, m)), kThreads, 0, c.stream>>>(c.dc, n, c.dr, m);
    c.launches += 2;
    if (equilibrate) {
        for (int it = 0; it < kRuizIters; ++it) {   // RUIZ_ITERS, problem.py:36
            // per-pass steps kept (eq_cstep[it], eq_rstep[it]) for the q / b-only replay
            double* cst = c.eq_cstep + (int64_t)it * n;
            double* rst = c.eq_rstep + (int64_t)it * m;
            ruiz_norms<<<grid_for(n + m), kThreads, 0, c.stream>>>(n, m, c.p_rp, c.p_v, c.at_rp, c.at_src, c.a_rp,
                                                                   c.a_v, c.eq_cnorm, c.eq_rnorm);
            if (c.eq_nblocks)
                ruiz_blocks<<<grid_for(c.eq_nblocks), kThreads, 0, c.stream>>>(c.eq_rnorm, c.eq_boff, c.eq_bdim,
                                                                               c.eq_nblocks);
            ruiz_steps<<<grid_for(n + m), kThreads, 0, c.stream>>>(n, m, c.eq_cnorm, c.eq_rnorm, c.dc, c.dr, cst,
                                                                   rst);
            ruiz_scale<<<grid_for(n + m), kThreads, 0, c.stream>>>(n, m, c.p_rp, c.p_ci, c.p_v, c.a_rp, c.a_ci,
                                                                   c.a_v, c.q, c.b, cst, rst);
            c.launches += c.eq_nblocks ? 4 : 3;
        }
        if (c.p_nnz)
            cudaMemcpyAsync(c.eq_p_ruiz, c.p_v, sizeof(double) * c.p_nnz, cudaMemcpyDeviceToDevice, c.stream);
        qmax_kernel<<<red_grid(n), kThreads, 0, c.stream>>>(c.q, n, c.eq_cobj, c.partials, c.counter);
        cost_scale<<<grid_for(std::max(c.p_nnz, n)), kThreads, 0, c.stream>>>(c.p_v, c.p_nnz, c.q, n, c.eq_cobj);
        c.launches += 2;
    } else {
        cudaMemcpyAsync(c.eq_cobj, &c.one, sizeof(double), cudaMemcpyHostToDevice, c.stream);
    }
    transpose_vals<<<grid_for(c.a_nnz), kThreads, 0, c.stream>>>(c.a_v, c.at_src, c.at_v, c.a_nnz);
    c.launches++;
    k_build_base(c);
    return CIPM_OK;
}

}  // namespace cipm
