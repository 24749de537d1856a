// Cone-family kernels, following the paper's mixed-parallel strategy
// (PAPER.md:499-578): the zero + nonnegative rows are one flat coalesced pass,
// every second-order cone is one warp (shuffle reductions in a fixed order),
// exponential / power cones are one thread each, PSD cones one thread each.
//
// Reference units replaced (cones/scaling.py, cones/steps.py, cones/set.py):
//   k_update_scaling      update_scaling + ScalingState.kkt_values   scaling.py:201-251
//   k_scatter_h           KKTSystem.set_scaling (in-place −H scatter) system.py:166-179
//   k_apply_h             apply_H                                     scaling.py:254-274
//   k_combined_ds         combined_ds                                 scaling.py:277-320
//   k_step_bound          step_length closed forms                    steps.py:40-105, psdcone.py:120
//   k_nsym_feasible_mask  exp/pow ×0.8 backtrack (32 candidates)      steps.py:110-131
//   k_neighborhood_mask   neighborhood_ok (per-cone part)             scaling.py:364-401
//   k_membership          is_in_cone / is_in_dual_cone (strict)       set.py:166-207
//   k_soc_residuals       soc_residuals_batch (bit-exact order)       steps.py:136-186
#include <cuda_runtime.h>

#include "common.cuh"
#include "ctx.hpp"
#include "nsym.cuh"
#include "psd.cuh"

namespace cipm {

namespace {

constexpr int kNbBatch = 8;   // neighbourhood candidates per batch

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ============================== nonneg =====================================

__global__ void nn_scaling(const double* s, const double* z, double* h, double* w, double* lam,
                           int64_t nn0, int64_t nnd, int* err) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nnd) return;
    double si = s[nn0 + i], zi = z[nn0 + i];
    if (!(si > 0.0) || !(zi > 0.0)) set_error(err, CIPM_E_SCALING);
    double r = si / zi;
    h[i] = r;
    w[i] = sqrt(si / zi);
    lam[i] = sqrt(si * zi);
}

template <typename T>
__global__ void nn_scatter(T* lval, const int64_t* map_diag, const double* h, int64_t row0, int64_t nnd) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nnd) return;
    int64_t p = map_diag[row0 + i];
    lval[p] = lval[p] + (T)(-h[i]);
}

template <typename T>
__global__ void blk_scatter(T* lval, const int64_t* map_hblk, const double* hv, int64_t cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    int64_t p = map_hblk[i];
    lval[p] = lval[p] + (T)(-hv[i]);
}

// out = alpha*u + beta*(H v) on zero + nonneg rows (H = 0 on zero rows)
__global__ void nn_apply_h(const double* h, const double* v, double* out, double alpha, const double* u,
                           double beta, int64_t zero_dim, int64_t lin, const double* skip) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= lin || (skip && *skip != 0.0)) return;
    double hv = i < zero_dim ? 0.0 : h[i - zero_dim] * v[i];
    double base = u ? alpha * u[i] : 0.0;
    out[i] = base + beta * hv;
}

__global__ void nn_combined_ds(const double* s, const double* z, const double* dz_a, const double* ds_a,
                               const double* w, const double* lam, const double* sc, double* out,
                               int64_t zero_dim, int64_t lin) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= lin) return;
    if (i < zero_dim) { out[i] = 0.0; return; }
    const double sigma = sc[CIPM_SC_SIGMA], mu = sc[CIPM_SC_MU];
    int64_t k = i - zero_dim;
    double lam2 = s[i] * z[i];
    double eta = ds_a[i] * dz_a[i];
    out[i] = w[k] * ((lam2 + eta) - sigma * mu) / lam[k];
}

__global__ void nn_step_bound(const double* z, const double* s, const double* dz, const double* ds,
                              int64_t nn0, int64_t nnd, double* sc) {
    __shared__ double smin[32];
    double mn = INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnd; i += (int64_t)gridDim.x * blockDim.x) {
        double d1 = dz[nn0 + i], d2 = ds[nn0 + i];
        if (d1 < 0.0) mn = fmin(mn, -z[nn0 + i] / d1);
        if (d2 < 0.0) mn = fmin(mn, -s[nn0 + i] / d2);
    }
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
    if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mn = fmin(mn, smin[w]);
        if (mn < INFINITY) atomic_min_pos(sc + CIPM_SC_ALPHA_WORK, mn);
    }
}

__global__ void nn_membership(const double* s, const double* z, int64_t zero_dim, int64_t lin, int* err) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= lin) return;
    if (i < zero_dim) {
        if (s[i] != 0.0) set_error(err, CIPM_E_INTERIOR);
    } else if (!(s[i] > 0.0) || !(z[i] > 0.0)) {
        set_error(err, CIPM_E_INTERIOR);
    }
}

// ================================ SOC ======================================
// one warp per cone; lane j handles entries 1 + j, 1 + j + 32, ...

struct SocArgs {
    int64_t nsoc;
    const int32_t* off;
    const int32_t* dim;
    int64_t base;     // first SOC row (index into soc_w / soc_lam = row - base)
    const int64_t* hptr;
};

__global__ void soc_scaling(SocArgs a, const double* s, const double* z, double* W, double* LAM, double* ETA,
                            double* hv, int* err) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (c >= a.nsoc) return;
    const int off = a.off[c], d = a.dim[c];
    const double* sv = s + off;
    const double* zv = z + off;
    double ss = 0.0, zz = 0.0;
    for (int j = 1 + lane; j < d; j += 32) { ss += sv[j] * sv[j]; zz += zv[j] * zv[j]; }
    ss = warp_sum(ss);
    zz = warp_sum(zz);
    const double rs = sv[0] * sv[0] - ss, rz = zv[0] * zv[0] - zz;
    if (rs <= 0.0 || rz <= 0.0 || sv[0] <= 0.0 || zv[0] <= 0.0 || !(rs == rs) || !(rz == rz)) {
        if (lane == 0) set_error(err, CIPM_E_SCALING);
        return;
    }
    const double aa = sqrt(rs), bb = sqrt(rz);
    double sbzb = 0.0;
    for (int j = 1 + lane; j < d; j += 32) sbzb += (sv[j] / aa) * (zv[j] / bb);
    sbzb = warp_sum(sbzb) + (sv[0] / aa) * (zv[0] / bb);
    const double gamma = sqrt((1.0 + sbzb) / 2.0);
    const double eta = sqrt(aa / bb);
    double* w = W + (off - a.base);
    const double w0 = (sv[0] / aa + zv[0] / bb) / (2.0 * gamma);
    for (int j = 1 + lane; j < d; j += 32) w[j] = (sv[j] / aa + (-(zv[j] / bb))) / (2.0 * gamma);
    if (lane == 0) w[0] = w0;
    __syncwarp();
    // λ = η W̄ z
    double cz = 0.0;
    for (int j = 1 + lane; j < d; j += 32) cz += w[j] * zv[j];
    cz = warp_sum(cz);
    double* lam = LAM + (off - a.base);
    for (int j = 1 + lane; j < d; j += 32) lam[j] = eta * ((zv[0] * w[j] + zv[j]) + (cz / (1.0 + w0)) * w[j]);
    if (lane == 0) {
        lam[0] = eta * (w0 * zv[0] + cz);
        ETA[c] = eta;
    }
    // dense block values η²(2ww' + I − 2e0e0'), upper triangle row-major
    const double e2 = eta * eta;
    double* hb = hv + a.hptr[c];
    const int tot = d * (d + 1) / 2;
    for (int k = lane; k < tot; k += 32) {
        // invert k -> (rl, cl) with rl <= cl
        int rl = 0, rem = k;
        while (rem >= d - rl) { rem -= d - rl; ++rl; }
        const int cl = rl + rem;
        const double wr = rl == 0 ? w0 : w[rl];
        const double wc = cl == 0 ? w0 : w[cl];
        double hval = 2.0 * wr * wc;
        if (rl == cl) { hval += 1.0; if (rl == 0) hval -= 2.0; }
        hb[k] = e2 * hval;
    }
}

// out = alpha*u + beta*H v on SOC rows
__global__ void soc_apply_h(SocArgs a, const double* W, const double* ETA, const double* v, double* out,
                            double alpha, const double* u, double beta, const double* skip) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (c >= a.nsoc || (skip && *skip != 0.0)) return;
    const int off = a.off[c], d = a.dim[c];
    const double* w = W + (off - a.base);
    const double* vv = v + off;
    double dot = 0.0;
    for (int j = lane; j < d; j += 32) dot += w[j] * vv[j];
    dot = warp_sum(dot);
    const double e2 = ETA[c] * ETA[c];
    for (int j = lane; j < d; j += 32) {
        const double jv = j == 0 ? vv[0] : -vv[j];
        const double hv = e2 * ((2.0 * w[j]) * dot - jv);
        const double base = u ? alpha * u[off + j] : 0.0;
        out[off + j] = base + beta * hv;
    }
}

__global__ void soc_combined_ds(SocArgs a, const double* W, const double* ETA, const double* LAM,
                                const double* dz_a, const double* ds_a, const double* sc, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (c >= a.nsoc) return;
    const int off = a.off[c], d = a.dim[c];
    const double* w = W + (off - a.base);
    const double* lam = LAM + (off - a.base);
    const double* dsv = ds_a + off;
    const double* dzv = dz_a + off;
    const double eta = ETA[c];
    const double w0 = w[0];
    const double sigma = sc[CIPM_SC_SIGMA], mu = sc[CIPM_SC_MU];
    double c1 = 0.0, c2 = 0.0, ll = 0.0;
    for (int j = 1 + lane; j < d; j += 32) { c1 += w[j] * dsv[j]; c2 += w[j] * dzv[j]; ll += lam[j] * lam[j]; }
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    ll = warp_sum(ll);
    // A = W̄^-1 ds / η, B = η W̄ dz
    const double A0 = (w0 * dsv[0] - c1) / eta;
    const double B0 = eta * (w0 * dzv[0] + c2);
    double ab = 0.0;
    for (int j = 1 + lane; j < d; j += 32) {
        const double Aj = ((-dsv[0] * w[j] + dsv[j]) + (c1 / (1.0 + w0)) * w[j]) / eta;
        const double Bj = eta * ((dzv[0] * w[j] + dzv[j]) + (c2 / (1.0 + w0)) * w[j]);
        ab += Aj * Bj;
    }
    ab = warp_sum(ab);
    double* o = out + off;
    // rhs = λ∘λ + A∘B, rhs0 -= σμ  (stored in out as scratch)
    const double lam0 = lam[0];
    const double r0 = ((lam0 * lam0 + ll) + (A0 * B0 + ab)) - sigma * mu;
    for (int j = 1 + lane; j < d; j += 32) {
        const double Aj = ((-dsv[0] * w[j] + dsv[j]) + (c1 / (1.0 + w0)) * w[j]) / eta;
        const double Bj = eta * ((dzv[0] * w[j] + dzv[j]) + (c2 / (1.0 + w0)) * w[j]);
        o[j] = (lam0 * lam[j] + lam0 * lam[j]) + (A0 * Bj + B0 * Aj);
    }
    __syncwarp();
    // arrow solve λ ∘ u = rhs
    double lr = 0.0;
    for (int j = 1 + lane; j < d; j += 32) lr += lam[j] * o[j];
    lr = warp_sum(lr);
    const double res = lam0 * lam0 - ll;
    const double u0 = (lam0 * r0 - lr) / res;
    for (int j = 1 + lane; j < d; j += 32) o[j] = (o[j] - u0 * lam[j]) / lam0;
    __syncwarp();
    // out = η W̄ u
    double cu = 0.0;
    for (int j = 1 + lane; j < d; j += 32) cu += w[j] * o[j];
    cu = warp_sum(cu);
    for (int j = 1 + lane; j < d; j += 32) o[j] = eta * ((u0 * w[j] + o[j]) + (cu / (1.0 + w0)) * w[j]);
    if (lane == 0) o[0] = eta * (w0 * u0 + cu);
}

__device__ inline double soc_bound(double c, double b, double aa, double v0, double dv0) {
    double r1 = INFINITY;
    bool have = false;
    double roots[2];
    int nr = 0;
    if (aa == 0.0) {
        if (b < 0.0) roots[nr++] = -c / b;
    } else {
        double disc = b * b - 4.0 * aa * c;
        if (disc >= 0.0) {
            double sq = sqrt(disc);
            double qq = b != 0.0 ? -0.5 * (b + copysign(sq, b)) : 0.5 * sq * (aa > 0 ? 1.0 : -1.0);
            if (qq != 0.0) { roots[nr++] = qq / aa; roots[nr++] = c / qq; }
            else roots[nr++] = 0.0;
        }
    }
    for (int i = 0; i < nr; ++i)
        if (roots[i] > 0.0) { r1 = have ? fmin(r1, roots[i]) : roots[i]; have = true; }
    double bound = r1;
    if (dv0 < 0.0) bound = fmin(bound, -v0 / dv0);
    return bound;
}

__global__ void soc_step_bound(SocArgs a, const double* z, const double* s, const double* dz, const double* ds,
                               double* sc) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (c >= a.nsoc) return;
    const int off = a.off[c], d = a.dim[c];
    double res = INFINITY;
    for (int side = 0; side < 2; ++side) {
        const double* v = (side == 0 ? z : s) + off;
        const double* dv = (side == 0 ? dz : ds) + off;
        double vv = 0.0, vd = 0.0, dd = 0.0;
        for (int j = 1 + lane; j < d; j += 32) { vv += v[j] * v[j]; vd += v[j] * dv[j]; dd += dv[j] * dv[j]; }
        vv = warp_sum(vv);
        vd = warp_sum(vd);
        dd = warp_sum(dd);
        const double cc = v[0] * v[0] - vv;
        const double bb = 2.0 * (v[0] * dv[0] - vd);
        const double aa = dv[0] * dv[0] - dd;
        res = fmin(res, soc_bound(cc, bb, aa, v[0], dv[0]));
    }
    if (lane == 0 && res < INFINITY) atomic_min_pos(sc + CIPM_SC_ALPHA_WORK, res);
}

// neighbourhood per SOC: rs*rz/(s'z) >= β μ_k for each candidate of the batch
__global__ void soc_neighborhood(SocArgs a, const double* s, const double* z, const double* ds, const double* dz,
                                 const double* nb, int nk, double beta, unsigned int* mask, int* err) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (c >= a.nsoc) return;
    const int off = a.off[c], d = a.dim[c];
    unsigned int bits = 0u;
    for (int k = 0; k < nk; ++k) {
        const double step = nb[16 + k];
        double ss = 0.0, zz = 0.0, sz = 0.0;
        for (int j = 1 + lane; j < d; j += 32) {
            const double st = s[off + j] + step * ds[off + j];
            const double zt = z[off + j] + step * dz[off + j];
            ss += st * st; zz += zt * zt; sz += st * zt;
        }
        ss = warp_sum(ss);
        zz = warp_sum(zz);
        sz = warp_sum(sz);
        const double s0 = s[off] + step * ds[off], z0 = z[off] + step * dz[off];
        const double rs = s0 * s0 - ss, rz = z0 * z0 - zz;
        if (rs <= 0.0 || rz <= 0.0 || s0 <= 0.0 || z0 <= 0.0) {
            if (lane == 0) set_error(err, CIPM_E_DOMAIN);
            continue;
        }
        const double dot = s0 * z0 + sz;
        if (!(rs * rz / dot < beta * nb[k])) bits |= 1u << k;
    }
    if (lane == 0 && bits != (1u << nk) - 1u) atomicAnd(mask, bits | ~((1u << nk) - 1u));
}

__global__ void soc_membership(SocArgs a, const double* s, const double* z, int* err) {
    const int lane = threadIdx.x & 31;
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (c >= a.nsoc) return;
    const int off = a.off[c], d = a.dim[c];
    double ss = 0.0, zz = 0.0;
    for (int j = 1 + lane; j < d; j += 32) { ss += s[off + j] * s[off + j]; zz += z[off + j] * z[off + j]; }
    ss = warp_sum(ss);
    zz = warp_sum(zz);
    if (lane == 0 && (!(s[off] > sqrt(ss)) || !(z[off] > sqrt(zz)))) set_error(err, CIPM_E_INTERIOR);
}

// bit-exact batched residual (steps.py:136-175): chunks of 8 left to right,
// then pairwise rounds with the odd partial carried
__global__ void soc_residuals_kernel(SocArgs a, const double* x, double* out) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsoc) return;
    const int off = a.off[c], d = a.dim[c];
    const int nu = d - 1;
    const int nch = (nu + 7) / 8;
    double part[64];
    double t = x[off];
    if (nu <= 0) { out[c] = t * t; return; }
    if (nch <= 64) {
        for (int q = 0; q < nch; ++q) {
            const int lo = off + 1 + 8 * q;
            const int hi = min(lo + 8, off + 1 + nu);
            double acc = 0.0;
            for (int k = lo; k < hi; ++k) acc = acc + x[k] * x[k];
            part[q] = acc;
        }
        int width = nch;
        while (width > 1) {
            const int half = width / 2;
            for (int q = 0; q < half; ++q) part[q] = part[2 * q] + part[2 * q + 1];
            if (width % 2 == 1) { part[half] = part[width - 1]; width = half + 1; }
            else width = half;
        }
        out[c] = t * t - part[0];
    } else {
        out[c] = NAN;   // dims > 513 are handled by the host-side check (never on the solve path)
    }
}

// ============================= exp / pow ===================================

struct NsymArgs {
    int64_t nexp, nsym;
    const int32_t* exp_off;
    const int32_t* pow_off;
    const double* pow_alpha;
    const int64_t* hptr_base;   // unused: blocks are 6 entries each starting at hbase
    int64_t hbase;
};

__device__ __forceinline__ void nsym_cone(const NsymArgs& a, int64_t c, int* off, int* kind, double* alpha) {
    if (c < a.nexp) { *off = a.exp_off[c]; *kind = 0; *alpha = 0.0; }
    else { *off = a.pow_off[c - a.nexp]; *kind = 1; *alpha = a.pow_alpha[c - a.nexp]; }
}

__global__ void nsym_scaling(NsymArgs a, const double* s, const double* z, const double* sc, double* H,
                             double* G, double* HS, double* ZT, double* hv, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsym) return;
    int off, kind;
    double al;
    nsym_cone(a, c, &off, &kind, &al);
    const double mu = sc[CIPM_SC_MU];
    double sv[3] = {s[off], s[off + 1], s[off + 2]};
    double zv[3] = {z[off], z[off + 1], z[off + 2]};
    double g[3], hs[9], zt[3], h[9];
    bool ok;
    int rc;
    if (kind == 0) {
        ok = exp_primal_ok(sv) && exp_dual_ok(zv);
        if (!ok) { set_error(err, CIPM_E_SCALING); return; }
        exp_grad(zv, g);
        exp_hess(zv, hs);
        rc = exp_conj(sv, zt);
    } else {
        ok = pow_primal_ok(sv, al) && pow_dual_ok(zv, al);
        if (!ok) { set_error(err, CIPM_E_SCALING); return; }
        pow_grad(zv, al, g);
        pow_hess(zv, al, hs);
        rc = pow_conj(sv, al, zt);
    }
    if (rc != 0) { set_error(err, rc == CIPM_E_DOMAIN ? CIPM_E_DOMAIN : CIPM_E_SCALING); return; }
    if (!bfgs_block(sv, zv, mu, g, hs, zt, h)) { set_error(err, CIPM_E_SCALING); return; }
    for (int i = 0; i < 9; ++i) { H[9 * c + i] = h[i]; HS[9 * c + i] = hs[i]; }
    for (int i = 0; i < 3; ++i) { G[3 * c + i] = g[i]; ZT[3 * c + i] = zt[i]; }
    double* hb = hv + a.hbase + 6 * c;
    hb[0] = h[0]; hb[1] = h[1]; hb[2] = h[2]; hb[3] = h[4]; hb[4] = h[5]; hb[5] = h[8];
}

__global__ void nsym_apply_h(NsymArgs a, const double* H, const double* v, double* out, double alpha,
                             const double* u, double beta, const double* skip) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsym || (skip && *skip != 0.0)) return;
    int off, kind;
    double al;
    nsym_cone(a, c, &off, &kind, &al);
    const double* h = H + 9 * c;
    for (int i = 0; i < 3; ++i) {
        const double hv = h[3 * i] * v[off] + h[3 * i + 1] * v[off + 1] + h[3 * i + 2] * v[off + 2];
        const double base = u ? alpha * u[off + i] : 0.0;
        out[off + i] = base + beta * hv;
    }
}

__global__ void nsym_combined_ds(NsymArgs a, const double* s, const double* z, const double* dz_a,
                                 const double* ds_a, const double* G, const double* HS, const double* sc,
                                 double* out, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsym) return;
    int off, kind;
    double al;
    nsym_cone(a, c, &off, &kind, &al);
    const double sigma = sc[CIPM_SC_SIGMA], mu = sc[CIPM_SC_MU];
    double zv[3] = {z[off], z[off + 1], z[off + 2]};
    double u[3] = {dz_a[off], dz_a[off + 1], dz_a[off + 2]};
    double third[9];
    bool ok = kind == 0 ? exp_third(zv, u, third) : pow_third(zv, u, al, third);
    if (!ok) { set_error(err, CIPM_E_DOMAIN); return; }
    double hs[9];
    for (int i = 0; i < 9; ++i) hs[i] = HS[9 * c + i];
    double w[3] = {ds_a[off], ds_a[off + 1], ds_a[off + 2]};
    double eta[3] = {0.0, 0.0, 0.0};
    if (lu_solve(hs, 3, w, 1)) {
        for (int i = 0; i < 3; ++i)
            eta[i] = (-0.5 * third[3 * i]) * w[0] + (-0.5 * third[3 * i + 1]) * w[1] + (-0.5 * third[3 * i + 2]) * w[2];
    }
    const double sm = sigma * mu;
    for (int i = 0; i < 3; ++i) out[off + i] = (s[off + i] + sm * G[3 * c + i]) + eta[i];
}

// exp/pow strict feasibility of s + α_k ds, z + α_k dz for 32 candidates α_k = α·bt^k
__global__ void nsym_feasible_mask(NsymArgs a, const double* s, const double* z, const double* ds,
                                   const double* dz, const double* alpha0, double bt, unsigned int* mask) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsym) return;
    int off, kind;
    double al;
    nsym_cone(a, c, &off, &kind, &al);
    unsigned int bits = 0u;
    double alpha = *alpha0;
    for (int k = 0; k < 32; ++k) {
        double st[3], zt[3];
        for (int i = 0; i < 3; ++i) { st[i] = s[off + i] + alpha * ds[off + i]; zt[i] = z[off + i] + alpha * dz[off + i]; }
        bool ok = kind == 0 ? (exp_primal_ok(st) && exp_dual_ok(zt)) : (pow_primal_ok(st, al) && pow_dual_ok(zt, al));
        if (ok) bits |= 1u << k;
        alpha *= bt;
    }
    if (bits != 0xffffffffu) atomicAnd(mask, bits);
}

__global__ void nsym_neighborhood(NsymArgs a, const double* s, const double* z, const double* ds,
                                  const double* dz, const double* nb, int nk, double beta, unsigned int* mask,
                                  int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsym) return;
    int off, kind;
    double al;
    nsym_cone(a, c, &off, &kind, &al);
    unsigned int bits = 0u;
    for (int k = 0; k < nk; ++k) {
        const double step = nb[16 + k];
        double st[3], zt[3], w[3], g[3];
        for (int i = 0; i < 3; ++i) { st[i] = s[off + i] + step * ds[off + i]; zt[i] = z[off + i] + step * dz[off + i]; }
        int rc = kind == 0 ? exp_conj(st, w) : pow_conj(st, al, w);
        bool okg = kind == 0 ? exp_grad(zt, g) : pow_grad(zt, al, g);
        if (rc != 0 || !okg) { set_error(err, rc == CIPM_E_SCALING ? CIPM_E_SCALING : CIPM_E_DOMAIN); continue; }
        const double dot = (-g[0]) * w[0] + (-g[1]) * w[1] + (-g[2]) * w[2];
        if (!(3.0 / dot < beta * nb[k])) bits |= 1u << k;
    }
    if (bits != (1u << nk) - 1u) atomicAnd(mask, bits | ~((1u << nk) - 1u));
}

__global__ void nsym_membership(NsymArgs a, const double* s, const double* z, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.nsym) return;
    int off, kind;
    double al;
    nsym_cone(a, c, &off, &kind, &al);
    const double* sv = s + off;
    const double* zv = z + off;
    bool ok;
    if (kind == 0) ok = exp_member(sv) && exp_dual_member(zv);
    else ok = pow_member(sv[0], sv[1], sv[2], al) && pow_member(zv[0] / al, zv[1] / (1.0 - al), zv[2], al);
    if (!ok) set_error(err, CIPM_E_INTERIOR);
}

// ================================ PSD ======================================

struct PsdArgs {
    int64_t npsd;
    const int32_t* off;
    const int32_t* side;
    const int64_t* mptr;    // side^2 prefix
    const int64_t* lptr;    // side prefix
    const int64_t* hptr;    // into hv
};

template <int MS>
__global__ void psd_scaling(PsdArgs a, const double* s, const double* z, double* R, double* RI, double* Q,
                            double* LAM, double* hv, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.npsd) return;
    const int n = a.side[c], off = a.off[c];
    if (n > MS) return;
    double r[MS * MS], ri[MS * MS], lam[MS], q[MS * MS];
    int rc = psd_nt<MS>(s + off, z + off, n, r, ri, lam);
    if (rc != 0) { set_error(err, CIPM_E_SCALING); return; }
    mm<MS>(r, r, n, q, 2);   // Q = R R'
    double* Rc = R + a.mptr[c];
    double* RIc = RI + a.mptr[c];
    double* Qc = Q + a.mptr[c];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            Rc[i * n + j] = r[i * MS + j];
            RIc[i * n + j] = ri[i * MS + j];
            Qc[i * n + j] = q[i * MS + j];
        }
    for (int i = 0; i < n; ++i) LAM[a.lptr[c] + i] = lam[i];
    // congruence matrix of X -> Q X Q in svec coordinates, upper triangle row-major
    const int d = n * (n + 1) / 2;
    int ka[MS * (MS + 1) / 2], kb[MS * (MS + 1) / 2];
    {
        int k = 0;
        for (int j = 0; j < n; ++j)
            for (int i = j; i < n; ++i) { ka[k] = i; kb[k] = j; ++k; }
    }
    double* hb = hv + a.hptr[c];
    int t = 0;
    for (int k = 0; k < d; ++k) {
        const int p = ka[k], qq = kb[k];          // row entry (p, qq), p >= qq
        const double sk = p == qq ? 1.0 : kSqrt2;
        for (int l = k; l < d; ++l) {
            const int i = ka[l], j = kb[l];
            double mv;
            if (i == j) mv = q[p * MS + i] * q[qq * MS + i];
            else mv = (q[p * MS + i] * q[qq * MS + j] + q[p * MS + j] * q[qq * MS + i]) / kSqrt2;
            hb[t++] = sk * mv;
        }
    }
}

template <int MS>
__global__ void psd_apply_h(PsdArgs a, const double* Q, const double* v, double* out, double alpha,
                            const double* u, double beta, const double* skip) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.npsd || (skip && *skip != 0.0)) return;
    const int n = a.side[c], off = a.off[c];
    if (n > MS) return;
    double q[MS * MS], X[MS * MS], T[MS * MS], Y[MS * MS], hv[MS * (MS + 1) / 2];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) q[i * MS + j] = Q[a.mptr[c] + i * n + j];
    smat<MS>(v + off, n, X);
    mm<MS>(q, X, n, T, 0);
    mm<MS>(T, q, n, Y, 0);
    svec<MS>(Y, n, hv);
    const int d = n * (n + 1) / 2;
    for (int k = 0; k < d; ++k) {
        const double base = u ? alpha * u[off + k] : 0.0;
        out[off + k] = base + beta * hv[k];
    }
}

template <int MS>
__global__ void psd_combined_ds(PsdArgs a, const double* R, const double* RI, const double* LAM,
                                const double* dz_a, const double* ds_a, const double* sc, double* out) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.npsd) return;
    const int n = a.side[c], off = a.off[c];
    if (n > MS) return;
    const double sigma = sc[CIPM_SC_SIGMA], mu = sc[CIPM_SC_MU];
    double r[MS * MS], ri[MS * MS], lam[MS], X[MS * MS], T[MS * MS], A[MS * MS], B[MS * MS];
    for (int i = 0; i < n; ++i) {
        lam[i] = LAM[a.lptr[c] + i];
        for (int j = 0; j < n; ++j) {
            r[i * MS + j] = R[a.mptr[c] + i * n + j];
            ri[i * MS + j] = RI[a.mptr[c] + i * n + j];
        }
    }
    smat<MS>(ds_a + off, n, X);
    mm<MS>(ri, X, n, T, 0);
    mm<MS>(T, ri, n, A, 2);          // Rinv ds Rinv'
    smat<MS>(dz_a + off, n, X);
    mm<MS>(r, X, n, T, 1);           // R' dz
    mm<MS>(T, r, n, B, 0);           // R' dz R
    mm<MS>(A, B, n, X, 0);
    mm<MS>(B, A, n, T, 0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double e = 0.5 * (X[i * MS + j] + T[i * MS + j]);
            double rhs = (i == j ? lam[i] * lam[i] : 0.0) + e - (i == j ? sigma * mu : 0.0);
            A[i * MS + j] = 2.0 * rhs / (lam[i] + lam[j]);
        }
    mm<MS>(r, A, n, T, 0);
    mm<MS>(T, r, n, X, 2);           // R U R'
    svec<MS>(X, n, out + off);
}

template <int MS>
__global__ void psd_step_bound(PsdArgs a, const double* z, const double* s, const double* dz, const double* ds,
                               double* sc, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.npsd) return;
    const int n = a.side[c], off = a.off[c];
    if (n > MS) return;
    double b1 = psd_step<MS>(z + off, dz + off, n);
    double b2 = psd_step<MS>(s + off, ds + off, n);
    if (b1 < 0.0 || b2 < 0.0) { set_error(err, CIPM_E_DOMAIN); return; }
    double b = fmin(b1, b2);
    if (b < INFINITY) atomic_min_pos(sc + CIPM_SC_ALPHA_WORK, b);
}

template <int MS>
__global__ void psd_neighborhood(PsdArgs a, const double* s, const double* z, const double* ds, const double* dz,
                                 const double* nb, int nk, double beta, unsigned int* mask, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.npsd) return;
    const int n = a.side[c], off = a.off[c];
    if (n > MS) return;
    const int d = n * (n + 1) / 2;
    unsigned int bits = 0u;
    double st[MS * (MS + 1) / 2], zt[MS * (MS + 1) / 2];
    for (int k = 0; k < nk; ++k) {
        const double step = nb[16 + k];
        for (int i = 0; i < d; ++i) { st[i] = s[off + i] + step * ds[off + i]; zt[i] = z[off + i] + step * dz[off + i]; }
        double tr;
        if (!psd_trace_inv<MS>(st, zt, n, &tr)) { set_error(err, CIPM_E_DOMAIN); continue; }
        if (!((double)n / tr < beta * nb[k])) bits |= 1u << k;
    }
    if (bits != (1u << nk) - 1u) atomicAnd(mask, bits | ~((1u << nk) - 1u));
}

template <int MS>
__global__ void psd_membership(PsdArgs a, const double* s, const double* z, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= a.npsd) return;
    const int n = a.side[c], off = a.off[c];
    if (n > MS) return;
    if (!psd_is_pd<MS>(s + off, n) || !psd_is_pd<MS>(z + off, n)) set_error(err, CIPM_E_INTERIOR);
}

// ============================== launch glue ================================

SocArgs soc_args(Ctx& c) {
    SocArgs a;
    a.nsoc = c.nsoc;
    a.off = c.soc_off;
    a.dim = c.soc_dim;
    a.base = c.lin;
    a.hptr = c.soc_hptr;
    return a;
}

NsymArgs nsym_args(Ctx& c) {
    NsymArgs a;
    a.nexp = c.nexp;
    a.nsym = c.nsym;
    a.exp_off = c.exp_off;
    a.pow_off = c.pow_off;
    a.pow_alpha = c.pow_alpha;
    a.hptr_base = nullptr;
    a.hbase = c.nsym_hbase;
    return a;
}

PsdArgs psd_args(Ctx& c) {
    PsdArgs a;
    a.npsd = c.npsd;
    a.off = c.psd_off;
    a.side = c.psd_side;
    a.mptr = c.psd_mptr;
    a.lptr = c.psd_lptr;
    a.hptr = c.psd_hptr;
    return a;
}

inline int warp_grid(int64_t nwarps) { return grid_for(nwarps * 32); }

#define PSD_DISPATCH(KERNEL, ...)                                                        \
    do {                                                                                 \
        if (c.psd_max_side <= 4) KERNEL<4><<<grid_for(c.npsd, 128), 128, 0, c.stream>>>(__VA_ARGS__); \
        else if (c.psd_max_side <= 8) KERNEL<8><<<grid_for(c.npsd, 64), 64, 0, c.stream>>>(__VA_ARGS__); \
        else KERNEL<16><<<grid_for(c.npsd, 32), 32, 0, c.stream>>>(__VA_ARGS__);         \
        c.launches++;                                                                    \
    } while (0)

}  // namespace

// ---------------------------------------------------------------------------

// one family's scaling update (bench / profiling: per-family timing); fam 0 nonneg, 1 SOC, 2 exp/pow, 3 PSD
void k_update_scaling_family(Ctx& c, int fam) {
    if (fam == 0 && c.nonneg_dim) {
        nn_scaling<<<grid_for(c.nonneg_dim), kThreads, 0, c.stream>>>(c.s, c.z, c.nn_h, c.nn_w, c.nn_lam,
                                                                      c.zero_dim, c.nonneg_dim, c.err);
        c.launches++;
    }
    if (fam == 1 && c.nsoc) {
        soc_scaling<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.s, c.z, c.soc_w, c.soc_lam,
                                                                  c.soc_eta, c.hv, c.err);
        c.launches++;
    }
    if (fam == 2 && c.nsym) {
        nsym_scaling<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.sc, c.ns_h, c.ns_grad,
                                                                  c.ns_hess, c.ns_zt, c.hv, c.err);
        c.launches++;
    }
    if (fam == 3 && c.npsd) PSD_DISPATCH(psd_scaling, psd_args(c), c.s, c.z, c.psd_r, c.psd_rinv, c.psd_q, c.psd_lam, c.hv, c.err);
}

void k_update_scaling(Ctx& c) {
    if (c.nonneg_dim) {
        nn_scaling<<<grid_for(c.nonneg_dim), kThreads, 0, c.stream>>>(c.s, c.z, c.nn_h, c.nn_w, c.nn_lam,
                                                                      c.zero_dim, c.nonneg_dim, c.err);
        c.launches++;
    }
    if (c.nsoc) {
        soc_scaling<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.s, c.z, c.soc_w, c.soc_lam,
                                                                  c.soc_eta, c.hv, c.err);
        c.launches++;
    }
    if (c.nsym) {
        nsym_scaling<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.sc, c.ns_h, c.ns_grad,
                                                                  c.ns_hess, c.ns_zt, c.hv, c.err);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_scaling, psd_args(c), c.s, c.z, c.psd_r, c.psd_rinv, c.psd_q, c.psd_lam, c.hv, c.err);
}

// hv (upper triangles of all dense blocks) lives in c.wm (sized >= hblk_total)
void k_scatter_h(Ctx& c) {
    if (c.precision == CIPM_FULL) {
        if (c.nonneg_dim) {
            nn_scatter<double><<<grid_for(c.nonneg_dim), kThreads, 0, c.stream>>>(
                (double*)c.lval, c.sym.map_diag, c.nn_h, c.n + c.zero_dim, c.nonneg_dim);
            c.launches++;
        }
        if (c.hblk_total) {
            blk_scatter<double><<<grid_for(c.hblk_total), kThreads, 0, c.stream>>>((double*)c.lval, c.sym.map_hblk,
                                                                                   c.hv, c.hblk_total);
            c.launches++;
        }
    } else {
        if (c.nonneg_dim) {
            nn_scatter<float><<<grid_for(c.nonneg_dim), kThreads, 0, c.stream>>>(
                (float*)c.lval, c.sym.map_diag, c.nn_h, c.n + c.zero_dim, c.nonneg_dim);
            c.launches++;
        }
        if (c.hblk_total) {
            blk_scatter<float><<<grid_for(c.hblk_total), kThreads, 0, c.stream>>>((float*)c.lval, c.sym.map_hblk,
                                                                                 c.hv, c.hblk_total);
            c.launches++;
        }
    }
}

void k_apply_h(Ctx& c, const double* v, double* out, double alpha, const double* u, double beta,
               const double* skip) {
    if (c.lin) {
        nn_apply_h<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.nn_h, v, out, alpha, u, beta, c.zero_dim, c.lin,
                                                               skip);
        c.launches++;
    }
    if (c.nsoc) {
        soc_apply_h<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.soc_w, c.soc_eta, v, out, alpha, u,
                                                                  beta, skip);
        c.launches++;
    }
    if (c.nsym) {
        nsym_apply_h<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.ns_h, v, out, alpha, u, beta, skip);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_apply_h, psd_args(c), c.psd_q, v, out, alpha, u, beta, skip);
}

void k_combined_ds(Ctx& c, const double* dz_a, const double* ds_a) {
    if (c.lin) {
        nn_combined_ds<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.s, c.z, dz_a, ds_a, c.nn_w, c.nn_lam, c.sc,
                                                                   c.dsc, c.zero_dim, c.lin);
        c.launches++;
    }
    if (c.nsoc) {
        soc_combined_ds<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.soc_w, c.soc_eta, c.soc_lam,
                                                                      dz_a, ds_a, c.sc, c.dsc);
        c.launches++;
    }
    if (c.nsym) {
        nsym_combined_ds<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, dz_a, ds_a, c.ns_grad,
                                                                      c.ns_hess, c.sc, c.dsc, c.err);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_combined_ds, psd_args(c), c.psd_r, c.psd_rinv, c.psd_lam, dz_a, ds_a, c.sc, c.dsc);
}

void k_step_bound(Ctx& c, const double* dz, const double* ds) {
    if (c.nonneg_dim) {
        nn_step_bound<<<red_grid(c.nonneg_dim), kThreads, 0, c.stream>>>(c.z, c.s, dz, ds, c.zero_dim, c.nonneg_dim,
                                                                         c.sc);
        c.launches++;
    }
    if (c.nsoc) {
        soc_step_bound<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.z, c.s, dz, ds, c.sc);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_step_bound, psd_args(c), c.z, c.s, dz, ds, c.sc, c.err);
}

void k_nsym_feasible_mask(Ctx& c, const double* dz, const double* ds, int k0) {
    (void)k0;
    nsym_feasible_mask<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, ds, dz,
                                                                    c.sc + CIPM_SC_ALPHA_WORK, c.backtrack, c.mask);
    c.launches++;
}

// uses nb[0..nk) = μ_k, nb[16+k] = trial step a_k; dz/ds of the combined direction
void k_neighborhood_mask(Ctx& c, int k0, int nk) {
    (void)k0;
    if (c.nsoc) {
        soc_neighborhood<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.s, c.z, c.ds[1], c.dz[1], c.nb,
                                                                       nk, c.beta, c.mask, c.err);
        c.launches++;
    }
    if (c.nsym) {
        nsym_neighborhood<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.ds[1], c.dz[1],
                                                                       c.nb, nk, c.beta, c.mask, c.err);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_neighborhood, psd_args(c), c.s, c.z, c.ds[1], c.dz[1], c.nb, nk, c.beta, c.mask, c.err);
}

void k_membership(Ctx& c) {
    if (c.lin) {
        nn_membership<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.s, c.z, c.zero_dim, c.lin, c.err);
        c.launches++;
    }
    if (c.nsoc) {
        soc_membership<<<warp_grid(c.nsoc), kThreads, 0, c.stream>>>(soc_args(c), c.s, c.z, c.err);
        c.launches++;
    }
    if (c.nsym) {
        nsym_membership<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.err);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_membership, psd_args(c), c.s, c.z, c.err);
}

void k_soc_residuals(Ctx& c, const double* x, double* out) {
    if (!c.nsoc) return;
    soc_residuals_kernel<<<grid_for(c.nsoc, 64), 64, 0, c.stream>>>(soc_args(c), x, out);
    c.launches++;
}

void k_scaling_values(Ctx& c, double* diag, double* blocks) {
    (void)diag;
    (void)blocks;
}

}  // namespace cipm
