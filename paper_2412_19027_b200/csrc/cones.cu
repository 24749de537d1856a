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
#include "psd_warp.cuh"
#include "psd_reg.cuh"
#include <algorithm>

namespace cipm {

namespace {


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

// lane group of G lanes per cone (G = 8 / 16 / 32 by the largest SOC dimension:
// C3's dims 3-10 use 8, four cones per warp); every lane runs the group sums (no
// early exit: groups of one warp stay in lockstep), stores are guarded
template <int G>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
    for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

#define SOC_GROUP_SETUP                                                                  \
    const int gl = threadIdx.x & (G - 1);                                               \
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;             \
    if (((blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) / G) >= a.nsoc) return; \
    const bool live = c < a.nsoc;                                                        \
    const int off = live ? a.off[c] : 0, d = live ? a.dim[c] : 0;

template <int G>
__global__ void soc_scaling(SocArgs a, const double* s, const double* z, double* W, double* LAM, double* ETA,
                            double* hv, int* err) {
    SOC_GROUP_SETUP
    const double* sv = s + off;
    const double* zv = z + off;
    double ss = 0.0, zz = 0.0;
    for (int j = 1 + gl; j < d; j += G) { ss += sv[j] * sv[j]; zz += zv[j] * zv[j]; }
    ss = gsum<G>(ss);
    zz = gsum<G>(zz);
    const double s0 = live ? sv[0] : 1.0, z0 = live ? zv[0] : 1.0;
    const double rs = s0 * s0 - ss, rz = z0 * z0 - zz;
    const bool bad = live && (rs <= 0.0 || rz <= 0.0 || s0 <= 0.0 || z0 <= 0.0 || !(rs == rs) || !(rz == rz));
    if (bad && gl == 0) set_error(err, CIPM_E_SCALING);
    const bool ok = live && !bad;
    const double aa = ok ? sqrt(rs) : 1.0, bb = ok ? sqrt(rz) : 1.0;
    double sbzb = 0.0;
    if (ok)
        for (int j = 1 + gl; j < d; j += G) sbzb += (sv[j] / aa) * (zv[j] / bb);
    sbzb = gsum<G>(sbzb) + (s0 / aa) * (z0 / bb);
    const double gamma = sqrt((1.0 + sbzb) / 2.0);
    const double eta = sqrt(aa / bb);
    double* w = W + (off - a.base);
    const double w0 = (s0 / aa + z0 / bb) / (2.0 * gamma);
    if (ok) {
        for (int j = 1 + gl; j < d; j += G) w[j] = (sv[j] / aa + (-(zv[j] / bb))) / (2.0 * gamma);
        if (gl == 0) w[0] = w0;
    }
    __syncwarp();
    // λ = η W̄ z
    double cz = 0.0;
    if (ok)
        for (int j = 1 + gl; j < d; j += G) cz += w[j] * zv[j];
    cz = gsum<G>(cz);
    if (!ok) return;                                   // no group sums below
    double* lam = LAM + (off - a.base);
    for (int j = 1 + gl; j < d; j += G) lam[j] = eta * ((z0 * w[j] + zv[j]) + (cz / (1.0 + w0)) * w[j]);
    if (gl == 0) {
        lam[0] = eta * (w0 * z0 + cz);
        ETA[c] = eta;
    }
    // dense block values η²(2ww' + I − 2e0e0'), upper triangle row-major
    const double e2 = eta * eta;
    double* hb = hv + a.hptr[c];
    const int tot = d * (d + 1) / 2;
    for (int k = gl; k < tot; k += G) {
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
template <int G>
__global__ void soc_apply_h(SocArgs a, const double* W, const double* ETA, const double* v, double* out,
                            double alpha, const double* u, double beta, const double* skip) {
    if (skip && *skip != 0.0) return;
    SOC_GROUP_SETUP
    const double* w = W + (off - a.base);
    const double* vv = v + off;
    double dot = 0.0;
    for (int j = gl; j < d; j += G) dot += w[j] * vv[j];
    dot = gsum<G>(dot);
    if (!live) return;
    const double e2 = ETA[c] * ETA[c];
    for (int j = gl; j < d; j += G) {
        const double jv = j == 0 ? vv[0] : -vv[j];
        const double hv = e2 * ((2.0 * w[j]) * dot - jv);
        const double base = u ? alpha * u[off + j] : 0.0;
        out[off + j] = base + beta * hv;
    }
}

template <int G>
__global__ void soc_combined_ds(SocArgs a, const double* W, const double* ETA, const double* LAM,
                                const double* dz_a, const double* ds_a, const double* sc, double* out) {
    SOC_GROUP_SETUP
    const double* w = W + (off - a.base);
    const double* lam = LAM + (off - a.base);
    const double* dsv = ds_a + off;
    const double* dzv = dz_a + off;
    const double eta = live ? ETA[c] : 1.0;
    const double w0 = live ? w[0] : 0.0;
    const double ds0 = live ? dsv[0] : 0.0, dz0 = live ? dzv[0] : 0.0, lam0 = live ? lam[0] : 1.0;
    const double sigma = sc[CIPM_SC_SIGMA], mu = sc[CIPM_SC_MU];
    double c1 = 0.0, c2 = 0.0, ll = 0.0;
    for (int j = 1 + gl; j < d; j += G) { c1 += w[j] * dsv[j]; c2 += w[j] * dzv[j]; ll += lam[j] * lam[j]; }
    c1 = gsum<G>(c1);
    c2 = gsum<G>(c2);
    ll = gsum<G>(ll);
    // A = W̄^-1 ds / η, B = η W̄ dz
    const double A0 = (w0 * ds0 - c1) / eta;
    const double B0 = eta * (w0 * dz0 + c2);
    double ab = 0.0;
    for (int j = 1 + gl; j < d; j += G) {
        const double Aj = ((-ds0 * w[j] + dsv[j]) + (c1 / (1.0 + w0)) * w[j]) / eta;
        const double Bj = eta * ((dz0 * w[j] + dzv[j]) + (c2 / (1.0 + w0)) * w[j]);
        ab += Aj * Bj;
    }
    ab = gsum<G>(ab);
    double* o = out + off;
    // rhs = λ∘λ + A∘B, rhs0 -= σμ  (stored in out as scratch)
    const double r0 = ((lam0 * lam0 + ll) + (A0 * B0 + ab)) - sigma * mu;
    for (int j = 1 + gl; j < d; j += G) {
        const double Aj = ((-ds0 * w[j] + dsv[j]) + (c1 / (1.0 + w0)) * w[j]) / eta;
        const double Bj = eta * ((dz0 * w[j] + dzv[j]) + (c2 / (1.0 + w0)) * w[j]);
        o[j] = (lam0 * lam[j] + lam0 * lam[j]) + (A0 * Bj + B0 * Aj);
    }
    __syncwarp();
    // arrow solve λ ∘ u = rhs
    double lr = 0.0;
    for (int j = 1 + gl; j < d; j += G) lr += lam[j] * o[j];
    lr = gsum<G>(lr);
    const double res = lam0 * lam0 - ll;
    const double u0 = (lam0 * r0 - lr) / res;
    for (int j = 1 + gl; j < d; j += G) o[j] = (o[j] - u0 * lam[j]) / lam0;
    __syncwarp();
    // out = η W̄ u
    double cu = 0.0;
    for (int j = 1 + gl; j < d; j += G) cu += w[j] * o[j];
    cu = gsum<G>(cu);
    for (int j = 1 + gl; j < d; j += G) o[j] = eta * ((u0 * w[j] + o[j]) + (cu / (1.0 + w0)) * w[j]);
    if (live && gl == 0) o[0] = eta * (w0 * u0 + cu);
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

template <int G>
__global__ void soc_step_bound(SocArgs a, const double* z, const double* s, const double* dz, const double* ds,
                               double* sc) {
    SOC_GROUP_SETUP
    double res = INFINITY;
    for (int side = 0; side < 2; ++side) {
        const double* v = (side == 0 ? z : s) + off;
        const double* dv = (side == 0 ? dz : ds) + off;
        double vv = 0.0, vd = 0.0, dd = 0.0;
        for (int j = 1 + gl; j < d; j += G) { vv += v[j] * v[j]; vd += v[j] * dv[j]; dd += dv[j] * dv[j]; }
        vv = gsum<G>(vv);
        vd = gsum<G>(vd);
        dd = gsum<G>(dd);
        if (live) {
            const double cc = v[0] * v[0] - vv;
            const double bb = 2.0 * (v[0] * dv[0] - vd);
            const double aa = dv[0] * dv[0] - dd;
            res = fmin(res, soc_bound(cc, bb, aa, v[0], dv[0]));
        }
    }
    // one atomic per warp (the minimum is order-independent)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) res = fmin(res, __shfl_xor_sync(0xffffffffu, res, o));
    if ((threadIdx.x & 31) == 0 && res < INFINITY) atomic_min_pos(sc + CIPM_SC_ALPHA_WORK, res);
}

// neighbourhood per SOC: rs*rz/(s'z) >= β μ_k for each candidate of the batch
template <int G>
__global__ void soc_neighborhood(SocArgs a, const double* s, const double* z, const double* ds, const double* dz,
                                 const double* nb, int nk, double beta, unsigned int* mask, int* err) {
    SOC_GROUP_SETUP
    unsigned int bits = live ? 0u : (1u << nk) - 1u;
    for (int k = 0; k < nk; ++k) {
        const double step = nb[16 + k];
        double ss = 0.0, zz = 0.0, sz = 0.0;
        for (int j = 1 + gl; j < d; j += G) {
            const double st = s[off + j] + step * ds[off + j];
            const double zt = z[off + j] + step * dz[off + j];
            ss += st * st; zz += zt * zt; sz += st * zt;
        }
        ss = gsum<G>(ss);
        zz = gsum<G>(zz);
        sz = gsum<G>(sz);
        if (!live) continue;
        const double s0 = s[off] + step * ds[off], z0 = z[off] + step * dz[off];
        const double rs = s0 * s0 - ss, rz = z0 * z0 - zz;
        if (rs <= 0.0 || rz <= 0.0 || s0 <= 0.0 || z0 <= 0.0) {
            if (gl == 0) set_error(err, CIPM_E_DOMAIN);
            continue;
        }
        const double dot = s0 * z0 + sz;
        if (!(rs * rz / dot < beta * nb[k])) bits |= 1u << k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bits &= __shfl_xor_sync(0xffffffffu, bits, o);
    if ((threadIdx.x & 31) == 0 && bits != (1u << nk) - 1u) atomicAnd(mask, bits | ~((1u << nk) - 1u));
}

template <int G>
__global__ void soc_membership(SocArgs a, const double* s, const double* z, int* err) {
    SOC_GROUP_SETUP
    double ss = 0.0, zz = 0.0;
    for (int j = 1 + gl; j < d; j += G) { ss += s[off + j] * s[off + j]; zz += z[off + j] * z[off + j]; }
    ss = gsum<G>(ss);
    zz = gsum<G>(zz);
    if (live && gl == 0 && (!(s[off] > sqrt(ss)) || !(z[off] > sqrt(zz)))) set_error(err, CIPM_E_INTERIOR);
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
// a lane group per cone (psd_warp.cuh): G = 8 / 16 / 32 lanes by the largest
// side, lane i of a group owns row i of the cone's matrices, which live in the
// group's shared-memory slice of PW_MATS matrices (nmax x ld) plus two svec
// vectors and the eigenvalue vector; sides up to 32 (problem.py:36)

struct PsdArgs {
    int64_t npsd;
    const int32_t* off;
    const int32_t* side;
    const int64_t* mptr;    // side^2 prefix
    const int64_t* lptr;    // side prefix
    const int64_t* hptr;    // into hv
    int nmax, ld, gw;       // largest side, leading dimension, lanes per cone
};

constexpr int PW_MATS = 6;
constexpr bool kPsdCyclicJacobi = false;   // true: the cyclic ordering everywhere

struct PwView {
    double* M[PW_MATS];
    double *v0, *v1, *lam;
};

__device__ __forceinline__ int pw_slice_doubles(const PsdArgs& a) {
    return PW_MATS * a.nmax * a.ld + 2 * (a.nmax * (a.nmax + 1) / 2) + a.nmax + 2;
}

__device__ __forceinline__ PwView pw_view(const PsdArgs& a, double* smem) {
    const int grp = threadIdx.x / a.gw;                // group index within the CTA
    double* base = smem + (int64_t)grp * pw_slice_doubles(a);
    PwView v;
    const int msz = a.nmax * a.ld;
    for (int k = 0; k < PW_MATS; ++k) v.M[k] = base + k * msz;
    const int dmax = a.nmax * (a.nmax + 1) / 2;
    v.v0 = base + PW_MATS * msz;
    v.v1 = v.v0 + dmax;
    v.lam = v.v1 + dmax;
    return v;
}

// grid-stride loop over the warp's cone batches (warp-uniform trip count); inside,
// c is this group's cone (or -1) and G its lane view with the warp-uniform bound
#define PSD_GROUP_LOOP(a)                                                                           \
    extern __shared__ __align__(16) double psd_smem[];                                              \
    PwView W = pw_view(a, psd_smem);                                                                \
    const int lane = threadIdx.x & 31;                                                              \
    const int cpw = 32 / a.gw;                                                                      \
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;                      \
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;                                  \
    for (int64_t base = wid * cpw; base < a.npsd; base += nwarps * cpw)                             \
        for (int once = 0; once < 1; ++once)                                                        \
            if (const int64_t c = base + lane / a.gw; true)                                         \
                if (const pw::Grp G = psd_group(a, c, lane); true)

__device__ __forceinline__ pw::Grp psd_group(const PsdArgs& a, int64_t c, int lane) {
    pw::Grp G;
    G.i = lane % a.gw;
    G.g = a.gw;
    G.n = c < a.npsd ? a.side[c] : 0;
    G.nu = __reduce_max_sync(0xffffffffu, (unsigned)G.n);
    return G;
}

// NT scaling (scaling.py PSD part, psdcone.py:98-117) + congruence block H = Q (x)s Q
__global__ void psd_scaling_w(PsdArgs a, const double* s, const double* z, double* R, double* RI, double* Q,
                              double* LAM, double* hv, int* err) {
    PSD_GROUP_LOOP(a) {
        const int n = G.n, ld = a.ld, i = G.i;
        const int off = n ? a.off[c] : 0;
        double *W0 = W.M[0], *W1 = W.M[1], *W2 = W.M[2], *W3 = W.M[3], *Rm = W.M[4], *RIm = W.M[5];
        const bool ok = pw::nt_factor(G, s + off, z + off, ld, W0, W1, W2, W3, Rm, RIm, W.lam);
        if (n && !ok && i == 0) set_error(err, CIPM_E_SCALING);
        pw::Grp H = G;
        if (!ok) H.n = 0;
        pw::mm(H, Rm, Rm, ld, W0, 2);               // Q = R R'
        const int nn = H.n;
        if (nn) {
            double* Rc = R + a.mptr[c];
            double* RIc = RI + a.mptr[c];
            double* Qc = Q + a.mptr[c];
            for (int e = i; e < nn * nn; e += G.g) {
                const int r = e / nn, j = e - r * nn;
                Rc[e] = Rm[r * ld + j];
                RIc[e] = RIm[r * ld + j];
                Qc[e] = W0[r * ld + j];
            }
            for (int k = i; k < nn; k += G.g) LAM[a.lptr[c] + k] = W.lam[k];
            // H(k, l), k <= l over svec indices, upper triangle row-major; row k = (p, q)
            const int d = nn * (nn + 1) / 2;
            double* hb = hv + a.hptr[c];
            int64_t rowoff = 0;
            int p = 0, q = 0;
            for (int k = 0; k < d; ++k) {
                const double sk = p == q ? 1.0 : pw::kR2;
                for (int l = k + i; l < d; l += G.g) {
                    int j = 0, rem = l;
                    while (rem >= nn - j) { rem -= nn - j; ++j; }
                    const int ii = j + rem;
                    double mv;
                    if (ii == j) mv = W0[p * ld + ii] * W0[q * ld + ii];
                    else mv = (W0[p * ld + ii] * W0[q * ld + j] + W0[p * ld + j] * W0[q * ld + ii]) / pw::kR2;
                    hb[rowoff + (l - k)] = sk * mv;
                }
                rowoff += d - k;
                if (++p == nn) { ++q; p = q; }
            }
        }
        __syncwarp();
    }
}

// out = alpha u + beta svec(Q smat(v) Q)
__global__ void psd_apply_h_w(PsdArgs a, const double* Q, const double* v, double* out, double alpha,
                              const double* u, double beta, const double* skip) {
    if (skip && *skip != 0.0) return;
    PSD_GROUP_LOOP(a) {
        const int n = G.n, ld = a.ld, i = G.i;
        const int off = n ? a.off[c] : 0;
        double *Qm = W.M[0], *X = W.M[1], *T = W.M[2];
        for (int e = i; e < n * n; e += G.g) Qm[(e / n) * ld + e % n] = Q[a.mptr[c] + e];
        __syncwarp();
        if (n) pw::smat(G, v + off, X, ld);
        else __syncwarp();
        pw::mm(G, Qm, X, ld, T, 0);
        pw::mm(G, T, Qm, ld, X, 0);
        pw::svec(G, X, ld, W.v0);
        const int d = n * (n + 1) / 2;
        for (int k = i; k < d; k += G.g) {
            const double b0 = u ? alpha * u[off + k] : 0.0;
            out[off + k] = b0 + beta * W.v0[k];
        }
        __syncwarp();
    }
}

// combined d_s (scaling.py:277-320, PSD part): R (2 (diag lam^2 + sym(A B) - sigma mu I) / (lam_i + lam_j)) R'
__global__ void psd_combined_ds_w(PsdArgs a, const double* R, const double* RI, const double* LAM,
                                  const double* dz_a, const double* ds_a, const double* sc, double* out) {
    const double sigma = sc[CIPM_SC_SIGMA], mu = sc[CIPM_SC_MU];
    PSD_GROUP_LOOP(a) {
        const int n = G.n, ld = a.ld, i = G.i;
        const int off = n ? a.off[c] : 0;
        double *r = W.M[0], *ri = W.M[1], *X = W.M[2], *T = W.M[3], *A = W.M[4], *B = W.M[5];
        for (int e = i; e < n * n; e += G.g) {
            r[(e / n) * ld + e % n] = R[a.mptr[c] + e];
            ri[(e / n) * ld + e % n] = RI[a.mptr[c] + e];
        }
        for (int k = i; k < n; k += G.g) W.lam[k] = LAM[a.lptr[c] + k];
        __syncwarp();
        if (n) pw::smat(G, ds_a + off, X, ld);
        else __syncwarp();
        pw::mm(G, ri, X, ld, T, 0);
        pw::mm(G, T, ri, ld, A, 2);                  // Rinv ds Rinv'
        if (n) pw::smat(G, dz_a + off, X, ld);
        else __syncwarp();
        pw::mm(G, r, X, ld, T, 1);                   // R' dz
        pw::mm(G, T, r, ld, B, 0);                   // R' dz R
        pw::mm(G, A, B, ld, X, 0);
        pw::mm(G, B, A, ld, T, 0);
        if (i < n)
            for (int j = 0; j < n; ++j) {
                const double e = 0.5 * (X[i * ld + j] + T[i * ld + j]);
                const double rhs = (i == j ? W.lam[i] * W.lam[i] : 0.0) + e - (i == j ? sigma * mu : 0.0);
                A[i * ld + j] = 2.0 * rhs / (W.lam[i] + W.lam[j]);
            }
        __syncwarp();
        pw::mm(G, r, A, ld, T, 0);
        pw::mm(G, T, r, ld, X, 2);                   // R U R'
        if (n) pw::svec(G, X, ld, out + off);
        else __syncwarp();
    }
}

// sup{alpha >= 0: mat(v) + alpha mat(dv) PSD} (psdcone.py:120-133); < 0 on DomainError
__device__ __forceinline__ double psd_step_w(const pw::Grp& G, const double* v, const double* dv, int ld,
                                             const PwView& W) {
    double *X = W.M[0], *Li = W.M[1], *D = W.M[2], *T = W.M[3];
    if (G.n) pw::smat(G, v, X, ld);
    else __syncwarp();
    const bool ok = pw::chol(G, X, ld);
    pw::Grp H = G;
    if (!ok) H.n = 0;
    pw::tri_inv(H, X, ld, Li);
    if (H.n) pw::smat(H, dv, D, ld);
    else __syncwarp();
    pw::mm(H, Li, D, ld, T, 0);
    pw::mm(H, T, Li, ld, X, 2);                      // Li D Li'
    // parallel-ordered Jacobi with D's slice as the rotation table (cyclic for tiny sides)
    static_assert(PW_MATS >= 4, "psd_step_w uses four matrices");
    const double lmin = (G.nu >= 3 && !kPsdCyclicJacobi) ? pw::sym_min_eig_par(H, X, ld, D) : pw::sym_min_eig(H, X, ld);
    if (!ok) return -1.0;
    return lmin >= 0.0 ? INFINITY : -1.0 / lmin;
}

__global__ void psd_step_bound_w(PsdArgs a, const double* z, const double* s, const double* dz, const double* ds,
                                 double* sc, int* err) {
    PSD_GROUP_LOOP(a) {
        const int off = G.n ? a.off[c] : 0;
        const double b1 = psd_step_w(G, z + off, dz + off, a.ld, W);
        const double b2 = psd_step_w(G, s + off, ds + off, a.ld, W);
        if (G.n && G.i == 0) {
            if (b1 < 0.0 || b2 < 0.0) set_error(err, CIPM_E_DOMAIN);
            else {
                const double b = fmin(b1, b2);
                if (b < INFINITY) atomic_min_pos(sc + CIPM_SC_ALPHA_WORK, b);
            }
        }
        __syncwarp();
    }
}

// tr(S^-1 Z^-1); false if either is not positive definite
__device__ __forceinline__ bool psd_trace_inv_w(const pw::Grp& G, const double* sv, const double* zv, int ld,
                                                const PwView& W, double* tr) {
    double *X = W.M[0], *Li = W.M[1], *Si = W.M[2], *Zi = W.M[3];
    if (G.n) pw::smat(G, sv, X, ld);
    else __syncwarp();
    bool ok = pw::chol(G, X, ld);
    pw::tri_inv(G, X, ld, Li);
    pw::mm(G, Li, Li, ld, Si, 1);                    // L^-T L^-1 = S^-1
    if (G.n) pw::smat(G, zv, X, ld);
    else __syncwarp();
    ok = pw::chol(G, X, ld) && ok;
    pw::tri_inv(G, X, ld, Li);
    pw::mm(G, Li, Li, ld, Zi, 1);
    double acc = 0.0;
    if (G.i < G.n)
        for (int j = 0; j < G.n; ++j) acc += Si[G.i * ld + j] * Zi[j * ld + G.i];
    *tr = pw::gsum(acc, G.g);
    return ok;
}

__global__ void psd_neighborhood_w(PsdArgs a, const double* s, const double* z, const double* ds, const double* dz,
                                   const double* nb, int nk, double beta, unsigned int* mask, int* err) {
    PSD_GROUP_LOOP(a) {
        const int n = G.n;
        const int off = n ? a.off[c] : 0;
        const int d = n * (n + 1) / 2;
        unsigned int bits = 0u;
        for (int k = 0; k < nk; ++k) {
            const double step = nb[16 + k];
            for (int e = G.i; e < d; e += G.g) {
                W.v0[e] = s[off + e] + step * ds[off + e];
                W.v1[e] = z[off + e] + step * dz[off + e];
            }
            __syncwarp();
            double tr;
            const bool ok = psd_trace_inv_w(G, W.v0, W.v1, a.ld, W, &tr);
            if (!n) continue;
            if (!ok) {
                if (G.i == 0) set_error(err, CIPM_E_DOMAIN);
                continue;
            }
            if (!((double)n / tr < beta * nb[k])) bits |= 1u << k;
        }
        if (n && G.i == 0 && bits != (1u << nk) - 1u) atomicAnd(mask, bits | ~((1u << nk) - 1u));
        __syncwarp();
    }
}

__global__ void psd_membership_w(PsdArgs a, const double* s, const double* z, int* err) {
    PSD_GROUP_LOOP(a) {
        const int off = G.n ? a.off[c] : 0;
        if (G.n) pw::smat(G, s + off, W.M[0], a.ld);
        else __syncwarp();
        const bool ok1 = pw::chol(G, W.M[0], a.ld);
        if (G.n) pw::smat(G, z + off, W.M[1], a.ld);
        else __syncwarp();
        const bool ok2 = pw::chol(G, W.M[1], a.ld);
        if (G.n && G.i == 0 && (!ok1 || !ok2)) set_error(err, CIPM_E_INTERIOR);
        __syncwarp();
    }
}

// ---- equal sides N <= 8: one thread per cone, matrices in registers (psd_reg.cuh) ----

// cone data of a warp's cones is contiguous (svec blocks and N x N blocks in cone
// order): staged through shared memory with coalesced loads, one padded (odd
// stride, few bank conflicts) row per cone, then each thread works on its own row
template <int PER, int STRIDE>
__device__ __forceinline__ void stage_rows(const double* __restrict__ src, int cnt, double* dst) {
    const int lane = threadIdx.x & 31, tot = cnt * PER;
    double v[PER];                                   // every load of the lane in flight at once
#pragma unroll
    for (int u = 0; u < PER; ++u) v[u] = lane + 32 * u < tot ? src[lane + 32 * u] : 0.0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int e = lane + 32 * u;
        if (e < tot) dst[(e / PER) * STRIDE + e % PER] = v[u];
    }
}

template <int N>
__global__ void __launch_bounds__(32) psd_step_bound_r(int64_t npsd, const int32_t* __restrict__ off_,
                                                       const double* z, const double* s, const double* dz,
                                                       const double* ds, double* sc, int* err) {
    // two threads per cone (even lane: z, odd lane: s), 16 cones per warp
    constexpr int T = pr::Tri<N>::T, ST = T | 1;
    __shared__ double sv[1][2][16 * ST], sd[1][2][16 * ST];
    const int lane = threadIdx.x & 31, w = 0;     // one warp per block (the staging buffers)
    const int64_t c0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) >> 1;
    const int cnt = (int)(npsd - c0 < 16 ? npsd - c0 : 16);
    if (cnt <= 0) return;
    const int o0 = off_[c0];
    stage_rows<T, ST>(z + o0, cnt, sv[w][0]);
    stage_rows<T, ST>(s + o0, cnt, sv[w][1]);
    stage_rows<T, ST>(dz + o0, cnt, sd[w][0]);
    stage_rows<T, ST>(ds + o0, cnt, sd[w][1]);
    __syncwarp();
    const int k = lane >> 1, which = lane & 1;
    double b = INFINITY;
    bool bad = false;
    if (k < cnt) {
        const double bb = pr::step_bound<N>(sv[w][which] + k * ST, sd[w][which] + k * ST);
        bad = bb < 0.0;
        b = bb;
    }
    // the cone's DomainError when either bound failed (psdcone.py), else its min
    const bool bad2 = bad || __shfl_xor_sync(0xffffffffu, (int)bad, 1);
    if (bad2) {
        if (bad) set_error(err, CIPM_E_DOMAIN);
        b = INFINITY;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = fmin(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (lane == 0 && b < INFINITY) atomic_min_pos(sc + CIPM_SC_ALPHA_WORK, b);
}

// out = alpha u + beta svec(Q smat(v) Q)
template <int N>
__global__ void __launch_bounds__(32) psd_apply_h_r(int64_t npsd, const int32_t* __restrict__ off_,
                                                    const int64_t* __restrict__ mptr, const double* Q,
                                                    const double* v, double* out, double alpha, const double* u,
                                                    double beta, const double* skip) {
    if (skip && *skip != 0.0) return;
    constexpr int T = pr::Tri<N>::T, ST = T | 1, NN = N * N, SQ = NN | 1;
    __shared__ double sQ[1][32 * SQ], sV[1][32 * ST];
    const int lane = threadIdx.x & 31, w = 0;     // one warp per block (the staging buffers)
    const int64_t c0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31);
    const int cnt = (int)(npsd - c0 < 32 ? npsd - c0 : 32);
    if (cnt <= 0) return;
    const int o0 = off_[c0];
    stage_rows<NN, SQ>(Q + mptr[c0], cnt, sQ[w]);
    stage_rows<T, ST>(v + o0, cnt, sV[w]);
    __syncwarp();
    if (lane < cnt) {
        const double* Qr = sQ[w] + lane * SQ;
        double Qs[T], X[T], Y[T];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) Qs[pr::P(i, j)] = Qr[i * N + j];
        pr::smat<N>(sV[w] + lane * ST, X);
        pr::congr_sym<N>(Qs, X, Y);
        double* Vr = sV[w] + lane * ST;
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
            for (int i = j; i < N; ++i) Vr[pr::SV(i, j, N)] = i == j ? Y[pr::P(i, i)] : pr::kR2 * Y[pr::P(i, j)];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const int e = lane + 32 * k;
        if (e < cnt * T) {
            const double hv = sV[w][(e / T) * ST + e % T];
            const double b0 = u ? alpha * u[o0 + e] : 0.0;
            out[o0 + e] = b0 + beta * hv;
        }
    }
}

template <int N>
__global__ void __launch_bounds__(32) psd_neighborhood_r(int64_t npsd, const int32_t* __restrict__ off_,
                                                         const double* s, const double* z, const double* ds,
                                                         const double* dz, const double* nb, int nk, double beta,
                                                         unsigned int* mask, int* err) {
    constexpr int T = pr::Tri<N>::T, ST = T | 1;
    __shared__ double sS[1][32 * ST], sZ[1][32 * ST], sDS[1][32 * ST], sDZ[1][32 * ST];
    const int lane = threadIdx.x & 31, w = 0;     // one warp per block (the staging buffers)
    const int64_t c0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31);
    const int cnt = (int)(npsd - c0 < 32 ? npsd - c0 : 32);
    if (cnt <= 0) return;
    const int o0 = off_[c0];
    stage_rows<T, ST>(s + o0, cnt, sS[w]);
    stage_rows<T, ST>(z + o0, cnt, sZ[w]);
    stage_rows<T, ST>(ds + o0, cnt, sDS[w]);
    stage_rows<T, ST>(dz + o0, cnt, sDZ[w]);
    __syncwarp();
    unsigned int bits = (1u << nk) - 1u;
    if (lane < cnt) {
        const double *sr = sS[w] + lane * ST, *zr = sZ[w] + lane * ST;
        const double *dsr = sDS[w] + lane * ST, *dzr = sDZ[w] + lane * ST;
        bits = 0u;
        for (int k = 0; k < nk; ++k) {
            const double step = nb[16 + k];
            double svk[T], zvk[T];
#pragma unroll
            for (int e = 0; e < T; ++e) {
                svk[e] = sr[e] + step * dsr[e];
                zvk[e] = zr[e] + step * dzr[e];
            }
            double Si[T], Zi[T];
            const bool ok1 = pr::sym_inv<N>(svk, Si);
            const bool ok2 = pr::sym_inv<N>(zvk, Zi);
            if (!ok1 || !ok2) {
                set_error(err, CIPM_E_DOMAIN);
                continue;
            }
            double tr = 0.0;                             // tr(S^-1 Z^-1), row by row as the warp version
#pragma unroll
            for (int i = 0; i < N; ++i) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) acc += Si[pr::P(i, j)] * Zi[pr::P(j, i)];
                tr += acc;
            }
            if (!((double)N / tr < beta * nb[k])) bits |= 1u << k;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bits &= __shfl_xor_sync(0xffffffffu, bits, o);
    if (lane == 0 && bits != (1u << nk) - 1u) atomicAnd(mask, bits | ~((1u << nk) - 1u));
}

// NT scaling (psdcone.py:98-117, pw::nt_factor) + the congruence block H = Q (x)s Q,
// one thread per cone: Ls, Lz, M = Lz' Ls, one-sided cyclic Jacobi SVD of M
// (M V = U diag(sig)), R = Ls V sig^-1/2, R^-1 = sig^1/2 V' Ls^-1
template <int N>
__global__ void __launch_bounds__(32) psd_scaling_r(int64_t npsd, const int32_t* __restrict__ off_,
                                                    const int64_t* __restrict__ mptr, const int64_t* __restrict__ lptr,
                                                    const int64_t* __restrict__ hptr, const double* s,
                                                    const double* z, double* R, double* RI, double* Q, double* LAM,
                                                    double* hv, int* err) {
    constexpr int T = pr::Tri<N>::T, ST = T | 1;
    __shared__ double sS[32 * ST], sZ[32 * ST];
    const int lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * 32;
    const int cnt = (int)(npsd - c0 < 32 ? npsd - c0 : 32);
    if (cnt <= 0) return;
    const int o0 = off_[c0];
    stage_rows<T, ST>(s + o0, cnt, sS);
    stage_rows<T, ST>(z + o0, cnt, sZ);
    __syncwarp();
    if (lane >= cnt) return;
    const int64_t c = c0 + lane;
    double Ls[T], Lz[T];
    pr::smat<N>(sS + lane * ST, Ls);
    pr::smat<N>(sZ + lane * ST, Lz);
    const bool ok1 = pr::chol<N>(Ls), ok2 = pr::chol<N>(Lz);
    if (!ok1 || !ok2) { set_error(err, CIPM_E_SCALING); return; }
    double U[N][N], V[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double v = 0.0;
#pragma unroll
            for (int k = (i > j ? i : j); k < N; ++k) v += Lz[pr::P(k, i)] * Ls[pr::P(k, j)];
            U[i][j] = v;
            V[i][j] = i == j ? 1.0 : 0.0;
        }
#pragma unroll 1
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rot = false;
        // cyclic order (as pw::jacobi_svd): the scaling feeds H, and the refinement
        // counts of the late iterations are sensitive to its rounding
#pragma unroll
        for (int p = 0; p < N - 1; ++p)
#pragma unroll
            for (int q = p + 1; q < N; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    al += U[k][p] * U[k][p];
                    be += U[k][q] * U[k][q];
                    ga += U[k][p] * U[k][q];
                }
                if (fabs(ga) <= 1e-15 * sqrt(al * be) || ga == 0.0) continue;
                rot = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    const double up = U[k][p], uq = U[k][q];
                    U[k][p] = cs * up - sn * uq;
                    U[k][q] = sn * up + cs * uq;
                    const double vp = V[k][p], vq = V[k][q];
                    V[k][p] = cs * vp - sn * vq;
                    V[k][q] = sn * vp + cs * vq;
                }
            }
        if (!rot) break;
    }
    double sig[N];
    bool pos = true;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double s2 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) s2 += U[k][j] * U[k][j];
        sig[j] = sqrt(s2);
        pos = pos && sig[j] > 0.0;
    }
    if (!pos) { set_error(err, CIPM_E_SCALING); return; }
    double Lsi[T];
    pr::tri_inv<N>(Ls, Lsi);
    double* Rc = R + mptr[c];
    double* RIc = RI + mptr[c];
    double Rm[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int k = 0; k <= i; ++k) a += Ls[pr::P(i, k)] * V[k][j];         // (Ls V)(i, j)
#pragma unroll
            for (int k = j; k < N; ++k) b += V[k][i] * Lsi[pr::P(k, j)];        // (V' Ls^-1)(i, j)
            Rm[i][j] = a / sqrt(sig[j]);
            Rc[i * N + j] = Rm[i][j];
            RIc[i * N + j] = b * sqrt(sig[i]);
        }
#pragma unroll
    for (int j = 0; j < N; ++j) LAM[lptr[c] + j] = sig[j];
    double Qs[T];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) v += Rm[i][k] * Rm[j][k];
            Qs[pr::P(i, j)] = v;
        }
    double* Qc = Q + mptr[c];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) Qc[i * N + j] = Qs[pr::P(i, j)];
    // H(k, l), k <= l over svec indices, upper triangle row-major (pw kernel's layout)
    double* hb = hv + hptr[c];
    int rowoff = 0;
#pragma unroll
    for (int qk = 0; qk < N; ++qk)
#pragma unroll
        for (int pk = qk; pk < N; ++pk) {
            const int k = pr::SV(pk, qk, N);
            const double sk = pk == qk ? 1.0 : pr::kR2;
#pragma unroll
            for (int jl = 0; jl < N; ++jl)
#pragma unroll
                for (int il = jl; il < N; ++il) {
                    const int l = pr::SV(il, jl, N);
                    if (l < k) continue;
                    double mv;
                    if (il == jl) mv = Qs[pr::P(pk, il)] * Qs[pr::P(qk, il)];
                    else mv = (Qs[pr::P(pk, il)] * Qs[pr::P(qk, jl)] + Qs[pr::P(pk, jl)] * Qs[pr::P(qk, il)]) / pr::kR2;
                    hb[rowoff + (l - k)] = sk * mv;
                }
            rowoff += T - k;
        }
}

template <int N>
__global__ void __launch_bounds__(128) psd_membership_r(int64_t npsd, const int32_t* __restrict__ off_,
                                                        const double* s, const double* z, int* err) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= npsd) return;
    const int off = off_[c];
    double A[pr::Tri<N>::T], B[pr::Tri<N>::T];
    pr::smat<N>(s + off, A);
    pr::smat<N>(z + off, B);
    const bool ok1 = pr::chol<N>(A), ok2 = pr::chol<N>(B);
    if (!ok1 || !ok2) set_error(err, CIPM_E_INTERIOR);
}

// dispatch on the uniform side (returns false: use the lane-group kernels)
#define PSD_REG_DISPATCH(KERNEL, ...) PSD_REG_DISPATCH_T(KERNEL, 1, 128, __VA_ARGS__)
#define PSD_REG_DISPATCH_T(KERNEL, TPC, BS, ...)                                              \
    ([&]() -> bool {                                                                          \
        const int g_ = (int)((c.npsd * (TPC) + (BS) - 1) / (BS));                             \
        switch (c.psd_uni) {                                                                  \
            case 1: KERNEL<1><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 2: KERNEL<2><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 3: KERNEL<3><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 4: KERNEL<4><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 5: KERNEL<5><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 6: KERNEL<6><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 7: KERNEL<7><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            case 8: KERNEL<8><<<g_, BS, 0, c.stream>>>(__VA_ARGS__); break;                  \
            default: return false;                                                            \
        }                                                                                     \
        c.launches++;                                                                         \
        return true;                                                                          \
    }())

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
    a.nmax = c.psd_max_side;
    a.ld = c.psd_max_side | 1;
    a.gw = c.psd_max_side <= 8 ? 8 : (c.psd_max_side <= 16 ? 16 : 32);
    return a;
}

// group-per-cone PSD launch: slices per warp = 32 / gw; warps per CTA from the slice
// size (<= 96 KiB per CTA)
inline size_t psd_slice_bytes(const PsdArgs& a) {
    return sizeof(double) * (size_t)(32 / a.gw) *
           (size_t)(PW_MATS * a.nmax * a.ld + 2 * (a.nmax * (a.nmax + 1) / 2) + a.nmax + 2);
}

#define PSD_DISPATCH(KERNEL, ...)                                                                      \
    do {                                                                                               \
        const PsdArgs pa_ = psd_args(c);                                                               \
        const size_t sl_ = psd_slice_bytes(pa_);                                                       \
        int wpb_ = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / sl_));                   \
        const size_t smem_ = sl_ * (size_t)wpb_;                                                       \
        if (smem_ > 48 * 1024) cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_); \
        const int64_t blocks_ = (c.npsd + (int64_t)wpb_ * (32 / pa_.gw) - 1) / ((int64_t)wpb_ * (32 / pa_.gw)); \
        KERNEL<<<(int)std::min<int64_t>(blocks_, 148 * 32), wpb_ * 32, smem_, c.stream>>>(__VA_ARGS__); \
        c.launches++;                                                                                  \
    } while (0)

}  // namespace

// ---------------------------------------------------------------------------

// KKTSystem seam: H v from the dense blocks in hv (packed upper triangle per block,
// the layout cipm_scaling_values returns), one thread per conic row past the
// zero / nonneg span (binary search of the row's block)
__global__ void blk_apply_h(const int32_t* __restrict__ boff, const int32_t* __restrict__ bdim,
                            const int64_t* __restrict__ bh, int64_t nblk, const double* __restrict__ hv,
                            const double* v, double* out, double alpha, const double* u, double beta, int64_t lin,
                            int64_t m, const double* skip) {
    const int64_t r = lin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= m || (skip && *skip != 0.0)) return;
    int64_t lo = 0, hi = nblk - 1;
    while (lo < hi) {                                  // last block with offset <= r
        const int64_t mid = (lo + hi + 1) >> 1;
        if (boff[mid] <= r) lo = mid;
        else hi = mid - 1;
    }
    const int off = boff[lo], d = bdim[lo], i = (int)(r - off);
    const double* H = hv + bh[lo];
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
        const int a = i < j ? i : j, b = i < j ? j : i;          // upper entry (a, b), a <= b
        acc += H[a * d - a * (a - 1) / 2 + (b - a)] * v[off + j];
    }
    const double base = u ? alpha * u[r] : 0.0;
    out[r] = base + beta * acc;
}

// SOC launch: G lanes per cone (c.soc_group), 256-thread blocks
#define SOC_LAUNCH(KERNEL, ...)                                                                       \
    do {                                                                                              \
        const int g_ = c.soc_group;                                                                   \
        const int nb_ = (int)((c.nsoc * g_ + kThreads - 1) / kThreads);                               \
        if (g_ == 8) KERNEL<8><<<nb_, kThreads, 0, c.stream>>>(__VA_ARGS__);                          \
        else if (g_ == 16) KERNEL<16><<<nb_, kThreads, 0, c.stream>>>(__VA_ARGS__);                   \
        else KERNEL<32><<<nb_, kThreads, 0, c.stream>>>(__VA_ARGS__);                                 \
        c.launches++;                                                                                 \
    } while (0)

// PSD NT scaling: register kernel for equal sides <= 8 (CIPM_PSD_SCALING_WARP=1: the
// lane-group kernel, experiments), lane-group kernel otherwise
static void k_psd_scaling(Ctx& c) {
    static const bool warp_env = getenv("CIPM_PSD_SCALING_WARP") != nullptr;
    if (!warp_env && PSD_REG_DISPATCH_T(psd_scaling_r, 1, 32, c.npsd, c.psd_off, c.psd_mptr, c.psd_lptr,
                                         c.psd_hptr, c.s, c.z, c.psd_r, c.psd_rinv, c.psd_q, c.psd_lam, c.hv, c.err))
        return;
    PSD_DISPATCH(psd_scaling_w, pa_, c.s, c.z, c.psd_r, c.psd_rinv, c.psd_q, c.psd_lam, c.hv, c.err);
}

// one family's scaling update (bench / profiling: per-family timing); fam 0 nonneg, 1 SOC, 2 exp/pow, 3 PSD
void k_update_scaling_family(Ctx& c, int fam) {
    if (fam == 0 && c.nonneg_dim) {
        nn_scaling<<<grid_for(c.nonneg_dim), kThreads, 0, c.stream>>>(c.s, c.z, c.nn_h, c.nn_w, c.nn_lam,
                                                                      c.zero_dim, c.nonneg_dim, c.err);
        c.launches++;
    }
    if (fam == 1 && c.nsoc) {
        SOC_LAUNCH(soc_scaling, soc_args(c), c.s, c.z, c.soc_w, c.soc_lam,
                                                                  c.soc_eta, c.hv, c.err);
    }
    if (fam == 2 && c.nsym) {
        nsym_scaling<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.sc, c.ns_h, c.ns_grad,
                                                                  c.ns_hess, c.ns_zt, c.hv, c.err);
        c.launches++;
    }
    if (fam == 3 && c.npsd) k_psd_scaling(c);
}

void k_update_scaling(Ctx& c) {
    if (c.nonneg_dim) {
        nn_scaling<<<grid_for(c.nonneg_dim), kThreads, 0, c.stream>>>(c.s, c.z, c.nn_h, c.nn_w, c.nn_lam,
                                                                      c.zero_dim, c.nonneg_dim, c.err);
        c.launches++;
    }
    if (c.nsoc) {
        SOC_LAUNCH(soc_scaling, soc_args(c), c.s, c.z, c.soc_w, c.soc_lam,
                                                                  c.soc_eta, c.hv, c.err);
    }
    if (c.nsym) {
        nsym_scaling<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.sc, c.ns_h, c.ns_grad,
                                                                  c.ns_hess, c.ns_zt, c.hv, c.err);
        c.launches++;
    }
    if (c.npsd) k_psd_scaling(c);
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
    if (c.host_scaling) {                 // H set by the host (cipm_kkt_set_scaling): the stored blocks
        if (c.lin) {
            nn_apply_h<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.nn_h, v, out, alpha, u, beta, c.zero_dim, c.lin,
                                                                   skip);
            c.launches++;
        }
        if (c.nblk) {
            blk_apply_h<<<grid_for(c.m - c.lin), kThreads, 0, c.stream>>>(c.blk_off, c.blk_dim, c.blk_hptr, c.nblk,
                                                                          c.hv, v, out, alpha, u, beta, c.lin, c.m,
                                                                          skip);
            c.launches++;
        }
        return;
    }
    if (c.lin) {
        nn_apply_h<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.nn_h, v, out, alpha, u, beta, c.zero_dim, c.lin,
                                                               skip);
        c.launches++;
    }
    if (c.nsoc) {
        SOC_LAUNCH(soc_apply_h, soc_args(c), c.soc_w, c.soc_eta, v, out, alpha, u,
                                                                  beta, skip);
    }
    if (c.nsym) {
        nsym_apply_h<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.ns_h, v, out, alpha, u, beta, skip);
        c.launches++;
    }
    if (c.npsd && !PSD_REG_DISPATCH_T(psd_apply_h_r, 1, 32, c.npsd, c.psd_off, c.psd_mptr, c.psd_q, v, out, alpha, u, beta, skip))
        PSD_DISPATCH(psd_apply_h_w, pa_, c.psd_q, v, out, alpha, u, beta, skip);
}

void k_combined_ds(Ctx& c, const double* dz_a, const double* ds_a) {
    if (c.lin) {
        nn_combined_ds<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.s, c.z, dz_a, ds_a, c.nn_w, c.nn_lam, c.sc,
                                                                   c.dsc, c.zero_dim, c.lin);
        c.launches++;
    }
    if (c.nsoc) {
        SOC_LAUNCH(soc_combined_ds, soc_args(c), c.soc_w, c.soc_eta, c.soc_lam,
                                                                      dz_a, ds_a, c.sc, c.dsc);
    }
    if (c.nsym) {
        nsym_combined_ds<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, dz_a, ds_a, c.ns_grad,
                                                                      c.ns_hess, c.sc, c.dsc, c.err);
        c.launches++;
    }
    if (c.npsd) PSD_DISPATCH(psd_combined_ds_w, pa_, c.psd_r, c.psd_rinv, c.psd_lam, dz_a, ds_a, c.sc, c.dsc);
}

void k_step_bound(Ctx& c, const double* dz, const double* ds) {
    if (c.nonneg_dim) {
        nn_step_bound<<<red_grid(c.nonneg_dim), kThreads, 0, c.stream>>>(c.z, c.s, dz, ds, c.zero_dim, c.nonneg_dim,
                                                                         c.sc);
        c.launches++;
    }
    if (c.nsoc) {
        SOC_LAUNCH(soc_step_bound, soc_args(c), c.z, c.s, dz, ds, c.sc);
    }
    if (c.npsd && !PSD_REG_DISPATCH_T(psd_step_bound_r, 2, 32, c.npsd, c.psd_off, c.z, c.s, dz, ds, c.sc, c.err))
        PSD_DISPATCH(psd_step_bound_w, pa_, c.z, c.s, dz, ds, c.sc, c.err);
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
        SOC_LAUNCH(soc_neighborhood, soc_args(c), c.s, c.z, c.ds[1], c.dz[1], c.nb,
                                                                       nk, c.beta, c.mask, c.err);
    }
    if (c.nsym) {
        nsym_neighborhood<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.ds[1], c.dz[1],
                                                                       c.nb, nk, c.beta, c.mask, c.err);
        c.launches++;
    }
    if (c.npsd && !PSD_REG_DISPATCH_T(psd_neighborhood_r, 1, 32, c.npsd, c.psd_off, c.s, c.z, c.ds[1], c.dz[1], c.nb, nk, c.beta, c.mask, c.err))
        PSD_DISPATCH(psd_neighborhood_w, pa_, c.s, c.z, c.ds[1], c.dz[1], c.nb, nk, c.beta, c.mask, c.err);
}

void k_membership(Ctx& c) {
    if (c.lin) {
        nn_membership<<<grid_for(c.lin), kThreads, 0, c.stream>>>(c.s, c.z, c.zero_dim, c.lin, c.err);
        c.launches++;
    }
    if (c.nsoc) {
        SOC_LAUNCH(soc_membership, soc_args(c), c.s, c.z, c.err);
    }
    if (c.nsym) {
        nsym_membership<<<grid_for(c.nsym, 128), 128, 0, c.stream>>>(nsym_args(c), c.s, c.z, c.err);
        c.launches++;
    }
    if (c.npsd && !PSD_REG_DISPATCH(psd_membership_r, c.npsd, c.psd_off, c.s, c.z, c.err))
        PSD_DISPATCH(psd_membership_w, pa_, c.s, c.z, c.err);
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
