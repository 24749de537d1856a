// C ABI of libcipm (include/cipm.h): context lifetime, host<->device plumbing
// and the Algorithm-1 step entry points.  Each entry point enqueues kernels on
// the context's stream; the ones that must return a decision to the host
// (residual scalars, refinement convergence, backtracking outcomes, take_step)
// synchronise once and return the latched device error word.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "symbolic.hpp"

namespace cipm {
// launchers defined in vec.cu that are not in ctx.hpp
void k_nsym_resolve(Ctx& c);
void k_step_store(Ctx& c, int which);
void k_nb_resolve(Ctx& c, int g0, int nk);
void k_kkt_residual_one(Ctx& c, int q);
void k_kkt_residual(Ctx& c, int nrhs);
void k_refine_finish(Ctx& c, int nrhs);
void k_refine_gather(Ctx& c, int nrhs);
void k_kkt_matvec_only(Ctx& c, int q);
void k_refine_init_one(Ctx& c, int q);
void k_copy(Ctx& c, const double* src, double* dst, int64_t n);
int factor_grid(Ctx& c);
int solve_grid(Ctx& c);
void k_warm_grids();

int occupancy_blocks(const void* kernel, int threads) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& e : cache)
        if (e.first == kernel) return e.second;
    static const bool plain = getenv("CIPM_RED_GRID_PLAIN") != nullptr;   // A/B probe: the 1184-block grid
    if (plain) return kMaxRedBlocks;
    int dev = 0, sms = 148, per_sm = 8;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int blocks = per_sm * sms;
    cache.emplace_back(kernel, blocks);
    return blocks;
}
}  // namespace cipm

using namespace cipm;

struct cipm_symbolic {
    Symbolic s;
};

struct cipm_ctx {
    Ctx c;
};

namespace {

// every host<->device copy goes through the context's stream: the stream is
// non-blocking, so a legacy-default-stream cudaMemcpy is NOT ordered after the
// allocation memsets / kernels queued on it (and could be zeroed by a later memset)
cudaError_t copy_sync(Ctx& c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c.stream);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(c.stream);
}

template <typename T>
int dalloc(Ctx& c, T** p, int64_t count) {
    *p = nullptr;
    size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
    cudaError_t e = cudaMalloc((void**)p, bytes);
    if (e != cudaSuccess) {
        fprintf(stderr, "[cipm] cudaMalloc(%zu) failed: %s\n", bytes, cudaGetErrorString(e));
        return CIPM_E_CUDA;
    }
    c.allocations.push_back((void*)*p);
    cudaMemsetAsync(*p, 0, bytes, c.stream);
    return CIPM_OK;
}

template <typename T, typename S>
int upload(Ctx& c, T** p, const S* host, int64_t count) {
    int rc = dalloc(c, p, count);
    if (rc) return rc;
    if (count <= 0) return CIPM_OK;
    std::vector<T> tmp((size_t)count);
    for (int64_t i = 0; i < count; ++i) tmp[i] = (T)host[i];
    CIPM_CUDA(copy_sync(c, *p, tmp.data(), sizeof(T) * count, cudaMemcpyHostToDevice));
    return CIPM_OK;
}

int sync_err(Ctx& c) {
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    CIPM_CUDA(cudaGetLastError());
    CIPM_CUDA(copy_sync(c, c.h_err, c.err, sizeof(int), cudaMemcpyDeviceToHost));
    return *c.h_err;
}

int read_sc(Ctx& c) {
    c.d2h_bytes += sizeof(double) * CIPM_SC_COUNT + sizeof(int);
    CIPM_CUDA(cudaMemcpyAsync(c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost, c.stream));
    CIPM_CUDA(cudaMemcpyAsync(c.h_err, c.err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    CIPM_CUDA(cudaGetLastError());
    return *c.h_err;
}

// refined solve of rb[q], q < nrhs; result in rbest[q] (kkt/system.py:279-314).
// Default: the whole refinement loop (t_max steps) is one CUDA graph per
// right-hand-side count; convergence / stall flags live on the device and the
// kernels of a finished right-hand side return immediately, so the host reads
// the state once at the end.  With profiling or tracing on, the eager loop
// below runs instead (per-step host decisions, per-launch events).
int refine_graph(Ctx& c, int nrhs, int* steps_out) {
    if (!c.refine_graph[nrhs]) {
        // graph = one WHILE conditional node; its body is one refinement step
        // (solve + residual + controller for every right-hand side) followed by
        // a 1-thread kernel that sets the loop condition from the device state
        cudaGraph_t g = nullptr;
        CIPM_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CIPM_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CIPM_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        const int64_t l0 = c.launches;
        CIPM_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        int active[2] = {1, nrhs > 1 ? 1 : 0};
        k_refine_step(c, nrhs, active, !c.resid_gathers);
        k_kkt_residual(c, nrhs);
        k_refine_continue(c, h, nrhs);
        cudaGraph_t captured = nullptr;
        cudaError_t e = cudaStreamEndCapture(c.stream, &captured);
        if (e != cudaSuccess) {
            fprintf(stderr, "[cipm] refinement graph capture failed: %s\n", cudaGetErrorString(e));
            cudaGraphDestroy(g);
            return CIPM_E_CUDA;
        }
        CIPM_CUDA(cudaGraphInstantiate(&c.refine_graph[nrhs], g, 0));
        cudaGraphDestroy(g);
        c.refine_graph_launches[nrhs] = c.launches - l0;
        c.launches = l0;
    }
    for (int q = 0; q < nrhs; ++q) k_refine_init_one(c, q);
    if (c.resid_gathers) k_refine_gather(c, nrhs);
    CIPM_CUDA(cudaMemsetAsync(c.refine_iter, 0, sizeof(int), c.stream));
    CIPM_CUDA(cudaGraphLaunch(c.refine_graph[nrhs], c.stream));
    k_refine_finish(c, nrhs);
    c.d2h_bytes += sizeof(double) * 16 + sizeof(int);
    CIPM_CUDA(cudaMemcpyAsync(c.h_rstate, c.rstate, sizeof(double) * 16, cudaMemcpyDeviceToHost, c.stream));
    CIPM_CUDA(cudaMemcpyAsync(c.h_err, c.err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (*c.h_err) return *c.h_err;
    int steps = (int)c.h_rstate[6];
    if (nrhs > 1) steps = std::max(steps, (int)c.h_rstate[14]);
    c.launches += c.refine_graph_launches[nrhs] * steps;
    if (steps_out) *steps_out = steps;
    c.h_sc[CIPM_SC_REFINE_STEPS] = steps;
    return CIPM_OK;
}

int refine(Ctx& c, int nrhs, int* steps_out) {
    if (c.use_graphs && !c.profile && !c.trace) return refine_graph(c, nrhs, steps_out);
    for (int q = 0; q < nrhs; ++q) k_refine_init_one(c, q);
    if (c.resid_gathers) k_refine_gather(c, nrhs);
    int active[2] = {1, nrhs > 1 ? 1 : 0};
    int steps = 0;
    for (int step = 1; step <= c.refine_max; ++step) {
        k_refine_step(c, nrhs, active, !c.resid_gathers);
        k_kkt_residual(c, nrhs);
        c.d2h_bytes += sizeof(double) * 16 + sizeof(int);
        CIPM_CUDA(cudaMemcpyAsync(c.h_rstate, c.rstate, sizeof(double) * 16, cudaMemcpyDeviceToHost, c.stream));
        CIPM_CUDA(cudaMemcpyAsync(c.h_err, c.err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        CIPM_CUDA(cudaStreamSynchronize(c.stream));
        if (*c.h_err) return *c.h_err;
        steps = step;
        bool any = false;
        for (int q = 0; q < nrhs; ++q) {
            if (active[q] && c.h_rstate[8 * q + 4] != 0.0) active[q] = 0;
            any = any || active[q];
        }
        if (!any) break;
    }
    k_refine_finish(c, nrhs);
    if (steps_out) *steps_out = steps;
    c.h_sc[CIPM_SC_REFINE_STEPS] = steps;
    return CIPM_OK;
}

int step_length(Ctx& c, int which) {
    k_step_init(c, which);
    k_step_bound(c, c.dz[which], c.ds[which]);
    k_step_finish(c, which);
    if (c.nsym) {
        for (int batch = 0; batch < 8; ++batch) {
            CIPM_CUDA(cudaMemsetAsync(c.mask, 0xff, sizeof(unsigned int), c.stream));
            k_nsym_feasible_mask(c, c.dz[which], c.ds[which], 32 * batch);
            k_nsym_resolve(c);
            int e = read_sc(c);
            if (e) return e;
            if (c.h_sc[CIPM_SC_T7] == 0.0) break;
        }
    }
    k_step_store(c, which);
    return CIPM_OK;
}

// one graph holding a single device WHILE node (default condition 1: the body runs at
// least once); body(h) enqueues the body's kernels, the last of which sets the condition
template <typename F>
int while_graph(Ctx& c, cudaGraphExec_t* exec, int64_t* body_launches, F&& body) {
    cudaGraph_t g = nullptr;
    CIPM_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CIPM_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CIPM_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t bodyg = np.conditional.phGraph_out[0];
    const int64_t l0 = c.launches;
    CIPM_CUDA(cudaStreamBeginCaptureToGraph(c.stream, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    body(h);
    cudaGraph_t captured = nullptr;
    cudaError_t e = cudaStreamEndCapture(c.stream, &captured);
    if (e != cudaSuccess) {
        fprintf(stderr, "[cipm] WHILE graph capture failed: %s\n", cudaGetErrorString(e));
        cudaGraphDestroy(g);
        return CIPM_E_CUDA;
    }
    CIPM_CUDA(cudaGraphInstantiate(exec, g, 0));
    cudaGraphDestroy(g);
    *body_launches = c.launches - l0;
    c.launches = l0;
    return CIPM_OK;
}

// refined solve without host readback (device loop): steps into a scalar slot
int refine_async(Ctx& c, int nrhs, int slot) {
    int tmp = 0;
    if (!c.refine_graph[nrhs]) {
        // build it through the synchronous path once (instantiation only happens there)
        int e = refine_graph(c, nrhs, &tmp);
        if (e) return e;
        k_refine_steps_store(c, nrhs, slot);
        return CIPM_OK;
    }
    for (int q = 0; q < nrhs; ++q) k_refine_init_one(c, q);
    if (c.resid_gathers) k_refine_gather(c, nrhs);
    CIPM_CUDA(cudaMemsetAsync(c.refine_iter, 0, sizeof(int), c.stream));
    CIPM_CUDA(cudaGraphLaunch(c.refine_graph[nrhs], c.stream));
    k_refine_finish(c, nrhs);
    c.launches += c.refine_graph_launches[nrhs] * 2;   // typical step count (the exact count is on the device)
    k_refine_steps_store(c, nrhs, slot);
    return CIPM_OK;
}

int64_t g_step_body_launches = 0, g_nb_body_launches = 0;

// step_length (steps.py:79-116) with the exp/pow backtracking as a device WHILE loop
int step_length_async(Ctx& c, int which) {
    k_step_init(c, which);
    k_step_bound(c, c.dz[which], c.ds[which]);
    k_step_finish(c, which);
    if (c.nsym) {
        if (!c.step_graph[which]) {
            int e = while_graph(c, &c.step_graph[which], &g_step_body_launches, [&](cudaGraphConditionalHandle h) {
                k_nsym_feasible_mask(c, c.dz[which], c.ds[which], 0);
                k_nsym_resolve_cond(c, h);
            });
            if (e) return e;
        }
        k_mask_init(c);
        CIPM_CUDA(cudaGraphLaunch(c.step_graph[which], c.stream));
        c.launches += g_step_body_launches;
    }
    k_step_store(c, which);
    return CIPM_OK;
}

// combined_step_size neighbourhood backtracking (ipm.py:350-366) as a device WHILE loop
int neighborhood_async(Ctx& c) {
    const int nk = 8;
    if (!c.nb_graph) {
        int e = while_graph(c, &c.nb_graph, &g_nb_body_launches, [&](cudaGraphConditionalHandle h) {
            k_mu_candidates(c, 0, nk);
            k_neighborhood_mask(c, 0, nk);
            k_nb_resolve_cond(c, nk, h);
        });
        if (e) return e;
    }
    k_mask_init(c);
    CIPM_CUDA(cudaGraphLaunch(c.nb_graph, c.stream));
    c.launches += g_nb_body_launches;
    return CIPM_OK;
}

}  // namespace

extern "C" {

int cipm_version(void) { return 100; }

int cipm_min_degree(int64_t dim, const int64_t* rowptr, const int64_t* colidx, int32_t* perm) {
    // treat the pattern as K with n = dim, m = 0 and no blocks: the graph is the symmetrised pattern
    SymbolicOptions opt;
    Symbolic s;
    std::vector<int64_t> arp(1, 0);
    int rc = analyze(dim, 0, rowptr, colidx, arp.data(), nullptr, 0, 0, nullptr, nullptr, opt, s);
    if (rc) return rc;
    for (int64_t k = 0; k < dim; ++k) perm[k] = s.md_perm[k];
    return CIPM_OK;
}

static void blocks_of(const cipm_problem_desc* d, std::vector<int64_t>& off, std::vector<int64_t>& dim) {
    for (int64_t i = 0; i < d->n_soc; ++i) { off.push_back(d->soc_off[i]); dim.push_back(d->soc_dim[i]); }
    for (int64_t i = 0; i < d->n_exp; ++i) { off.push_back(d->exp_off[i]); dim.push_back(3); }
    for (int64_t i = 0; i < d->n_pow; ++i) { off.push_back(d->pow_off[i]); dim.push_back(3); }
    for (int64_t i = 0; i < d->n_psd; ++i) {
        off.push_back(d->psd_off[i]);
        dim.push_back(d->psd_side[i] * (d->psd_side[i] + 1) / 2);
    }
}

int cipm_symbolic_create(const cipm_problem_desc* d, int ordering, cipm_symbolic** out) {
    return cipm_symbolic_create_ex(d, ordering, 0, out);
}

int cipm_symbolic_create_ex(const cipm_problem_desc* d, int ordering, int64_t nd_leaf, cipm_symbolic** out) {
    CIPM_NVTX("cipm_symbolic_create_ex");
    if (!d || !out || ordering < 0 || ordering > 4 || nd_leaf < 0) return CIPM_E_ARG;
    auto* h = new cipm_symbolic();
    std::vector<int64_t> off, dim;
    blocks_of(d, off, dim);
    SymbolicOptions opt;
    opt.ordering = ordering;
    if (nd_leaf > 0) opt.nd_leaf = nd_leaf;
    int rc = analyze(d->n, d->m, d->p_rowptr, d->p_colidx, d->a_rowptr, d->a_colidx, d->zero_dim + d->nonneg_dim,
                     (int64_t)off.size(), off.data(), dim.data(), opt, h->s);
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return CIPM_OK;
}

int cipm_symbolic_info_get(const cipm_symbolic* sym, cipm_symbolic_info* info) {
    if (!sym || !info) return CIPM_E_ARG;
    const Symbolic& s = sym->s;
    info->dim = s.dim;
    info->nsuper = s.nsuper;
    info->nnz_l = s.nnz_l;
    info->nnz_storage = s.nnz_storage;
    info->n_updates = s.n_updates;
    info->max_width = s.max_width;
    info->max_rows = s.max_rows;
    info->height = s.height;
    info->flops = s.flops;
    info->ordering = s.ordering_used;
    return CIPM_OK;
}

int cipm_symbolic_array(const cipm_symbolic* sym, const char* name, void* dst, int64_t* count) {
    if (!sym || !name) return CIPM_E_ARG;
    const Symbolic& s = sym->s;
    std::string nm(name);
    const void* src = nullptr;
    int64_t cnt = 0;
    size_t es = 0;
#define ARR(NAME, VEC)                                           \
    if (nm == NAME) { src = VEC.data(); cnt = (int64_t)VEC.size(); es = sizeof(VEC[0]); }
    ARR("perm", s.perm)
    ARR("md_perm", s.md_perm)
    ARR("sn_col", s.sn_col)
    ARR("sn_rptr", s.sn_rptr)
    ARR("sn_rows", s.sn_rows)
    ARR("sn_loff", s.sn_loff)
    ARR("sn_parent", s.sn_parent)
    ARR("upd_ptr", s.upd_ptr)
    ARR("upd_src", s.upd_src)
    ARR("upd_p0", s.upd_p0)
    ARR("upd_p1", s.upd_p1)
    ARR("order", s.order)
    ARR("map_p", s.map_p)
    ARR("map_a", s.map_a)
    ARR("map_diag", s.map_diag)
    ARR("map_hblk", s.map_hblk)
    ARR("cb_off", s.cb_off)
    ARR("push_pos", s.push_pos)
    ARR("irow_ptr", s.irow_ptr)
    ARR("inbox_tgt", s.inbox_tgt)
    ARR("cv_off", s.cv_off)
    ARR("vpush_pos", s.vpush_pos)
    ARR("vcol_ptr", s.vcol_ptr)
    ARR("vt_lo", s.vt_lo)
    ARR("vt_hi", s.vt_hi)
    ARR("vn_lo", s.vn_lo)
    ARR("vn_hi", s.vn_hi)
    ARR("tfold_cols", s.tfold_cols)
    ARR("tier", s.tier)
    ARR("level", s.level)
    ARR("desc32", s.desc32)
    ARR("tiny", s.tiny)
#undef ARR
    if (!es) return CIPM_E_ARG;
    if (count) *count = cnt;
    if (dst && cnt) memcpy(dst, src, es * (size_t)cnt);
    return CIPM_OK;
}

void cipm_symbolic_destroy(cipm_symbolic* sym) { delete sym; }

int cipm_ctx_create(const cipm_problem_desc* d, const cipm_symbolic* symh, const cipm_settings* st, cipm_ctx** out) {
    CIPM_NVTX("cipm_ctx_create");
    if (!d || !symh || !st || !out) return CIPM_E_ARG;
    for (int64_t i = 0; i < d->n_psd; ++i)
        if (d->psd_side[i] > 32) {      // problem.py:36 PSD_MAX_SIDE (one warp per cone, lane = row)
            fprintf(stderr, "[cipm] PSD side %lld > 32 exceeds the reference's limit\n", (long long)d->psd_side[i]);
            return CIPM_E_ARG;
        }
    auto* h = new cipm_ctx();
    Ctx& c = h->c;
    c.device = st->device;
    CIPM_CUDA(cudaSetDevice(c.device));
    if (st->stream) {
        c.stream = (cudaStream_t)st->stream;
    } else {
        // highest priority: the critical path of the dense tail (diagonal blocks, next
        // panel) is preferred over the side streams' bulk work
        int lo = 0, hi = 0;
        CIPM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CIPM_CUDA(cudaStreamCreateWithPriority(&c.stream, cudaStreamNonBlocking, hi));
        c.own_stream = true;
    }
    c.n = d->n;
    c.m = d->m;
    c.dim = d->n + d->m;
    c.precision = st->precision;
    c.delta_s = st->delta_s;
    c.delta_d = st->delta_d;
    c.beta = st->beta;
    c.backtrack = st->backtrack;
    c.step_scale = st->step_scale;
    c.refine_abs = st->refine_abs;
    c.refine_rel = st->refine_rel;
    c.refine_max = st->refine_max;
    if (const char* e = getenv("CIPM_NO_GRAPHS")) c.use_graphs = atoi(e) == 0;
    c.zero_dim = d->zero_dim;
    c.nonneg_dim = d->nonneg_dim;
    c.lin = d->zero_dim + d->nonneg_dim;
    c.nsoc = d->n_soc;
    c.nexp = d->n_exp;
    c.npow = d->n_pow;
    c.npsd = d->n_psd;
    c.nsym = c.nexp + c.npow;
    c.p_nnz = d->p_rowptr[d->n];
    c.a_nnz = d->a_rowptr[d->m];
    int rc = 0;
#define TRY(x)                  \
    do {                        \
        rc = (x);               \
        if (rc) {               \
            cipm_ctx_destroy(h); \
            return rc;          \
        }                       \
    } while (0)

    // cone tables
    std::vector<int64_t> soc_h(c.nsoc), psd_m(c.npsd), psd_l(c.npsd), psd_h(c.npsd);
    int64_t hp = 0;
    c.soc_rows = 0;
    int64_t soc_maxd = 0;
    for (int64_t i = 0; i < c.nsoc; ++i) {
        soc_h[i] = hp;
        hp += d->soc_dim[i] * (d->soc_dim[i] + 1) / 2;
        c.soc_rows += d->soc_dim[i];
        soc_maxd = std::max<int64_t>(soc_maxd, d->soc_dim[i]);
    }
    c.nsym_hbase = hp;
    hp += 6 * c.nsym;
    int64_t mp = 0, lp = 0;
    c.psd_max_side = 0;
    double psd_deg = 0;
    for (int64_t i = 0; i < c.npsd; ++i) {
        int64_t sd = d->psd_side[i];
        psd_m[i] = mp;
        psd_l[i] = lp;
        psd_h[i] = hp;
        mp += sd * sd;
        lp += sd;
        int64_t tdim = sd * (sd + 1) / 2;
        hp += tdim * (tdim + 1) / 2;
        c.psd_max_side = std::max<int>(c.psd_max_side, (int)sd);
        psd_deg += (double)sd;
    }
    // lanes per SOC cone (entries 1..d-1 strided over the group): 8 up to 17 rows
    c.soc_group = soc_maxd <= 17 ? 8 : (soc_maxd <= 33 ? 16 : 32);
    if (getenv("CIPM_SOC_WARP")) c.soc_group = 32;
    c.hblk_total = hp;
    {
        // dense H blocks in hv (SOC, exp, pow, PSD): row offset, size, packed upper start
        std::vector<int32_t> bo, bdim;
        std::vector<int64_t> bh;
        for (int64_t i = 0; i < c.nsoc; ++i) { bo.push_back((int32_t)d->soc_off[i]); bdim.push_back((int32_t)d->soc_dim[i]); bh.push_back(soc_h[i]); }
        for (int64_t i = 0; i < d->n_exp; ++i) { bo.push_back((int32_t)d->exp_off[i]); bdim.push_back(3); bh.push_back(c.nsym_hbase + 6 * i); }
        for (int64_t i = 0; i < d->n_pow; ++i) { bo.push_back((int32_t)d->pow_off[i]); bdim.push_back(3); bh.push_back(c.nsym_hbase + 6 * (d->n_exp + i)); }
        for (int64_t i = 0; i < c.npsd; ++i) {
            const int64_t sd = d->psd_side[i];
            bo.push_back((int32_t)d->psd_off[i]); bdim.push_back((int32_t)(sd * (sd + 1) / 2)); bh.push_back(psd_h[i]);
        }
        c.nblk = (int64_t)bo.size();
        if (c.nblk) {
            TRY(upload(c, &c.blk_off, bo.data(), c.nblk));
            TRY(upload(c, &c.blk_dim, bdim.data(), c.nblk));
            TRY(upload(c, &c.blk_hptr, bh.data(), c.nblk));
        }
    }
    {
        bool uni = c.npsd > 0 && c.psd_max_side <= 8 && !getenv("CIPM_PSD_WARP");
        for (int64_t i = 0; i < c.npsd && uni; ++i) uni = d->psd_side[i] == c.psd_max_side;
        c.psd_uni = uni ? c.psd_max_side : 0;
    }
    for (int64_t i = 0; i < c.nsoc; ++i) c.host_blocks.emplace_back(0, (int)d->soc_dim[i]);
    for (int64_t i = 0; i < c.npsd; ++i) c.host_blocks.emplace_back(3, (int)d->psd_side[i]);
    c.psd_mat_total = mp;
    c.psd_lam_total = lp;
    c.nu = (double)c.nonneg_dim + (double)c.nsoc + 3.0 * (double)c.nsym + psd_deg;
    TRY(upload(c, &c.soc_off, d->soc_off, c.nsoc));
    TRY(upload(c, &c.soc_dim, d->soc_dim, c.nsoc));
    TRY(upload(c, &c.soc_hptr, soc_h.data(), c.nsoc));
    TRY(upload(c, &c.exp_off, d->exp_off, c.nexp));
    TRY(upload(c, &c.pow_off, d->pow_off, c.npow));
    TRY(upload(c, &c.pow_alpha, d->pow_alpha, c.npow));
    TRY(upload(c, &c.psd_off, d->psd_off, c.npsd));
    TRY(upload(c, &c.psd_side, d->psd_side, c.npsd));
    TRY(upload(c, &c.psd_mptr, psd_m.data(), c.npsd));
    TRY(upload(c, &c.psd_lptr, psd_l.data(), c.npsd));
    TRY(upload(c, &c.psd_hptr, psd_h.data(), c.npsd));

    // problem patterns (+ transpose of A)
    TRY(upload(c, &c.p_rp, d->p_rowptr, c.n + 1));
    TRY(upload(c, &c.p_ci, d->p_colidx, c.p_nnz));
    TRY(dalloc(c, &c.p_v, c.p_nnz));
    TRY(upload(c, &c.a_rp, d->a_rowptr, c.m + 1));
    TRY(upload(c, &c.a_ci, d->a_colidx, c.a_nnz));
    TRY(dalloc(c, &c.a_v, c.a_nnz));
    {
        std::vector<int64_t> trp(c.n + 1, 0), tci(c.a_nnz), tsrc(c.a_nnz);
        for (int64_t p = 0; p < c.a_nnz; ++p) trp[d->a_colidx[p] + 1]++;
        for (int64_t j = 0; j < c.n; ++j) trp[j + 1] += trp[j];
        std::vector<int64_t> fill(trp.begin(), trp.end() - 1);
        for (int64_t r = 0; r < c.m; ++r)
            for (int64_t p = d->a_rowptr[r]; p < d->a_rowptr[r + 1]; ++p) {
                int64_t t = fill[d->a_colidx[p]]++;
                tci[t] = r;
                tsrc[t] = p;
            }
        TRY(upload(c, &c.at_rp, trp.data(), c.n + 1));
        TRY(upload(c, &c.at_ci, tci.data(), c.a_nnz));
        TRY(upload(c, &c.at_src, tsrc.data(), c.a_nnz));
        TRY(dalloc(c, &c.at_v, c.a_nnz));
    }
    TRY(dalloc(c, &c.q, c.n));
    TRY(dalloc(c, &c.b, c.m));
    TRY(dalloc(c, &c.a_user, c.a_nnz));
    TRY(dalloc(c, &c.b_user, c.m));
    TRY(dalloc(c, &c.p_user, c.p_nnz));
    TRY(dalloc(c, &c.q_user, c.n));
    TRY(dalloc(c, &c.a_src, c.a_nnz));
    TRY(dalloc(c, &c.b_src, c.m));
    TRY(dalloc(c, &c.eq_cnorm, c.n));
    TRY(dalloc(c, &c.eq_rnorm, c.m));
    TRY(dalloc(c, &c.eq_cstep, 10 * c.n));      // per Ruiz pass (replayed on q / b-only updates)
    TRY(dalloc(c, &c.eq_rstep, 10 * c.m));
    TRY(dalloc(c, &c.eq_p_ruiz, c.p_nnz));
    TRY(dalloc(c, &c.eq_cobj, 1));
    {
        std::vector<int64_t> bo, bd;
        blocks_of(d, bo, bd);
        c.eq_nblocks = (int64_t)bo.size();
        TRY(upload(c, &c.eq_boff, bo.data(), c.eq_nblocks));
        TRY(upload(c, &c.eq_bdim, bd.data(), c.eq_nblocks));
    }
    TRY(dalloc(c, &c.dr, c.m));
    TRY(dalloc(c, &c.dc, c.n));

    // iterate / work
    TRY(dalloc(c, &c.x, c.n));
    TRY(dalloc(c, &c.z, c.m));
    TRY(dalloc(c, &c.s, c.m));
    TRY(dalloc(c, &c.bx, c.n));
    TRY(dalloc(c, &c.bz, c.m));
    TRY(dalloc(c, &c.bs, c.m));
    TRY(dalloc(c, &c.gx, c.n));
    TRY(dalloc(c, &c.gz, c.m));
    for (int k = 0; k < 2; ++k) {
        TRY(dalloc(c, &c.dx[k], c.n));
        TRY(dalloc(c, &c.dz[k], c.m));
        TRY(dalloc(c, &c.ds[k], c.m));
    }
    TRY(dalloc(c, &c.col2, c.dim));
    TRY(dalloc(c, &c.sol1, c.dim));
    TRY(dalloc(c, &c.dsc, c.m));
    TRY(dalloc(c, &c.wn, c.n));
    TRY(dalloc(c, &c.wn2, c.n));
    TRY(dalloc(c, &c.wm, c.m));
    TRY(dalloc(c, &c.hv, c.hblk_total));

    // scaling state
    TRY(dalloc(c, &c.nn_h, c.nonneg_dim));
    TRY(dalloc(c, &c.nn_w, c.nonneg_dim));
    TRY(dalloc(c, &c.nn_lam, c.nonneg_dim));
    TRY(dalloc(c, &c.soc_w, c.soc_rows));
    TRY(dalloc(c, &c.soc_lam, c.soc_rows));
    TRY(dalloc(c, &c.soc_eta, c.nsoc));
    TRY(dalloc(c, &c.ns_h, 9 * c.nsym));
    TRY(dalloc(c, &c.ns_grad, 3 * c.nsym));
    TRY(dalloc(c, &c.ns_hess, 9 * c.nsym));
    TRY(dalloc(c, &c.ns_zt, 3 * c.nsym));
    TRY(dalloc(c, &c.psd_r, c.psd_mat_total));
    TRY(dalloc(c, &c.psd_rinv, c.psd_mat_total));
    TRY(dalloc(c, &c.psd_q, c.psd_mat_total));
    TRY(dalloc(c, &c.psd_lam, c.psd_lam_total));

    // symbolic -> device
    const Symbolic& S = symh->s;
    if (S.dim != c.dim) {
        cipm_ctx_destroy(h);
        return CIPM_E_DIM;
    }
    c.host_sym = S;
    c.sym.nsuper = S.nsuper;
    c.sym.nnz_storage = S.nnz_storage;
    TRY(upload(c, &c.sym.perm, S.perm.data(), c.dim));
    {
        std::vector<int32_t> ip(c.dim);
        for (int64_t k = 0; k < c.dim; ++k) ip[S.perm[k]] = (int32_t)k;
        TRY(upload(c, &c.sym.iperm, ip.data(), c.dim));
    }
    TRY(upload(c, &c.sym.sn_col, S.sn_col.data(), S.nsuper + 1));
    TRY(upload(c, &c.sym.sn_rptr, S.sn_rptr.data(), S.nsuper + 1));
    TRY(upload(c, &c.sym.sn_rows, S.sn_rows.data(), (int64_t)S.sn_rows.size()));
    TRY(upload(c, &c.sym.sn_loff, S.sn_loff.data(), S.nsuper + 1));
    TRY(upload(c, &c.sym.sn_parent, S.sn_parent.data(), S.nsuper));
    TRY(upload(c, &c.sym.sn_nchild, S.sn_nchild.data(), S.nsuper));
    TRY(upload(c, &c.sym.upd_ptr, S.upd_ptr.data(), S.nsuper + 1));
    TRY(upload(c, &c.sym.upd_src, S.upd_src.data(), (int64_t)S.upd_src.size()));
    TRY(upload(c, &c.sym.upd_p0, S.upd_p0.data(), (int64_t)S.upd_p0.size()));
    TRY(upload(c, &c.sym.upd_p1, S.upd_p1.data(), (int64_t)S.upd_p1.size()));
    TRY(upload(c, &c.sym.order, S.order.data(), S.nsuper));
    TRY(upload(c, &c.sym.sign, S.sign.data(), c.dim));
    TRY(upload(c, &c.sym.map_p, S.map_p.data(), (int64_t)S.map_p.size()));
    TRY(upload(c, &c.sym.map_a, S.map_a.data(), (int64_t)S.map_a.size()));
    TRY(upload(c, &c.sym.map_diag, S.map_diag.data(), c.dim));
    TRY(upload(c, &c.sym.map_hblk, S.map_hblk.data(), (int64_t)S.map_hblk.size()));
    TRY(upload(c, &c.sym.cb_off, S.cb_off.data(), S.nsuper + 1));
    TRY(upload(c, &c.sym.push_pos, S.push_pos.data(), (int64_t)S.push_pos.size()));
    TRY(upload(c, &c.sym.irow_ptr, S.irow_ptr.data(), (int64_t)S.irow_ptr.size()));
    TRY(upload(c, &c.sym.inbox_tgt, S.inbox_tgt.data(), (int64_t)S.inbox_tgt.size()));
    TRY(upload(c, &c.sym.cv_off, S.cv_off.data(), S.nsuper + 1));
    TRY(upload(c, &c.sym.vpush_pos, S.vpush_pos.data(), (int64_t)S.vpush_pos.size()));
    TRY(upload(c, &c.sym.vcol_ptr, S.vcol_ptr.data(), (int64_t)S.vcol_ptr.size()));
    TRY(upload(c, &c.sym.vt_lo, S.vt_lo.data(), (int64_t)S.vt_lo.size()));
    TRY(upload(c, &c.sym.vt_hi, S.vt_hi.data(), (int64_t)S.vt_hi.size()));
    TRY(upload(c, &c.sym.vn_lo, S.vn_lo.data(), (int64_t)S.vn_lo.size()));
    TRY(upload(c, &c.sym.vn_hi, S.vn_hi.data(), (int64_t)S.vn_hi.size()));
    TRY(upload(c, &c.sym.tfold_cols, S.tfold_cols.data(), (int64_t)S.tfold_cols.size()));
    c.sym.ntfold = (int64_t)S.tfold_cols.size();
    TRY(upload(c, &c.sym.desc32, S.desc32.data(), (int64_t)S.desc32.size()));
    TRY(upload(c, &c.sym.desc64, S.desc64.data(), (int64_t)S.desc64.size()));
    TRY(upload(c, &c.sym.need, S.need.data(), (int64_t)S.need.size()));
    TRY(upload(c, &c.sym.start_solve, S.start_solve.data(), (int64_t)S.start_solve.size()));
    TRY(upload(c, &c.sym.start_fac_warp, S.start_fac_warp.data(), (int64_t)S.start_fac_warp.size()));
    TRY(upload(c, &c.sym.start_fac_cta, S.start_fac_cta.data(), (int64_t)S.start_fac_cta.size()));
    TRY(upload(c, &c.sym.vin_col, S.vin_col.data(), (int64_t)S.vin_col.size()));
    TRY(upload(c, &c.sym.tiny, S.tiny.data(), (int64_t)S.tiny.size()));
    {
        const int64_t nt = (int64_t)S.tiny.size();
        std::vector<int32_t> td((size_t)std::max<int64_t>(nt, 1) * 4), tr((size_t)std::max<int64_t>(nt, 1));
        for (int64_t k = 0; k < nt; ++k) {
            const int32_t J = S.tiny[k];
            const int32_t w = S.sn_col[J + 1] - S.sn_col[J], r = (int32_t)(S.sn_rptr[J + 1] - S.sn_rptr[J]);
            if (S.sn_loff[J] > INT32_MAX || S.cv_off[J] > INT32_MAX) {
                cipm_ctx_destroy(h);
                return CIPM_E_DIM;
            }
            td[4 * k] = S.sn_col[J];
            td[4 * k + 1] = (int32_t)S.sn_loff[J];
            td[4 * k + 2] = (int32_t)S.cv_off[J];
            td[4 * k + 3] = w | (r << 8);
            tr[k] = (int32_t)S.sn_rptr[J];
        }
        int32_t* tdp = nullptr;
        TRY(upload(c, &tdp, td.data(), (int64_t)td.size()));
        c.sym.tdesc = reinterpret_cast<int4*>(tdp);
        TRY(upload(c, &c.sym.trptr, tr.data(), (int64_t)tr.size()));
    }
    TRY(upload(c, &c.sym.bwd_order, S.bwd_order.data(), (int64_t)S.bwd_order.size()));
    c.sym.ninbox = S.cb_off[S.nsuper];
    c.sym.nv = S.cv_off[S.nsuper];
    if ((int64_t)S.map_hblk.size() != c.hblk_total) {
        fprintf(stderr, "[cipm] H block map size mismatch (%zu vs %lld)\n", S.map_hblk.size(),
                (long long)c.hblk_total);
        cipm_ctx_destroy(h);
        return CIPM_E_DIM;
    }
    const size_t es = c.precision == CIPM_FULL ? sizeof(double) : sizeof(float);
    {
        void* p = nullptr;
        CIPM_CUDA(cudaMalloc(&p, es * std::max<int64_t>(S.nnz_storage, 1)));
        c.allocations.push_back(p);
        c.lval = p;
        CIPM_CUDA(cudaMalloc(&p, es * std::max<int64_t>(c.dim, 1)));
        c.allocations.push_back(p);
        c.dvec = p;
        CIPM_CUDA(cudaMalloc(&p, es * 2 * std::max<int64_t>(c.dim, 1)));
        c.allocations.push_back(p);
        c.rt = p;
        CIPM_CUDA(cudaMalloc(&p, es * std::max<int64_t>(c.sym.ninbox, 1)));
        c.allocations.push_back(p);
        c.inbox = p;
        CIPM_CUDA(cudaMalloc(&p, es * 2 * std::max<int64_t>(c.sym.nv, 1)));
        c.allocations.push_back(p);
        c.vin = p;
    }
    {
        int64_t inv_total = 0, flag_total = 0;
        tail_setup(c, &inv_total, &flag_total);
        size_t widest = 0;
        for (const auto& lv : c.tail_levels) widest = std::max(widest, lv.size());
        if (widest > 1) {
            const int P = (int)std::min<size_t>(widest, 8);
            c.tail_pool.resize(P);
            c.tail_pool_side.resize(P);
            c.tail_pool_ev.resize(4 * P);
            for (int k = 0; k < P; ++k) {
                CIPM_CUDA(cudaStreamCreateWithFlags(&c.tail_pool[k], cudaStreamNonBlocking));
                CIPM_CUDA(cudaStreamCreateWithFlags(&c.tail_pool_side[k], cudaStreamNonBlocking));
            }
            for (auto& e : c.tail_pool_ev) CIPM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CIPM_CUDA(cudaEventCreateWithFlags(&c.tail_fork, cudaEventDisableTiming));
        }
        void* p = nullptr;
        CIPM_CUDA(cudaMalloc(&p, es * std::max<int64_t>(inv_total, 1)));
        c.allocations.push_back(p);
        c.tinv = p;
        TRY(dalloc(c, &c.tflags, flag_total));
    }
    TRY(dalloc(c, &c.sf_flag, S.nsuper));    // zero: tiny leaves / tail never use the solve form
    if (const char* e = getenv("CIPM_SF_TAU")) c.sf_tau = atof(e);
    // the solve form pays off where the sweeps dominate (mixed precision: several refinement
    // steps per solve); in FP64 the extra pass costs more than the GEMV sweeps save
    c.solve_form = c.precision == CIPM_MIXED;
    if (const char* e = getenv("CIPM_SOLVE_FORM")) c.solve_form = atoi(e) != 0;
    TRY(dalloc(c, &c.fac_count, S.nsuper));
    TRY(dalloc(c, &c.bwd_done, S.nsuper));
    TRY(dalloc(c, &c.tickets, 8));
    TRY(dalloc(c, &c.refine_iter, 1));
    TRY(dalloc(c, &c.sn_maxd, S.nsuper));
    TRY(dalloc(c, &c.bumps, 1));
    TRY(dalloc(c, &c.rb, 2 * c.dim));
    TRY(dalloc(c, &c.rx, 2 * c.dim));
    TRY(dalloc(c, &c.rr, 2 * c.dim));
    TRY(dalloc(c, &c.rbest, 2 * c.dim));
    TRY(dalloc(c, &c.rstate, 16));
    TRY(dalloc(c, &c.partials, (int64_t)kMaxRedBlocks * 16));
    TRY(dalloc(c, &c.counter, 1));
    TRY(dalloc(c, &c.sc, CIPM_SC_COUNT));
    TRY(dalloc(c, &c.err, 1));
    TRY(dalloc(c, &c.nb, 64));
    TRY(dalloc(c, &c.mask, 4));
    CIPM_CUDA(cudaMallocHost((void**)&c.h_sc, sizeof(double) * CIPM_SC_COUNT));
    CIPM_CUDA(cudaMallocHost((void**)&c.h_err, sizeof(int)));
    CIPM_CUDA(cudaMallocHost((void**)&c.h_rstate, sizeof(double) * 16));
    for (int i = 0; i < 4; ++i) CIPM_CUDA(cudaEventCreate(&c.ev[i]));
    CIPM_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    CIPM_CUDA(cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming));
    CIPM_CUDA(cudaEventCreateWithFlags(&c.join_ev, cudaEventDisableTiming));
    CIPM_CUDA(cudaStreamCreateWithFlags(&c.tail_side, cudaStreamNonBlocking));
    for (auto& e : c.tail_ev) CIPM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.resid_gathers = fused_resid_ok(c) && !getenv("CIPM_NO_RESID_GATHER");
    c.factor_blocks = factor_grid(c);
    c.solve_blocks = solve_grid(c);
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    k_warm_grids();
    *out = h;
#undef TRY
    return CIPM_OK;
}

int cipm_ctx_set_values(cipm_ctx* h, const double* pv, const double* av, const double* q, const double* b,
                        const double* dr, const double* dc, double c_obj) {
    CIPM_NVTX("cipm_ctx_set_values");
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    c.eq_valid = false;                          // host-scaled values: no recorded Ruiz passes
    CIPM_CUDA(cudaSetDevice(c.device));
    if (c.p_nnz) CIPM_CUDA(cudaMemcpyAsync(c.p_v, pv, sizeof(double) * c.p_nnz, cudaMemcpyHostToDevice, c.stream));
    if (c.a_nnz) {
        CIPM_CUDA(cudaMemcpyAsync(c.a_v, av, sizeof(double) * c.a_nnz, cudaMemcpyHostToDevice, c.stream));
        std::vector<int64_t> src(c.a_nnz);
        CIPM_CUDA(copy_sync(c, src.data(), c.at_src, sizeof(int64_t) * c.a_nnz, cudaMemcpyDeviceToHost));
        std::vector<double> tv(c.a_nnz);
        for (int64_t t = 0; t < c.a_nnz; ++t) tv[t] = av[src[t]];
        CIPM_CUDA(copy_sync(c, c.at_v, tv.data(), sizeof(double) * c.a_nnz, cudaMemcpyHostToDevice));
    }
    CIPM_CUDA(cudaMemcpyAsync(c.q, q, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
    CIPM_CUDA(cudaMemcpyAsync(c.b, b, sizeof(double) * c.m, cudaMemcpyHostToDevice, c.stream));
    CIPM_CUDA(cudaMemcpyAsync(c.dr, dr, sizeof(double) * c.m, cudaMemcpyHostToDevice, c.stream));
    CIPM_CUDA(cudaMemcpyAsync(c.dc, dc, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
    c.c_obj = c_obj;
    c.h2d_bytes += (int64_t)sizeof(double) * (c.p_nnz + 2 * c.a_nnz + 2 * c.n + 2 * c.m);
    k_build_base(c);
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    return CIPM_OK;
}

int cipm_ctx_set_reorder(cipm_ctx* h, const int64_t* row_perm, const int64_t* a_src) {
    if (!h || (h->c.m && !row_perm) || (h->c.a_nnz && !a_src)) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaSetDevice(c.device));
    if (c.m) CIPM_CUDA(copy_sync(c, c.b_src, row_perm, sizeof(int64_t) * c.m, cudaMemcpyHostToDevice));
    if (c.a_nnz) CIPM_CUDA(copy_sync(c, c.a_src, a_src, sizeof(int64_t) * c.a_nnz, cudaMemcpyHostToDevice));
    c.have_reorder = true;
    return CIPM_OK;
}

int cipm_ctx_set_problem(cipm_ctx* h, const double* p_values, const double* a_values, const double* q,
                         const double* b, int equilibrate) {
    CIPM_NVTX("cipm_ctx_set_problem");
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    if (!c.have_reorder) return CIPM_E_ARG;
    CIPM_CUDA(cudaSetDevice(c.device));
    // a NULL array keeps the raw values of the previous call (parametric re-solve:
    // only the changed arrays cross PCIe); the first call must pass all four
    const bool have = c.have_user_values;
    if (!have && ((!p_values && c.p_nnz) || (!a_values && c.a_nnz) || (!q && c.n) || (!b && c.m)))
        return CIPM_E_ARG;
    if (p_values && c.p_nnz) {
        CIPM_CUDA(cudaMemcpyAsync(c.p_user, p_values, sizeof(double) * c.p_nnz, cudaMemcpyHostToDevice, c.stream));
        c.h2d_bytes += (int64_t)sizeof(double) * c.p_nnz;
    }
    if (a_values && c.a_nnz) {
        CIPM_CUDA(cudaMemcpyAsync(c.a_user, a_values, sizeof(double) * c.a_nnz, cudaMemcpyHostToDevice, c.stream));
        c.h2d_bytes += (int64_t)sizeof(double) * c.a_nnz;
    }
    if (q && c.n) {
        CIPM_CUDA(cudaMemcpyAsync(c.q_user, q, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
        c.h2d_bytes += (int64_t)sizeof(double) * c.n;
    }
    if (b && c.m) {
        CIPM_CUDA(cudaMemcpyAsync(c.b_user, b, sizeof(double) * c.m, cudaMemcpyHostToDevice, c.stream));
        c.h2d_bytes += (int64_t)sizeof(double) * c.m;
    }
    c.have_user_values = true;
    // q / b-only update of an equilibrated problem: replay the recorded Ruiz passes
    const bool replay = equilibrate && c.eq_valid && !p_values && !a_values && !getenv("CIPM_NO_RUIZ_REPLAY");
    if (c.p_nnz && !replay)
        CIPM_CUDA(cudaMemcpyAsync(c.p_v, c.p_user, sizeof(double) * c.p_nnz, cudaMemcpyDeviceToDevice, c.stream));
    if (c.n) CIPM_CUDA(cudaMemcpyAsync(c.q, c.q_user, sizeof(double) * c.n, cudaMemcpyDeviceToDevice, c.stream));
    int rc = k_set_problem(c, equilibrate != 0, replay);
    if (rc) return rc;
    c.eq_valid = equilibrate != 0;
    CIPM_CUDA(cudaMemcpyAsync(&c.c_obj, c.eq_cobj, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    CIPM_CUDA(cudaGetLastError());
    return CIPM_OK;
}

int cipm_ctx_get_equilibration(cipm_ctx* h, double* d_row, double* d_col, double* c_obj) {
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (d_row && c.m) CIPM_CUDA(copy_sync(c, d_row, c.dr, sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    if (d_col && c.n) CIPM_CUDA(copy_sync(c, d_col, c.dc, sizeof(double) * c.n, cudaMemcpyDeviceToHost));
    if (c_obj) *c_obj = c.c_obj;
    c.d2h_bytes += (int64_t)sizeof(double) * ((d_row ? c.m : 0) + (d_col ? c.n : 0));
    return CIPM_OK;
}

void cipm_ctx_destroy(cipm_ctx* h) {
    if (!h) return;
    Ctx& c = h->c;
    cudaSetDevice(c.device);
    if (c.stream) cudaStreamSynchronize(c.stream);
    for (void* p : c.allocations) cudaFree(p);
    if (c.h_sc) cudaFreeHost(c.h_sc);
    if (c.h_err) cudaFreeHost(c.h_err);
    if (c.h_rstate) cudaFreeHost(c.h_rstate);
    for (int i = 0; i < 4; ++i)
        if (c.ev[i]) cudaEventDestroy(c.ev[i]);
    for (auto e : c.ev_pool) cudaEventDestroy(e);
    if (c.fork_ev) cudaEventDestroy(c.fork_ev);
    if (c.join_ev) cudaEventDestroy(c.join_ev);
    if (c.side) cudaStreamDestroy(c.side);
    for (auto e : c.tail_ev)
        if (e) cudaEventDestroy(e);
    if (c.tail_side) cudaStreamDestroy(c.tail_side);
    for (auto e : c.tail_pool_ev) cudaEventDestroy(e);
    for (auto st : c.tail_pool) cudaStreamDestroy(st);
    for (auto st : c.tail_pool_side) cudaStreamDestroy(st);
    if (c.tail_fork) cudaEventDestroy(c.tail_fork);
    for (auto& g : c.refine_graph)
        if (g) cudaGraphExecDestroy(g);
    if (c.factor_graph) cudaGraphExecDestroy(c.factor_graph);
    for (auto& g : c.step_graph)
        if (g) cudaGraphExecDestroy(g);
    if (c.nb_graph) cudaGraphExecDestroy(c.nb_graph);
    if (c.t_start) cudaEventDestroy(c.t_start);
    if (c.t_stop) cudaEventDestroy(c.t_stop);
    if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
    delete h;
}

int cipm_sync(cipm_ctx* h) {
    if (!h) return CIPM_E_ARG;
    return sync_err(h->c);
}

int cipm_device_bytes(const cipm_ctx* h, int64_t* bytes) {
    if (!h || !bytes) return CIPM_E_ARG;
    size_t f = 0, t = 0;
    cudaMemGetInfo(&f, &t);
    *bytes = (int64_t)(t - f);
    return CIPM_OK;
}

int cipm_init_iterate(cipm_ctx* h) {
    CIPM_NVTX("cipm_init_iterate");
    Ctx& c = h->c;
    CIPM_CUDA(cudaSetDevice(c.device));
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    k_init_iterate(c);
    return read_sc(c);
}

int cipm_residuals(cipm_ctx* h, double* out) {
    CIPM_NVTX("cipm_residuals");
    Ctx& c = h->c;
    k_residuals(c);
    int e = read_sc(c);
    if (out) memcpy(out, c.h_sc, sizeof(double) * CIPM_SC_COUNT);
    return e;
}

int cipm_save_best(cipm_ctx* h) {
    k_copy_best(h->c);
    return CIPM_OK;
}

int cipm_update_scaling(cipm_ctx* h) {
    CIPM_NVTX("cipm_update_scaling");
    k_update_scaling(h->c);
    return CIPM_OK;
}

int cipm_factor(cipm_ctx* h) {
    CIPM_NVTX("cipm_factor");
    Ctx& c = h->c;
    c.num_numeric++;
    // the whole factorisation (assembly, persistent tiers, dense tail) is a static
    // launch sequence: after one eager run it is captured once and replayed as a graph
    if (!c.use_graphs || c.profile || c.trace || c.factor_runs++ == 0) {
        k_assemble(c);
        return k_factor(c);
    }
    if (!c.factor_graph) {
        cudaGraph_t g = nullptr;
        const int64_t l0 = c.launches;
        CIPM_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
        k_assemble(c);
        k_factor(c);
        CIPM_CUDA(cudaStreamEndCapture(c.stream, &g));
        CIPM_CUDA(cudaGraphInstantiate(&c.factor_graph, g, 0));
        cudaGraphDestroy(g);
        c.factor_graph_launches = c.launches - l0;
        c.launches = l0;
    }
    CIPM_CUDA(cudaGraphLaunch(c.factor_graph, c.stream));
    c.launches += c.factor_graph_launches;
    return CIPM_OK;
}

int cipm_solve_affine(cipm_ctx* h, int* steps) {
    CIPM_NVTX("cipm_solve_affine");
    Ctx& c = h->c;
    k_affine_rhs(c);
    int e = refine(c, 2, steps);
    if (e) return e;
    k_copy(c, c.rbest, c.col2, c.dim);
    k_copy(c, c.rbest + c.dim, c.sol1, c.dim);
    k_directions_prep_den(c);
    k_recover_direction(c, 0, c.sol1, 0.0);
    return CIPM_OK;
}

int cipm_step_affine(cipm_ctx* h) { return step_length(h->c, 0); }

int cipm_solve_combined(cipm_ctx* h, int* steps) {
    CIPM_NVTX("cipm_solve_combined");
    Ctx& c = h->c;
    k_combined_ds(c, c.dz[0], c.ds[0]);
    k_combined_rhs(c);
    int e = refine(c, 1, steps);
    if (e) return e;
    k_copy(c, c.rbest, c.sol1, c.dim);
    k_recover_direction(c, 1, c.sol1, 0.0);
    return CIPM_OK;
}

int cipm_step_combined(cipm_ctx* h, double* alpha) {
    CIPM_NVTX("cipm_step_combined");
    Ctx& c = h->c;
    int e = step_length(c, 1);
    if (e) return e;
    const int nk = 8;
    for (int g0 = 0; g0 < 4096; g0 += nk) {
        k_mu_candidates(c, g0, nk);
        k_neighborhood_mask(c, g0, nk);
        k_nb_resolve(c, g0, nk);
        e = read_sc(c);
        if (e) return e;
        if (c.h_sc[CIPM_SC_T7] == 0.0) break;
    }
    if (alpha) *alpha = c.h_sc[CIPM_SC_ALPHA_FINAL];
    return CIPM_OK;
}

int cipm_take_step(cipm_ctx* h) {
    CIPM_NVTX("cipm_take_step");
    Ctx& c = h->c;
    k_take_step(c);
    return read_sc(c);
}

int cipm_loop_begin(cipm_ctx* h, double norm_q, double norm_b, double eps_feas, double eps_inf, int max_iter) {
    CIPM_NVTX("cipm_loop_begin");
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaSetDevice(c.device));
    c.loop_norm_q = norm_q;
    c.loop_norm_b = norm_b;
    c.loop_eps_feas = eps_feas;
    c.loop_eps_inf = eps_inf;
    c.loop_max_iter = max_iter;
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    k_init_iterate(c);
    k_loop_init(c);
    return CIPM_OK;
}

int cipm_loop_check(cipm_ctx* h, int iteration, double* sc_out) {
    CIPM_NVTX("cipm_loop_check");
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    k_residuals(c);
    k_iter_control(c, iteration);
    const int e = read_sc(c);                      // the one blocking read of the iteration
    if (sc_out) memcpy(sc_out, c.h_sc, sizeof(double) * CIPM_SC_COUNT);
    return e;
}

// CIPM_BODY_TIMING=1 (probes only): host enqueue time and device time of each
// segment of cipm_loop_body, on stderr (one line per iteration)
struct BodyTimer {
    Ctx& c;
    bool on;
    std::vector<std::pair<const char*, double>> host;
    std::vector<cudaEvent_t> ev;
    std::chrono::steady_clock::time_point t0;
    explicit BodyTimer(Ctx& cc) : c(cc) {
        static const bool env = getenv("CIPM_BODY_TIMING") != nullptr;
        on = env;
        if (on) mark("start");
    }
    void mark(const char* name) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        host.emplace_back(name, ev.empty() ? 0.0 : std::chrono::duration<double, std::micro>(t - t0).count());
        t0 = t;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, c.stream);
        ev.push_back(e);
    }
    ~BodyTimer() {
        if (!on) return;
        cudaEventSynchronize(ev.back());
        fprintf(stderr, "[body]");
        for (size_t k = 1; k < ev.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[k - 1], ev[k]);
            fprintf(stderr, " %s=%.0f/%.0f", host[k].first, host[k].second, ms * 1000.f);
        }
        fprintf(stderr, " (host/device us)\n");
        for (auto e : ev) cudaEventDestroy(e);
    }
};

int cipm_loop_body(cipm_ctx* h) {
    CIPM_NVTX("cipm_loop_body");
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    int e;
    const bool eager = !c.use_graphs || c.profile || c.trace;
    BodyTimer bt(c);
    k_update_scaling(c);
    bt.mark("scaling");
    e = cipm_factor(h);
    if (e) return e;
    bt.mark("factor");
    // affine direction (two right-hand sides: col2 and the affine RHS)
    k_affine_rhs(c);
    if (eager) {
        int steps = 0;
        e = refine(c, 2, &steps);
    } else {
        e = refine_async(c, 2, CIPM_SC_REF_STEPS_A);
    }
    if (e) return e;
    bt.mark("solve_a");
    k_copy(c, c.rbest, c.col2, c.dim);
    k_copy(c, c.rbest + c.dim, c.sol1, c.dim);
    k_directions_prep_den(c);
    k_recover_direction(c, 0, c.sol1, 0.0);
    e = eager ? step_length(c, 0) : step_length_async(c, 0);
    if (e) return e;
    bt.mark("step_a");
    // combined direction
    k_combined_ds(c, c.dz[0], c.ds[0]);
    k_combined_rhs(c);
    if (eager) {
        int steps = 0;
        e = refine(c, 1, &steps);
    } else {
        e = refine_async(c, 1, CIPM_SC_REF_STEPS_C);
    }
    if (e) return e;
    bt.mark("solve_c");
    k_copy(c, c.rbest, c.sol1, c.dim);
    k_recover_direction(c, 1, c.sol1, 0.0);
    if (eager) {
        double alpha = 0.0;
        e = cipm_step_combined(h, &alpha);
    } else {
        e = step_length_async(c, 1);
        if (!e) e = neighborhood_async(c);
    }
    if (e) return e;
    bt.mark("step_c");
    k_take_step(c);
    bt.mark("take");
    return CIPM_OK;
}

int cipm_read_scalars(cipm_ctx* h, double* out) {
    int e = read_sc(h->c);
    if (out) memcpy(out, h->c.h_sc, sizeof(double) * CIPM_SC_COUNT);
    return e;
}

int cipm_get_iterate(cipm_ctx* h, int which, double* x, double* z, double* s, double* tkm) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    c.d2h_bytes += (int64_t)sizeof(double) * ((x ? c.n : 0) + (z ? c.m : 0) + (s ? c.m : 0) + (tkm ? CIPM_SC_COUNT : 0));
    const double* px = which ? c.bx : c.x;
    const double* pz = which ? c.bz : c.z;
    const double* ps = which ? c.bs : c.s;
    if (x) CIPM_CUDA(copy_sync(c, x, px, sizeof(double) * c.n, cudaMemcpyDeviceToHost));
    if (z) CIPM_CUDA(copy_sync(c, z, pz, sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    if (s) CIPM_CUDA(copy_sync(c, s, ps, sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    if (tkm) {
        CIPM_CUDA(copy_sync(c, c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost));
        tkm[0] = c.h_sc[CIPM_SC_TAU];
        tkm[1] = c.h_sc[CIPM_SC_KAPPA];
        tkm[2] = c.h_sc[CIPM_SC_MU];
    }
    return CIPM_OK;
}

int cipm_get_solution(cipm_ctx* h, int which, int certificate, double* x, double* z, double* s, double* tkm) {
    CIPM_NVTX("cipm_get_solution");
    if (!h || (h && h->c.n && !x) || (h->c.m && (!z || !s))) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaSetDevice(c.device));
    double* out = c.rb;                          // refinement scratch, 2 (n + m) >= n + 2 m doubles
    k_recover_solution(c, which, certificate, out);
    CIPM_CUDA(cudaGetLastError());
    if (c.n) CIPM_CUDA(cudaMemcpyAsync(x, out, sizeof(double) * c.n, cudaMemcpyDeviceToHost, c.stream));
    if (c.m) {
        CIPM_CUDA(cudaMemcpyAsync(z, out + c.n, sizeof(double) * c.m, cudaMemcpyDeviceToHost, c.stream));
        CIPM_CUDA(cudaMemcpyAsync(s, out + c.n + c.m, sizeof(double) * c.m, cudaMemcpyDeviceToHost, c.stream));
    }
    if (tkm) CIPM_CUDA(cudaMemcpyAsync(c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost, c.stream));
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    c.d2h_bytes += (int64_t)sizeof(double) * (c.n + 2 * c.m + (tkm ? CIPM_SC_COUNT : 0));
    if (tkm) {
        const bool best = which != 0;
        tkm[0] = c.h_sc[best ? CIPM_SC_BEST_TAU : CIPM_SC_TAU];
        tkm[1] = c.h_sc[best ? CIPM_SC_BEST_KAPPA : CIPM_SC_KAPPA];
        tkm[2] = c.h_sc[best ? CIPM_SC_BEST_MU : CIPM_SC_MU];
    }
    return CIPM_OK;
}

int cipm_set_iterate(cipm_ctx* h, const double* x, const double* z, const double* s, const double* tkm) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (x) CIPM_CUDA(copy_sync(c, c.x, x, sizeof(double) * c.n, cudaMemcpyHostToDevice));
    if (z) CIPM_CUDA(copy_sync(c, c.z, z, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    if (s) CIPM_CUDA(copy_sync(c, c.s, s, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    if (tkm) {
        CIPM_CUDA(copy_sync(c, c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost));
        c.h_sc[CIPM_SC_TAU] = tkm[0];
        c.h_sc[CIPM_SC_KAPPA] = tkm[1];
        c.h_sc[CIPM_SC_MU] = tkm[2];
        CIPM_CUDA(copy_sync(c, c.sc, c.h_sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyHostToDevice));
    }
    return CIPM_OK;
}

int cipm_kkt_solve(cipm_ctx* h, const double* rhs, double* x, int* steps, double* residual) {
    CIPM_NVTX("cipm_kkt_solve");
    Ctx& c = h->c;
    CIPM_CUDA(cudaMemcpyAsync(c.rb, rhs, sizeof(double) * c.dim, cudaMemcpyHostToDevice, c.stream));
    int e = refine(c, 1, steps);
    if (e) return e;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    CIPM_CUDA(copy_sync(c, x, c.rbest, sizeof(double) * c.dim, cudaMemcpyDeviceToHost));
    if (residual) *residual = c.h_rstate[7];
    return CIPM_OK;
}

// KKTSystem seam (kkt/system.py:152-314): H from the host, K x, refined solves
// with the stall flag, refinement settings
int cipm_kkt_set_scaling(cipm_ctx* h, const double* diag, const double* blocks) {
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaSetDevice(c.device));
    if (c.nonneg_dim && diag)
        CIPM_CUDA(cudaMemcpyAsync(c.nn_h, diag + c.zero_dim, sizeof(double) * c.nonneg_dim, cudaMemcpyHostToDevice,
                                  c.stream));
    if (c.hblk_total && blocks)
        CIPM_CUDA(cudaMemcpyAsync(c.hv, blocks, sizeof(double) * c.hblk_total, cudaMemcpyHostToDevice, c.stream));
    c.h2d_bytes += (int64_t)sizeof(double) * (c.nonneg_dim + c.hblk_total);
    c.host_scaling = true;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    return CIPM_OK;
}

int cipm_kkt_matvec(cipm_ctx* h, const double* x, double* out) {
    if (!h || !x || !out) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaSetDevice(c.device));
    CIPM_CUDA(cudaMemcpyAsync(c.rx, x, sizeof(double) * c.dim, cudaMemcpyHostToDevice, c.stream));
    CIPM_CUDA(cudaMemsetAsync(c.rb, 0, sizeof(double) * c.dim, c.stream));
    CIPM_CUDA(cudaMemsetAsync(c.rstate, 0, sizeof(double) * 8, c.stream));   // rhs 0 active
    k_kkt_matvec_only(c, 0);                                                 // rr = 0 - K x
    std::vector<double> r(c.dim);
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    CIPM_CUDA(copy_sync(c, r.data(), c.rr, sizeof(double) * c.dim, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < c.dim; ++i) out[i] = -r[i];
    return CIPM_OK;
}

int cipm_kkt_solve_ex(cipm_ctx* h, const double* rhs, double* x, int* steps, double* residual, int* stalled) {
    int e = cipm_kkt_solve(h, rhs, x, steps, residual);
    if (e) return e;
    if (stalled) *stalled = h->c.h_rstate[4] == 2.0 ? 1 : 0;
    return CIPM_OK;
}

int cipm_set_refinement(cipm_ctx* h, double t_abs, double t_rel, int t_max) {
    if (!h || !(t_abs > 0.0) || !(t_rel > 0.0) || t_max < 1) return CIPM_E_ARG;
    Ctx& c = h->c;
    c.refine_abs = t_abs;
    c.refine_rel = t_rel;
    if (t_max != c.refine_max) {
        c.refine_max = t_max;
        for (auto& g : c.refine_graph)          // the step bound is captured in the graphs
            if (g) {
                cudaGraphExecDestroy(g);
                g = nullptr;
            }
    }
    return CIPM_OK;
}

int cipm_apply_h(cipm_ctx* h, const double* v, double* out) {
    Ctx& c = h->c;
    double *dv = nullptr, *dout = nullptr;
    CIPM_CUDA(cudaMalloc(&dv, sizeof(double) * std::max<int64_t>(c.m, 1)));
    CIPM_CUDA(cudaMalloc(&dout, sizeof(double) * std::max<int64_t>(c.m, 1)));
    CIPM_CUDA(copy_sync(c, dv, v, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    k_apply_h(c, dv, dout, 0.0, nullptr, 1.0);
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    CIPM_CUDA(copy_sync(c, out, dout, sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    cudaFree(dv);
    cudaFree(dout);
    return *c.h_err;
}

int cipm_scaling_values(cipm_ctx* h, double* diag, double* blocks) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (diag) {
        std::vector<double> tmp(c.lin, 0.0);
        if (c.nonneg_dim)
            CIPM_CUDA(copy_sync(c, tmp.data() + c.zero_dim, c.nn_h, sizeof(double) * c.nonneg_dim,
                                 cudaMemcpyDeviceToHost));
        memcpy(diag, tmp.data(), sizeof(double) * c.lin);
    }
    if (blocks && c.hblk_total) CIPM_CUDA(copy_sync(c, blocks, c.hv, sizeof(double) * c.hblk_total, cudaMemcpyDeviceToHost));
    return sync_err(c);
}

int cipm_get_direction(cipm_ctx* h, int combined, double* dx, double* dz, double* ds, double* dtk) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    const int w = combined ? 1 : 0;
    if (dx) CIPM_CUDA(copy_sync(c, dx, c.dx[w], sizeof(double) * c.n, cudaMemcpyDeviceToHost));
    if (dz) CIPM_CUDA(copy_sync(c, dz, c.dz[w], sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    if (ds) CIPM_CUDA(copy_sync(c, ds, c.ds[w], sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    if (dtk) {
        CIPM_CUDA(copy_sync(c, c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost));
        dtk[0] = c.h_sc[w ? CIPM_SC_DTAU_C : CIPM_SC_DTAU_A];
        dtk[1] = c.h_sc[w ? CIPM_SC_DKAPPA_C : CIPM_SC_DKAPPA_A];
    }
    return CIPM_OK;
}

int cipm_get_vector(cipm_ctx* h, const char* name, double* out, int64_t* count) {
    Ctx& c = h->c;
    std::string nm(name ? name : "");
    const double* src = nullptr;
    int64_t cnt = 0;
    if (nm == "x") { src = c.x; cnt = c.n; }
    else if (nm == "z") { src = c.z; cnt = c.m; }
    else if (nm == "s") { src = c.s; cnt = c.m; }
    else if (nm == "gx") { src = c.gx; cnt = c.n; }
    else if (nm == "gz") { src = c.gz; cnt = c.m; }
    else if (nm == "dsc") { src = c.dsc; cnt = c.m; }
    else if (nm == "col2") { src = c.col2; cnt = c.dim; }
    else if (nm == "sol1") { src = c.sol1; cnt = c.dim; }
    else if (nm == "nn_h") { src = c.nn_h; cnt = c.nonneg_dim; }
    else if (nm == "hv") { src = c.hv; cnt = c.hblk_total; }
    else return CIPM_E_ARG;
    if (count) *count = cnt;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (out && cnt) CIPM_CUDA(copy_sync(c, out, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    return CIPM_OK;
}

int cipm_soc_residuals(cipm_ctx* h, const double* x, double* out) {
    Ctx& c = h->c;
    double *dx = nullptr, *dout = nullptr;
    CIPM_CUDA(cudaMalloc(&dx, sizeof(double) * std::max<int64_t>(c.m, 1)));
    CIPM_CUDA(cudaMalloc(&dout, sizeof(double) * std::max<int64_t>(c.nsoc, 1)));
    CIPM_CUDA(copy_sync(c, dx, x, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    k_soc_residuals(c, dx, dout);
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (c.nsoc) CIPM_CUDA(copy_sync(c, out, dout, sizeof(double) * c.nsoc, cudaMemcpyDeviceToHost));
    cudaFree(dx);
    cudaFree(dout);
    return CIPM_OK;
}

// ---- kernel-level seams (tests: the reference's L1 functions one at a time) ----

int cipm_set_direction(cipm_ctx* h, int which, const double* dx, const double* dz, const double* ds,
                       const double* dtk) {
    if (!h || which < 0 || which > 1) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    if (dx && c.n) CIPM_CUDA(copy_sync(c, c.dx[which], dx, sizeof(double) * c.n, cudaMemcpyHostToDevice));
    if (dz && c.m) CIPM_CUDA(copy_sync(c, c.dz[which], dz, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    if (ds && c.m) CIPM_CUDA(copy_sync(c, c.ds[which], ds, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    if (dtk) {
        CIPM_CUDA(copy_sync(c, c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost));
        c.h_sc[which ? CIPM_SC_DTAU_C : CIPM_SC_DTAU_A] = dtk[0];
        c.h_sc[which ? CIPM_SC_DKAPPA_C : CIPM_SC_DKAPPA_A] = dtk[1];
        CIPM_CUDA(copy_sync(c, c.sc, c.h_sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyHostToDevice));
    }
    return CIPM_OK;
}

int cipm_step_length(cipm_ctx* h, int which, double* alpha) {
    if (!h || which < 0 || which > 1) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    int e = step_length(c, which);
    if (e) return e;
    e = read_sc(c);
    if (alpha) *alpha = c.h_sc[which ? CIPM_SC_ALPHA_C : CIPM_SC_ALPHA_A];
    return e;
}

int cipm_combined_ds(cipm_ctx* h, const double* dz_a, const double* ds_a, double sigma, double mu, double* out) {
    if (!h || !dz_a || !ds_a || !out) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    CIPM_CUDA(copy_sync(c, c.h_sc, c.sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyDeviceToHost));
    c.h_sc[CIPM_SC_SIGMA] = sigma;
    c.h_sc[CIPM_SC_MU] = mu;
    CIPM_CUDA(copy_sync(c, c.sc, c.h_sc, sizeof(double) * CIPM_SC_COUNT, cudaMemcpyHostToDevice));
    if (c.m) {
        CIPM_CUDA(copy_sync(c, c.dz[0], dz_a, sizeof(double) * c.m, cudaMemcpyHostToDevice));
        CIPM_CUDA(copy_sync(c, c.ds[0], ds_a, sizeof(double) * c.m, cudaMemcpyHostToDevice));
    }
    k_combined_ds(c, c.dz[0], c.ds[0]);
    int e = sync_err(c);
    if (c.m) CIPM_CUDA(copy_sync(c, out, c.dsc, sizeof(double) * c.m, cudaMemcpyDeviceToHost));
    return e;
}

int cipm_neighborhood_ok(cipm_ctx* h, double mu, double beta, int* ok) {
    if (!h || !ok || !(mu > 0.0)) return CIPM_E_ARG;
    Ctx& c = h->c;
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    if (c.m) {
        CIPM_CUDA(cudaMemsetAsync(c.dz[1], 0, sizeof(double) * c.m, c.stream));
        CIPM_CUDA(cudaMemsetAsync(c.ds[1], 0, sizeof(double) * c.m, c.stream));
    }
    const double beta0 = c.beta;
    c.beta = beta;
    k_mu_candidates(c, 0, 1, mu);
    k_neighborhood_mask(c, 0, 1);
    c.beta = beta0;
    unsigned int bits = 0;
    CIPM_CUDA(cudaMemcpyAsync(&bits, c.mask, sizeof(unsigned int), cudaMemcpyDeviceToHost, c.stream));
    int e = sync_err(c);
    *ok = (bits & 1u) ? 1 : 0;
    return e;
}

int cipm_membership(cipm_ctx* h, const double* s, const double* z, int* in_cone, int* in_dual) {
    if (!h) return CIPM_E_ARG;
    Ctx& c = h->c;
    for (int side = 0; side < 2; ++side) {
        const double* v = side == 0 ? s : z;
        int* flag = side == 0 ? in_cone : in_dual;
        if (!v || !flag) continue;
        // the other side is the unit point (interior of both the cone and its dual)
        CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
        k_init_iterate(c);
        if (c.m) CIPM_CUDA(copy_sync(c, side == 0 ? c.s : c.z, v, sizeof(double) * c.m, cudaMemcpyHostToDevice));
        k_membership(c);
        int e = sync_err(c);
        if (e != CIPM_OK && e != CIPM_E_INTERIOR) return e;
        *flag = e == CIPM_OK ? 1 : 0;
    }
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    return sync_err(c);
}

int cipm_kkt_counters(cipm_ctx* h, int64_t* out) {
    if (!h || !out) return CIPM_E_ARG;
    Ctx& c = h->c;
    int32_t bumps = 0;
    CIPM_CUDA(copy_sync(c, &bumps, c.bumps, sizeof(int32_t), cudaMemcpyDeviceToHost));
    out[0] = c.num_numeric;
    out[1] = bumps;
    return CIPM_OK;
}

// Kernel-class timing at the current iterate (bench roofline): CUDA events on the
// context stream around `reps` back-to-back launches of each class; out[2k] = ms
// per launch, out[2k+1] = algorithmic bytes per launch (SURVEY.md §8d formulas,
// 8-byte values, 4-byte indices).  Classes: 0 fused residual SpMV (resid_n +
// resid_m), 1 KKT refinement matvec r = b - K x (one right-hand side), 2-5 the
// scaling update of the nonneg / SOC / exp+pow / PSD family.
int cipm_kernel_classes(cipm_ctx* h, int reps, double* out) {
    if (!h || !out || reps < 1) return CIPM_E_ARG;
    Ctx& c = h->c;
    cudaEvent_t e0, e1;
    CIPM_CUDA(cudaEventCreate(&e0));
    CIPM_CUDA(cudaEventCreate(&e1));
    auto timed = [&](auto&& fn) -> double {
        fn();                                             // warm
        cudaEventRecord(e0, c.stream);
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1, c.stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        return (double)ms / reps;
    };
    const double n = (double)c.n, m = (double)c.m, dim = (double)c.dim;
    const double nnzp = (double)c.p_nnz, nnza = (double)c.a_nnz;
    for (int k = 0; k < 12; ++k) out[k] = 0.0;
    out[0] = timed([&] { k_residuals(c); });
    out[1] = 12.0 * (nnzp + 2.0 * nnza) + 8.0 * (3.0 * n + 4.0 * m);
    // one refinement matvec on right-hand side 0 (rstate forced active for the timing)
    CIPM_CUDA(cudaMemsetAsync(c.rstate, 0, sizeof(double) * 8, c.stream));
    out[2] = timed([&] { k_kkt_matvec_only(c, 0); });
    out[3] = 12.0 * (nnzp + 2.0 * nnza) + 8.0 * (double)c.hblk_total + 8.0 * (double)c.nonneg_dim + 24.0 * dim;
    // scaling families
    double soc_bytes = 0.0, psd_bytes = 0.0;
    {
        for (size_t i = 0; i < c.host_blocks.size(); ++i) {
            const double d = (double)c.host_blocks[i].second;
            const int kind = c.host_blocks[i].first;
            if (kind == 0) soc_bytes += 2 * 8 * d + 2 * 8 * d + 8 + 8 * d * (d + 1) / 2;
            if (kind == 3) {
                const double sd = d;                      // side
                const double sv = sd * (sd + 1) / 2;
                psd_bytes += 2 * 8 * sv + 3 * 8 * sd * sd + 8 * sd + 8 * sv * (sv + 1) / 2;
            }
        }
    }
    if (c.nonneg_dim) { out[4] = timed([&] { k_update_scaling_family(c, 0); }); out[5] = 40.0 * (double)c.nonneg_dim; }
    if (c.nsoc) { out[6] = timed([&] { k_update_scaling_family(c, 1); }); out[7] = soc_bytes; }
    if (c.nsym) { out[8] = timed([&] { k_update_scaling_family(c, 2); }); out[9] = 288.0 * (double)c.nsym; }
    if (c.npsd) { out[10] = timed([&] { k_update_scaling_family(c, 3); }); out[11] = psd_bytes; }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // timing only: a failure latched by the kernels at this iterate (e.g. the scaling
    // of a final exp/pow iterate that ended the solve) is not an error of this call
    const int e = sync_err(c);
    CIPM_CUDA(cudaMemsetAsync(c.err, 0, sizeof(int), c.stream));
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    return e == CIPM_E_CUDA ? e : CIPM_OK;
}

int cipm_io_bytes(cipm_ctx* h, int64_t* h2d, int64_t* d2h, int reset) {
    if (h2d) *h2d = h->c.h2d_bytes;
    if (d2h) *d2h = h->c.d2h_bytes;
    if (reset) h->c.h2d_bytes = h->c.d2h_bytes = 0;
    return CIPM_OK;
}

int cipm_launch_count(cipm_ctx* h, int64_t* count, int reset) {
    if (count) *count = h->c.launches;
    if (reset) h->c.launches = 0;
    return CIPM_OK;
}

int cipm_profile(cipm_ctx* h, int enable) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    c.profile = enable != 0;
    c.solve_rhs = 0;
    c.ev_factor.clear();
    c.ev_solve.clear();
    return CIPM_OK;
}

int cipm_kernel_stats(cipm_ctx* h, double* out) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    double fs = 0.0, ss = 0.0;
    for (auto& pr : c.ev_factor) {
        float ms = 0.f;
        CIPM_CUDA(cudaEventElapsedTime(&ms, c.ev_pool[pr.first], c.ev_pool[pr.second]));
        fs += ms;
    }
    for (auto& pr : c.ev_solve) {
        float ms = 0.f;
        CIPM_CUDA(cudaEventElapsedTime(&ms, c.ev_pool[pr.first], c.ev_pool[pr.second]));
        ss += ms;
    }
    out[0] = fs;
    out[1] = (double)c.ev_factor.size();
    out[2] = ss;
    out[3] = (double)c.ev_solve.size();
    out[4] = (double)c.solve_rhs;
    c.solve_rhs = 0;
    c.ev_factor.clear();
    c.ev_solve.clear();
    return CIPM_OK;
}

int cipm_timer(cipm_ctx* h, int op, double* ms) {
    Ctx& c = h->c;
    if (!c.t_start) {
        CIPM_CUDA(cudaEventCreate(&c.t_start));
        CIPM_CUDA(cudaEventCreate(&c.t_stop));
    }
    if (op == 0) {
        CIPM_CUDA(cudaEventRecord(c.t_start, c.stream));
        return CIPM_OK;
    }
    CIPM_CUDA(cudaEventRecord(c.t_stop, c.stream));
    CIPM_CUDA(cudaEventSynchronize(c.t_stop));
    float v = 0.f;
    CIPM_CUDA(cudaEventElapsedTime(&v, c.t_start, c.t_stop));
    if (ms) *ms = v;
    return CIPM_OK;
}

int cipm_trace(cipm_ctx* h, int enable, int64_t* out) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t cnt = 12 * (int64_t)c.sym.nsuper;
    if (enable) {
        if (!c.trace) {
            CIPM_CUDA(cudaMalloc(&c.trace, sizeof(int64_t) * cnt));
            c.allocations.push_back(c.trace);
        }
        CIPM_CUDA(cudaMemsetAsync(c.trace, 0, sizeof(int64_t) * cnt, c.stream));
        return CIPM_OK;
    }
    if (c.trace && out) CIPM_CUDA(copy_sync(c, out, c.trace, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost));
    c.trace = nullptr;   // stays allocated until destroy
    return CIPM_OK;
}

int cipm_kernel_times(cipm_ctx* h, double* factor_ms, double* solve_ms) {
    Ctx& c = h->c;
    CIPM_CUDA(cudaStreamSynchronize(c.stream));
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, c.ev[0], c.ev[1]) != cudaSuccess) a = -1.f;
    if (cudaEventElapsedTime(&b, c.ev[2], c.ev[3]) != cudaSuccess) b = -1.f;
    cudaGetLastError();
    if (factor_ms) *factor_ms = a;
    if (solve_ms) *solve_ms = b;
    return CIPM_OK;
}

}  // extern "C"
