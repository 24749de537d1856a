// Device-resident state of one problem instance (one cipm_ctx).
//
// HBM layout (structure of arrays, one flat buffer per field):
//   problem   P (CSR full), A (CSR), A' (CSR of the transpose), q, b, Dr, Dc
//   iterate   x (n), z (m), s (m), best copies, G rows, directions
//   scaling   nonneg h/w/λ (nnd); SOC w/λ (rows), η (cones);
//             exp/pow H(9)/∇f(3)/∇²f(9)/z̃(3) per cone; PSD R/R⁻¹/Q (side²), λ (side)
//   factor    supernodal panels (T = double | float), base image, D, schedule
//   scalars   Scalars block + error word + reduction partials
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "symbolic.hpp"

namespace cipm {

struct DevSymbolic {
    int32_t nsuper = 0;
    int32_t* perm = nullptr;        // dim: permuted position -> original index
    int32_t* iperm = nullptr;       // dim: original index -> permuted position
    int32_t* sn_col = nullptr;      // nsuper+1
    int64_t* sn_rptr = nullptr;     // nsuper+1
    int32_t* sn_rows = nullptr;
    int64_t* sn_loff = nullptr;     // nsuper+1
    int32_t* sn_parent = nullptr;
    int32_t* sn_nchild = nullptr;
    int64_t* upd_ptr = nullptr;
    int32_t* upd_src = nullptr;
    int32_t* upd_p0 = nullptr;
    int32_t* upd_p1 = nullptr;
    int32_t* order = nullptr;
    int8_t* sign = nullptr;         // permuted order
    int64_t* map_p = nullptr;
    int64_t* map_a = nullptr;
    int64_t* map_diag = nullptr;
    int64_t* map_hblk = nullptr;
    int64_t* cb_off = nullptr;
    int64_t* push_pos = nullptr;
    int64_t* irow_ptr = nullptr;
    int32_t* inbox_tgt = nullptr;
    int64_t* cv_off = nullptr;
    int32_t* vpush_pos = nullptr;    // int32 on the device (half the push-position traffic)
    int64_t* vcol_ptr = nullptr;
    int64_t *vt_lo = nullptr, *vt_hi = nullptr, *vn_lo = nullptr, *vn_hi = nullptr;
    int32_t* tfold_cols = nullptr;
    int64_t ntfold = 0;
    int32_t* desc32 = nullptr;
    int64_t* desc64 = nullptr;
    int32_t* need = nullptr;
    int32_t* start_solve = nullptr;
    int32_t* start_fac_warp = nullptr;
    int32_t* start_fac_cta = nullptr;
    uint8_t* vin_col = nullptr;
    int32_t* tiny = nullptr;
    int4* tdesc = nullptr;           // tiny leaves {c0, loff, cvo, w | r << 8}
    int32_t* trptr = nullptr;        // tiny leaves: sn_rptr
    int32_t* bwd_order = nullptr;
    int64_t nnz_storage = 0;
    int64_t ninbox = 0, nv = 0;
};

// one supernode of the dense tail (dense.cu), in topological order
struct TailNode {
    int32_t J = 0, c0 = 0, w = 0, r = 0, parent = -1, nbd = 0;
    int64_t r0 = 0, loff = 0, inv_off = 0, flag_off = 0;
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // side stream: the solve-form pass runs beside the dense tail factorisation
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // dense-tail look-ahead: the bulk of each trailing update runs on tail_side
    // while the next panel is factored on the main stream
    cudaStream_t tail_side = nullptr;
    cudaEvent_t tail_ev[3] = {nullptr, nullptr, nullptr};
    // independent tail nodes of one level run as parallel branches: slot k has a
    // main stream, a look-ahead side stream and 4 events (look-ahead x3, join)
    std::vector<std::vector<int>> tail_levels;
    std::vector<cudaStream_t> tail_pool, tail_pool_side;
    std::vector<cudaEvent_t> tail_pool_ev;
    cudaEvent_t tail_fork = nullptr;
    bool own_stream = false;
    int64_t n = 0, m = 0, dim = 0;
    int precision = CIPM_FULL;
    double delta_s = 1e-8, delta_d = 0.0, beta = 1e-6, backtrack = 0.8, step_scale = 0.99;
    double refine_abs = 1e-12, refine_rel = 1e-12;
    int refine_max = 10;
    int64_t zero_dim = 0, nonneg_dim = 0, lin = 0;
    int64_t nsoc = 0, nexp = 0, npow = 0, npsd = 0, soc_rows = 0, nsym = 0;
    int64_t psd_mat_total = 0, psd_lam_total = 0, hblk_total = 0;
    int psd_max_side = 0;
    int psd_uni = 0;
    // KKTSystem seam: H given by the host (cipm_kkt_set_scaling); the block tables of hv
    int32_t *blk_off = nullptr, *blk_dim = nullptr;
    int64_t* blk_hptr = nullptr;
    int64_t nblk = 0;
    bool host_scaling = false;
    int soc_group = 32;              // lanes per SOC cone: 8 / 16 / 32 by the largest SOC dimension                 // all PSD sides equal and <= 8: thread-per-cone kernels (psd_reg.cuh)
    double nu = 0.0;                 // barrier degree
    double c_obj = 1.0;
    int64_t p_nnz = 0, a_nnz = 0;

    // cone tables
    int32_t *soc_off = nullptr, *soc_dim = nullptr;      // row offsets (z coordinates)
    int64_t* soc_hptr = nullptr;                         // into map_hblk per SOC
    int32_t* exp_off = nullptr;
    int32_t* pow_off = nullptr;
    double* pow_alpha = nullptr;
    int32_t *psd_off = nullptr, *psd_side = nullptr;
    int64_t *psd_mptr = nullptr, *psd_lptr = nullptr, *psd_hptr = nullptr;
    int64_t nsym_hbase = 0;                              // map_hblk base of exp/pow blocks

    // problem data (scaled)
    int64_t *p_rp = nullptr, *p_ci = nullptr;
    double* p_v = nullptr;
    int64_t *a_rp = nullptr, *a_ci = nullptr;
    double* a_v = nullptr;
    int64_t *at_rp = nullptr, *at_ci = nullptr, *at_src = nullptr;
    double* at_v = nullptr;
    double *q = nullptr, *b = nullptr, *dr = nullptr, *dc = nullptr;
    // device-side setup (setup.cu): user-order raw values, reorder maps, Ruiz work
    double *a_user = nullptr, *b_user = nullptr;
    double *p_user = nullptr, *q_user = nullptr;   // raw user values (P, q are scaled in place)
    bool have_user_values = false;
    int64_t *a_src = nullptr, *b_src = nullptr;
    bool have_reorder = false;
    double *eq_cnorm = nullptr, *eq_rnorm = nullptr, *eq_cstep = nullptr, *eq_rstep = nullptr, *eq_cobj = nullptr;
    double* eq_p_ruiz = nullptr;   // Ruiz-scaled P before the cost scaling (q / b-only replay)
    bool eq_valid = false;         // eq_cstep / eq_rstep (10 passes) and eq_p_ruiz match the device P, A
    int32_t *eq_boff = nullptr, *eq_bdim = nullptr;
    int64_t eq_nblocks = 0;
    double one = 1.0;

    // iterate and work vectors
    double *x = nullptr, *z = nullptr, *s = nullptr;
    double *bx = nullptr, *bz = nullptr, *bs = nullptr;
    double best_tkm[3] = {0, 0, 0};
    double *gx = nullptr, *gz = nullptr;
    double *dx[2] = {nullptr, nullptr}, *dz[2] = {nullptr, nullptr}, *ds[2] = {nullptr, nullptr};
    double *col2 = nullptr, *sol1 = nullptr;             // dim each ([x; z] order)
    double* dsc = nullptr;                               // combined d_s (m)
    double *wn = nullptr, *wn2 = nullptr;                // n-sized scratch
    double* wm = nullptr;                                // m-sized scratch
    double* hv = nullptr;                                // upper triangles of every dense H block

    // scaling state
    double *nn_h = nullptr, *nn_w = nullptr, *nn_lam = nullptr;
    double *soc_w = nullptr, *soc_lam = nullptr, *soc_eta = nullptr;
    double *ns_h = nullptr, *ns_grad = nullptr, *ns_hess = nullptr, *ns_zt = nullptr;
    double *psd_r = nullptr, *psd_rinv = nullptr, *psd_q = nullptr, *psd_lam = nullptr;

    // factor
    Symbolic host_sym;               // copy kept for stats / host-side checks
    DevSymbolic sym;
    void* lval = nullptr;            // panels (T)
    void* dvec = nullptr;            // D (T), permuted order
    int32_t* fac_count = nullptr;    // children finished (factor / forward solve)
    int32_t* bwd_done = nullptr;     // backward solve completion flags
    int32_t* tickets = nullptr;      // [0] factor, [1] forward, [2] backward
    double* sn_maxd = nullptr;       // subtree max |D|
    int32_t* bumps = nullptr;
    void* inbox = nullptr;           // factor contribution inbox (T)
    void* vin = nullptr;             // solve contribution inbox, 2 x nv (T)
    int factor_blocks = 0, solve_blocks = 0, factor_smem = 0;
    int64_t factor_slice = 0;        // per-warp panel slice (elements) of the factor kernel
    int factor_cta_smem = 0, factor_cta_blocks = 0;   // mid-tier CTA kernel
    int64_t solve_slice = 0;         // per-warp panel slice (elements) of the solve kernels
    int64_t solve_form_slice = 0;    // per-warp panel slice of the solve-form pass
    int solve_form_blocks = 1;
    int solve_form_inv = 0;          // per-warp Linv buffer (max non-tail width squared)
    int8_t* sf_flag = nullptr;       // per supernode: panel in solve form (1) or plain L (0)
    double sf_tau = 16.0;            // growth bound max |L11^-1| for the solve form (CIPM_SF_TAU)
    bool solve_form = false;         // panels in solve form (default: mixed precision, CIPM_SOLVE_FORM)
    // dense tail (dense.cu)
    std::vector<TailNode> tail;
    void* tinv = nullptr;            // inverses of the 64x64 diagonal blocks (T)
    int32_t* tflags = nullptr;       // per tail node: fwd flags, bwd flags, 2 tickets
    int64_t tflag_total = 0;
    bool resid_gathers = false;      // LP/QP: the fused residual writes the permuted RHS (no gather pass)

    // refinement (up to 2 right-hand sides, [rhs][dim])
    double *rb = nullptr, *rx = nullptr, *rr = nullptr, *rbest = nullptr;
    void* rt = nullptr;              // permuted work vector (T)
    double* rstate = nullptr;        // per rhs: best, prev, ups, target, done, improved, steps, resid
    int32_t* rflags = nullptr;       // per rhs: active (host-visible via rstate)

    // reductions / scalars
    double* partials = nullptr;
    unsigned int* counter = nullptr;
    double* sc = nullptr;            // CIPM_SC_COUNT doubles
    int* err = nullptr;
    double* nb = nullptr;            // neighbourhood sums [2][32]
    unsigned int* mask = nullptr;    // candidate masks
    double* h_sc = nullptr;          // pinned host copy of sc
    int* h_err = nullptr;
    double* h_rstate = nullptr;

    int64_t launches = 0;
    int64_t h2d_bytes = 0, d2h_bytes = 0;   // host<->device traffic of the public API
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // profiling: CUDA-event pairs around every factorisation / triangular-solve launch
    bool profile = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_factor, ev_solve;
    int64_t solve_rhs = 0;            // right-hand sides processed by the profiled solve launches
    cudaEvent_t t_start = nullptr, t_stop = nullptr;
    float factor_ms = 0.f, solve_ms = 0.f;

    int64_t* trace = nullptr;        // cipm_trace: per-supernode timelines
    // refinement as one CUDA graph per right-hand-side count (device-side convergence flags)
    cudaGraphExec_t refine_graph[3] = {nullptr, nullptr, nullptr};
    int64_t refine_graph_launches[3] = {0, 0, 0};
    int* refine_iter = nullptr;      // steps taken by the graph-driven refinement loop
    cudaGraphExec_t factor_graph = nullptr;
    int64_t factor_graph_launches = 0;
    int64_t factor_runs = 0;
    int64_t num_numeric = 0;         // numeric factorisations (KKTSystem.num_numeric, system.py:261)
    bool use_graphs = true;
    // device-side loop (cipm_loop_*): control parameters and the backtracking graphs
    double loop_norm_q = 0.0, loop_norm_b = 0.0, loop_eps_feas = 1e-8, loop_eps_inf = 1e-8;
    int loop_max_iter = 200;
    cudaGraphExec_t step_graph[2] = {nullptr, nullptr};     // step_length(which) incl. exp/pow WHILE
    cudaGraphExec_t nb_graph = nullptr;                      // neighbourhood WHILE

    std::vector<void*> allocations;
    std::vector<std::pair<int, int>> host_blocks;   // (kind 0 SOC dim / 3 PSD side) for bench byte counts
};

inline cudaEvent_t pooled_event(Ctx& c, size_t idx) {
    while (c.ev_pool.size() <= idx) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c.ev_pool.push_back(e);
    }
    return c.ev_pool[idx];
}

// ---- launchers (implemented in vec.cu / cones.cu / ldl.cu) ----
// vec.cu
void k_init_iterate(Ctx& c);
void k_residuals(Ctx& c);
void k_copy_best(Ctx& c);
void k_directions_prep_den(Ctx& c);          // den of the τ-step (col2 fixed per iteration)
void k_affine_rhs(Ctx& c);                   // rb[1] = [gx; -(gz - s)], rb[0] = [-q; b]
void k_combined_rhs(Ctx& c);                 // rb[0] = [f gx; -(f gz - dsc)]
void k_recover_direction(Ctx& c, int which, const double* sol, double dkappa_rhs_slot_is_combined);
void k_take_step(Ctx& c);
void k_recover_solution(Ctx& c, int which, int cert, double* out);   // ipm.py:383-407 into out[n + 2m]
void k_step_init(Ctx& c, int which);         // α bound from τ/κ
void k_step_finish(Ctx& c, int which);       // α check + σ
void k_kkt_residual(Ctx& c, int nrhs, const int* active_host);
void k_mu_candidates(Ctx& c, int k0, int nk, double mu_fixed = -1.0);
void k_refine_continue(Ctx& c, cudaGraphConditionalHandle h, int nrhs);
void k_loop_init(Ctx& c);
void k_iter_control(Ctx& c, int it);
void k_nsym_resolve_cond(Ctx& c, cudaGraphConditionalHandle h);
void k_mask_init(Ctx& c);
void k_nb_resolve_cond(Ctx& c, int nk, cudaGraphConditionalHandle h);
void k_refine_steps_store(Ctx& c, int nrhs, int slot);
// cones.cu
void k_update_scaling(Ctx& c);
void k_update_scaling_family(Ctx& c, int fam);
void k_scatter_h(Ctx& c);
void k_apply_h(Ctx& c, const double* v, double* out, double alpha, const double* u, double beta,
               const double* skip = nullptr);
void k_combined_ds(Ctx& c, const double* dz_a, const double* ds_a);
void k_step_bound(Ctx& c, const double* dz, const double* ds);
void k_nsym_feasible_mask(Ctx& c, const double* dz, const double* ds, int k0);
void k_neighborhood_mask(Ctx& c, int k0, int nk);
void k_membership(Ctx& c);
void k_soc_residuals(Ctx& c, const double* x, double* out);
void k_scaling_values(Ctx& c, double* diag, double* blocks);
// ldl.cu
void k_build_base(Ctx& c);
void k_assemble(Ctx& c);
int k_factor(Ctx& c);
void k_refine_step(Ctx& c, int nrhs, const int* active_host, bool gather = true);
bool fused_resid_ok(const Ctx& c);
// setup.cu
int k_set_problem(Ctx& c, bool equilibrate, bool replay);
// dense.cu
void tail_setup(Ctx& c, int64_t* inv_total, int64_t* flag_total);
void k_tail_factor(Ctx& c);
void k_tail_forward(Ctx& c, void* x, int act0, int act1);
void k_tail_backward(Ctx& c, void* x, int act0, int act1);
bool tail_is_single_root(const Ctx& c);
void k_root_solve(Ctx& c, void* x, int act0, int act1);   // tail = one dense root: fwd + D + bwd in one CTA

}  // namespace cipm
