/*
 * libcipm — C ABI of the B200-native (sm_100a) interior-point hot path.
 *
 * Drop-in boundary for the per-iteration work of the reference solver
 * (/root/reference/pkg/src/conic_ipm).  Every entry point below names the
 * reference interface it replaces; the Python host
 * (paper_2412_19027_b200/solver.py) calls them through ctypes in the same
 * order as the reference loop (ipm.py:427-482).
 *
 * Conventions
 *  - plain pointers and sizes only; host pointers unless documented;
 *  - every function returns an int status: CIPM_OK (0) or a negative
 *    CIPM_E_* code; nothing throws or aborts across the ABI;
 *  - numerical failures detected on the device are latched in a device error
 *    word and surface as the return code of the next synchronising call
 *    (cipm_residuals, cipm_step_combined, cipm_sync);
 *  - one context = one problem instance = one CUDA stream; not re-entrant.
 */
#ifndef CIPM_H
#define CIPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped to exception types by paper_2412_19027_b200/exceptions.py) */
#define CIPM_OK 0
#define CIPM_E_SCALING (-1)        /* ScalingFailure        (cones/scaling.py:79,154)   */
#define CIPM_E_STEP (-2)           /* StepTooSmall          (cones/steps.py:97,106; ipm.py:366) */
#define CIPM_E_FACTOR (-3)         /* FactorizationFailure  (kkt/system.py:259-260)     */
#define CIPM_E_DENOM (-4)          /* DegenerateDenominator (ipm.py:331-332)            */
#define CIPM_E_INTERIOR (-5)       /* LostInterior          (ipm.py:374-377)            */
#define CIPM_E_DOMAIN (-6)         /* DomainError           (cones/scaling.py:372,379)  */
#define CIPM_E_PATTERN (-7)        /* PatternMismatch                                   */
#define CIPM_E_DIM (-8)            /* DimensionMismatch                                 */
#define CIPM_E_CUDA (-20)          /* CUDA runtime failure                              */
#define CIPM_E_ARG (-21)           /* invalid argument                                  */

/* precision modes (kkt/system.py:28-29) */
#define CIPM_FULL 0
#define CIPM_MIXED 1

/* device scalar block layout (cipm_read_scalars) */
enum {
    CIPM_SC_TAU = 0, CIPM_SC_KAPPA, CIPM_SC_MU,
    CIPM_SC_GTAU,                 /* κ + q'x + b'z + x'Px/τ                          */
    CIPM_SC_XPX, CIPM_SC_QX, CIPM_SC_BZ,
    CIPM_SC_NRM_GX,               /* max |g_x / Dc|                                  */
    CIPM_SC_NRM_ATZ,              /* max |A'z / Dc|                                  */
    CIPM_SC_NRM_PX,               /* max |P x / Dc|                                  */
    CIPM_SC_NRM_XU,               /* max |Dc x|                                      */
    CIPM_SC_NRM_GZ,               /* max |g_z / Dr|                                  */
    CIPM_SC_NRM_AXS,              /* max |(A x + s) / Dr|                            */
    CIPM_SC_NRM_ZU,               /* max |Dr z|                                      */
    CIPM_SC_NRM_SU,               /* max |s / Dr|                                    */
    CIPM_SC_DEN,                  /* τ-step denominator (ipm.py:328-330)             */
    CIPM_SC_DTAU_A, CIPM_SC_DKAPPA_A, CIPM_SC_DTAU_C, CIPM_SC_DKAPPA_C,
    CIPM_SC_ALPHA_A, CIPM_SC_SIGMA, CIPM_SC_ALPHA_C, CIPM_SC_ALPHA_FINAL,
    CIPM_SC_T0, CIPM_SC_T1, CIPM_SC_T2, CIPM_SC_T3, CIPM_SC_T4, CIPM_SC_T5, CIPM_SC_T6, CIPM_SC_T7,
    CIPM_SC_ALPHA_WORK,           /* running step bound (atomic min)                 */
    CIPM_SC_SZ,                   /* s'z                                             */
    CIPM_SC_BUMPS,                /* dynamically regularised pivots (last factor)    */
    CIPM_SC_REFINE_STEPS,         /* refinement steps of the last solve              */
    /* device-side loop control (cipm_loop_*: the Algorithm-1 decisions of ipm.py:427-457) */
    CIPM_SC_NB_BATCH,             /* neighbourhood candidates evaluated so far        */
    CIPM_SC_BEST_FLAG,            /* this iteration improved the best iterate (copied) */
    CIPM_SC_REF_STEPS_A, CIPM_SC_REF_STEPS_C,   /* refinement steps, affine / combined */
    CIPM_SC_STATUS = 40,          /* 0 running, 1 optimal, 2 primal infeasible, 3 dual
                                     infeasible, 4 max iterations, 5 insufficient progress */
    CIPM_SC_BEST_SCORE, CIPM_SC_BEST_VALID,
    CIPM_SC_STALL_MU, CIPM_SC_STALL_RP, CIPM_SC_STALL_RD, CIPM_SC_STALL_CNT,
    CIPM_SC_BEST_TAU, CIPM_SC_BEST_KAPPA, CIPM_SC_BEST_MU,
    CIPM_SC_BEST_GP, CIPM_SC_BEST_GD, CIPM_SC_BEST_RP, CIPM_SC_BEST_RD,
    CIPM_SC_BEST_R1, CIPM_SC_BEST_R2, CIPM_SC_BEST_R3,
    CIPM_SC_CUR_R1, CIPM_SC_CUR_R2, CIPM_SC_CUR_R3,
    CIPM_SC_COUNT = 64
};

typedef struct cipm_symbolic cipm_symbolic;
typedef struct cipm_ctx cipm_ctx;
typedef struct cipm_batch cipm_batch;

/* Problem structure after cone reordering (problem.py:177-210): rows are
 * [zero | nonneg | SOC... | exp... | pow... | PSD...]; offsets are row indices
 * into the m conic rows. */
typedef struct {
    int64_t n, m;
    const int64_t *p_rowptr, *p_colidx;   /* P, full symmetric CSR (n x n)  */
    const int64_t *a_rowptr, *a_colidx;   /* A, CSR (m x n)                 */
    int64_t zero_dim, nonneg_dim;
    int64_t n_soc;  const int64_t *soc_off, *soc_dim;
    int64_t n_exp;  const int64_t *exp_off;
    int64_t n_pow;  const int64_t *pow_off; const double *pow_alpha;
    int64_t n_psd;  const int64_t *psd_off, *psd_side;
} cipm_problem_desc;

typedef struct {
    int precision;                 /* CIPM_FULL | CIPM_MIXED                         */
    double delta_s, delta_d;       /* static / dynamic regularisation (system.py:35-42) */
    double beta, backtrack, step_scale;     /* ipm.py:63-65                          */
    double refine_abs, refine_rel; int refine_max;   /* RefinementSettings            */
    int device;
    void *stream;                  /* cudaStream_t (NULL = create a private stream)  */
} cipm_settings;

typedef struct {
    int64_t dim, nsuper, nnz_l, nnz_storage, n_updates, max_width, max_rows, height;
    double flops;
    int64_t ordering;              /* ordering used: 0 minimum degree (reference), 1 natural, 2 nested dissection */
} cipm_symbolic_info;

int cipm_version(void);

/* --- symbolic analysis (replaces kkt/system.py:87-148 + :188-240, ordering.py:15-53) --- */
/* ordering: 0 = the reference's exact minimum degree (ordering.py:15-53), 1 = natural,
 * 2 = nested dissection, 3 = auto (MD below 20k rows, else ND when its fill and flops
 * stay within 1.25x / 1.5x of MD's) */
int cipm_symbolic_create(const cipm_problem_desc *desc, int ordering, cipm_symbolic **out);
/* same, with the nested-dissection leaf size (parts up to nd_leaf rows are ordered by MD; 0 = default 256) */
int cipm_symbolic_create_ex(const cipm_problem_desc *desc, int ordering, int64_t nd_leaf, cipm_symbolic **out);
int cipm_symbolic_info_get(const cipm_symbolic *sym, cipm_symbolic_info *info);
/* copy a named symbolic array ("perm", "sn_col", "sn_rptr", "sn_rows", "sn_loff", "sn_parent",
 * "upd_ptr", "upd_src", "upd_p0", "upd_p1", "order", "map_p", "map_a", "map_diag", "map_hblk") */
int cipm_symbolic_array(const cipm_symbolic *sym, const char *name, void *dst, int64_t *count);
void cipm_symbolic_destroy(cipm_symbolic *sym);
/* the reference's exact minimum-degree order of a symmetric pattern (ordering.py:15-53) */
int cipm_min_degree(int64_t dim, const int64_t *rowptr, const int64_t *colidx, int32_t *perm);

/* --- context (replaces Solver.__init__ device state, ipm.py:150-171, and KKTSystem) --- */
int cipm_ctx_create(const cipm_problem_desc *desc, const cipm_symbolic *sym,
                    const cipm_settings *settings, cipm_ctx **out);
/* scaled problem values + equilibration (problem.py:222-284 output); H2D copy */
int cipm_ctx_set_values(cipm_ctx *ctx, const double *p_values, const double *a_values,
                        const double *q, const double *b, const double *d_row,
                        const double *d_col, double c_obj);
/* device-side problem setup (replaces the host reorder_cones + equilibrate, problem.py:177-284,
 * for the parametric re-solve path ipm.py:187-221): row_perm[i] = user row of reordered row i,
 * a_src[k] = user A-value index of reordered A nonzero k (set once) */
int cipm_ctx_set_reorder(cipm_ctx *ctx, const int64_t *row_perm, const int64_t *a_src);
/* raw USER-order values (P full symmetric values, A values, q, b) -> H2D, reorder, 10 Ruiz
 * rounds (bitwise the reference's arithmetic) when equilibrate != 0, factor base image.
 * After the first call a NULL array keeps the device's previous raw values (update_data
 * with only q / b changed sends only q / b). */
int cipm_ctx_set_problem(cipm_ctx *ctx, const double *p_values, const double *a_values,
                         const double *q, const double *b, int equilibrate);
/* the equilibration of the last set_problem: d_row (m), d_col (n), c_obj */
int cipm_ctx_get_equilibration(cipm_ctx *ctx, double *d_row, double *d_col, double *c_obj);
void cipm_ctx_destroy(cipm_ctx *ctx);
int cipm_sync(cipm_ctx *ctx);
int cipm_device_bytes(const cipm_ctx *ctx, int64_t *bytes);

/* --- Algorithm-1 steps (ipm.py:411-482) --- */
int cipm_init_iterate(cipm_ctx *ctx);                     /* unit_init, set.py:91-112       */
int cipm_residuals(cipm_ctx *ctx, double *scalars_out);   /* ipm.py:233-280 + G rows :284   */
int cipm_save_best(cipm_ctx *ctx);                        /* best = state.copy()  ipm.py:430 */
int cipm_update_scaling(cipm_ctx *ctx);                   /* scaling.py:229-251             */
int cipm_factor(cipm_ctx *ctx);                           /* set_scaling + numeric_factor   */
int cipm_solve_affine(cipm_ctx *ctx, int *refine_steps);  /* col2 + affine directions       */
int cipm_step_affine(cipm_ctx *ctx);                      /* step_length + centering        */
int cipm_solve_combined(cipm_ctx *ctx, int *refine_steps);/* combined_rhs + directions      */
int cipm_step_combined(cipm_ctx *ctx, double *alpha);     /* combined_step_size ipm.py:350  */
int cipm_take_step(cipm_ctx *ctx);                        /* take_step ipm.py:368           */
int cipm_read_scalars(cipm_ctx *ctx, double *out);
/* which: 0 = current iterate, 1 = best iterate.  x (n), z (m), s (m), tkm[3] = τ, κ, μ */
int cipm_get_iterate(cipm_ctx *ctx, int which, double *x, double *z, double *s, double *tkm);
int cipm_set_iterate(cipm_ctx *ctx, const double *x, const double *z, const double *s, const double *tkm);
/* solution recovery on the device (ipm.py:383-407, replaces the host unscale + row scatter):
 * x = Dc x' (/ τ), z = Dr z' / c (/ τ), s = s' / Dr (/ τ) in the user's row order; no
 * division by τ when certificate != 0.  which: 0 = current, 1 = best iterate; tkm[3] = τ, κ, μ
 * of that iterate (may be NULL). */
int cipm_get_solution(cipm_ctx *ctx, int which, int certificate, double *x, double *z, double *s, double *tkm);

/* --- operator-level seams (tests / observers) --- */
/* refined KKT solve of K x = rhs with the current factor (system.py:279-314) */
int cipm_kkt_solve(cipm_ctx *ctx, const double *rhs, double *x, int *steps, double *residual);
/* KKTSystem seam (kkt/system.py:64-314; a device-backed drop-in for the class):
 * set_scaling(diag, blocks) — H from the host: diag over the zero + nonneg rows, blocks
 * packed upper triangles in the order of cipm_scaling_values; the factorisation and the
 * refinement residual then use these values (replaces system.py:166-184).
 * matvec — the unregularised K x (system.py:273-277).
 * solve_ex — cipm_kkt_solve plus RefineResult.stalled (system.py:279-314).
 * set_refinement — RefinementSettings t_abs, t_rel, t_max (system.py:45-54). */
int cipm_kkt_set_scaling(cipm_ctx *ctx, const double *diag, const double *blocks);
int cipm_kkt_matvec(cipm_ctx *ctx, const double *x, double *out);
int cipm_kkt_solve_ex(cipm_ctx *ctx, const double *rhs, double *x, int *steps, double *residual, int *stalled);
int cipm_set_refinement(cipm_ctx *ctx, double t_abs, double t_rel, int t_max);
/* H v with the current scaling (scaling.py:254-274) */
int cipm_apply_h(cipm_ctx *ctx, const double *v, double *out);
/* dense -H block values as scattered into the factor (for tests): returns the
 * diagonal over zero+nonneg rows and the concatenated upper triangles of blocks */
int cipm_scaling_values(cipm_ctx *ctx, double *diag, double *blocks);
/* directions of the last affine / combined solve: dx (n), dz (m), ds (m), dtk[2] */
int cipm_get_direction(cipm_ctx *ctx, int combined, double *dx, double *dz, double *ds, double *dtk);
/* copy a named device vector ("x","z","s","gx","gz","dsc","col2","sol1","nn_h","hv") to the host */
int cipm_get_vector(cipm_ctx *ctx, const char *name, double *out, int64_t *count);
/* per-cone batched SOC residuals t^2 - |u|^2 with the reference's fixed order (steps.py:136-175) */
int cipm_soc_residuals(cipm_ctx *ctx, const double *x, double *out);
/* ---- device-side loop (one blocking read per IPM iteration) ----
 * cipm_loop_begin: unit start (set.py:91-112) and the control state; the norms are
 *   ||q||inf, ||b||inf of the unscaled reordered data (ipm.py:184-185).
 * cipm_loop_check: residuals (ipm.py:233-251) and, on the device, the best-iterate
 *   bookkeeping, Eq.(8) termination, Eq.(9) infeasibility, max_iter and the stall
 *   window (ipm.py:427-457); then ONE synchronisation: the scalar block (status in
 *   CIPM_SC_STATUS) is copied to sc_out.  Returns a CIPM_E_* code if the previous
 *   iteration body latched a numerical failure.
 * cipm_loop_body: one iteration body (scaling, factorisation, affine and combined
 *   refined solves, step lengths with their backtracking loops as device WHILE
 *   graphs, neighbourhood search, take_step) enqueued without any host round trip. */
int cipm_loop_begin(cipm_ctx *ctx, double norm_q, double norm_b, double eps_feas, double eps_inf, int max_iter);
int cipm_loop_check(cipm_ctx *ctx, int iteration, double *sc_out);
int cipm_loop_body(cipm_ctx *ctx);

/* ---- kernel-level seams: the reference's L1 cone functions one call at a time
 * (tests/test_gpu_seams.py checks them against tests/golden/kernels.json) ---- */
/* set direction `which` (0 affine, 1 combined): dx (n), dz (m), ds (m), dtk = {dtau, dkappa};
 * NULL arrays are left unchanged */
int cipm_set_direction(cipm_ctx *ctx, int which, const double *dx, const double *dz, const double *ds,
                       const double *dtk);
/* step_length (cones/steps.py:79-116) of direction `which` at the current iterate
 * (tau, kappa from cipm_set_iterate); CIPM_E_STEP below 1e-11 */
int cipm_step_length(cipm_ctx *ctx, int which, double *alpha);
/* combined_ds (cones/scaling.py:277-320) at the current scaling (cipm_update_scaling):
 * out (m) from the affine dz_a, ds_a, sigma, mu */
int cipm_combined_ds(cipm_ctx *ctx, const double *dz_a, const double *ds_a, double sigma, double mu,
                     double *out);
/* neighborhood_ok (cones/scaling.py:364-401) of the current s, z at the given mu, beta; ok = 0 / 1 */
int cipm_neighborhood_ok(cipm_ctx *ctx, double mu, double beta, int *ok);
/* is_in_cone(s) / is_in_dual_cone(z), strict (cones/set.py:166-207); overwrites the iterate */
int cipm_membership(cipm_ctx *ctx, const double *s, const double *z, int *in_cone, int *in_dual);
/* KKTSystem counters (kkt/system.py:78-79,261-262): out[0] = numeric factorisations
 * since the context was created (num_numeric), out[1] = pivots bumped by the dynamic
 * regularisation in the last factorisation (last_bumped_pivots) */
int cipm_kkt_counters(cipm_ctx *ctx, int64_t *out);
/* bench roofline: per-launch time (ms) and algorithmic bytes of the kernel classes
 * at the current iterate, out[12] = {residual SpMV, KKT matvec, scaling nonneg, SOC,
 * exp+pow, PSD} x {ms, bytes}; reps timed launches each (CUDA events, context stream) */
int cipm_kernel_classes(cipm_ctx *ctx, int reps, double *out);
/* host<->device bytes moved by the API since the last reset (bench e2e accounting) */
int cipm_io_bytes(cipm_ctx *ctx, int64_t *h2d, int64_t *d2h, int reset);
/* kernel launches issued since the last reset (bench accounting) */
int cipm_launch_count(cipm_ctx *ctx, int64_t *count, int reset);
/* per-launch CUDA-event timing of the factorisation and triangular-solve kernels:
 * cipm_profile(enable) clears and (de)activates; cipm_kernel_stats returns
 * out[5] = {factor ms total, factor launches, solve ms total, solve launch pairs, rhs solved} */
int cipm_profile(cipm_ctx *ctx, int enable);
int cipm_kernel_stats(cipm_ctx *ctx, double *out);
/* CUDA events on the context stream: op 0 records the start, op 1 the stop and
 * returns the elapsed milliseconds */
int cipm_timer(cipm_ctx *ctx, int op, double *ms);
/* per-task timeline of the persistent kernels (profiling seam): enable=1 arms it;
 * enable=0 copies out[12*nsuper] = per supernode: forward {start, start, gathered, triangle,
 * pushed, done} ns of the last forward sweep, then factor {start, start, staged, gathered,
 * factored, done} of the last factorisation */
int cipm_trace(cipm_ctx *ctx, int enable, int64_t *out);
/* CUDA-event time (ms) of the last numeric factorisation and last triangular solve */
int cipm_kernel_times(cipm_ctx *ctx, double *factor_ms, double *solve_ms);

/* --- batched independent instances sharing one pattern (C5b; replaces the
 * reference's per-instance Solver loop under bench --jobs, bench.py:98-113).
 * Zero + nonnegative cones, full precision.  One CTA runs one instance's whole
 * IPM (ipm.py:411-496) on the device.  Values are the per-instance SCALED data
 * (after reorder_cones + equilibrate, problem.py:177-284), instance-major:
 * V = [P values | A values] (count x (nnzP + nnzA)), q (count x n), b, Dr
 * (count x m), Dc (count x n), c_obj / norm_q / norm_b (count; the norms are
 * ‖q‖∞, ‖b‖∞ of the reordered unscaled data, ipm.py:184-185). --- */
int cipm_batch_create(const cipm_problem_desc *desc, int count, const cipm_settings *settings,
                      double eps_feas, double eps_inf, int max_iter, cipm_batch **out);
/* info[9] = {count, n, m, nnz(L), shared bytes per instance CTA, in shared memory (1) or workspace (0),
 *           CTA-parallel factorisation (1) or sequential (0), dense root width, leaf groups} */
int cipm_batch_info(const cipm_batch *b, int64_t *info);
int cipm_batch_set_values(cipm_batch *b, const double *V, const double *q, const double *bvec,
                          const double *d_row, const double *d_col, const double *c_obj,
                          const double *norm_q, const double *norm_b);
/* device-side setup per instance (replaces the host reorder + equilibration): the
 * reorder maps once (row_perm[i] = user row of reordered row i, a_src[k] = user A-value
 * index of reordered nonzero k), then raw USER-order values per solve: V = [P | A] (user
 * order), q, b.  Results then come back unscaled, divided by tau (not for infeasibility
 * certificates) and in the user's row order. */
int cipm_batch_set_reorder(cipm_batch *b, const int64_t *row_perm, const int64_t *a_src);
/* NULL V / q / bvec (after the first call) keep the device's previous raw arrays */
int cipm_batch_set_raw_values(cipm_batch *b, const double *V, const double *q, const double *bvec,
                              int equilibrate);
/* run every instance to termination; *ms = CUDA-event time of the launch */
int cipm_batch_solve(cipm_batch *b, double *ms);
/* status[count] (0 optimal, 1 primal_inf, 2 dual_inf, 3 almost_optimal, 4 max_iterations,
 * 6 insufficient_progress, 7 numerical_error); res[count][9] = {g_p, g_d, ‖r_p‖, ‖r_d‖, τ, κ, μ,
 * μ_initial, iterations}; x/z/s: the reported (current or best) SCALED iterate */
int cipm_batch_results(cipm_batch *b, int32_t *status, double *res, double *x, double *z, double *s);
int cipm_batch_io_bytes(cipm_batch *b, int64_t *h2d, int64_t *d2h, int reset);
void cipm_batch_destroy(cipm_batch *b);

#ifdef __cplusplus
}
#endif
#endif /* CIPM_H */
