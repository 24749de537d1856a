// Batched independent instances sharing one sparsity pattern (batch.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace cipm {

constexpr double STALL_IMP = 0.99;   // ipm.py:36 STALL_IMPROVEMENT

// Pattern tables shared by every instance (device pointers, int32).
struct BatchPattern {
    int n = 0, m = 0, zero_dim = 0, nonneg_dim = 0;
    int nnz_p = 0, nnz_a = 0, nnz_l = 0;
    const int32_t *p_rp = nullptr, *p_ci = nullptr;          // P full symmetric CSR
    const int32_t *a_rp = nullptr, *a_ci = nullptr;          // A CSR
    const int32_t *at_rp = nullptr, *at_ci = nullptr, *at_src = nullptr;   // A' CSR (+ source in A)
    // permuted upper CSC of K (reference order) and the value source of every entry:
    // src >= 0: V[src] (P values then A values); src == -1: structural zero; src <= -2: -h[-src-2]
    const int32_t *cp = nullptr, *ci = nullptr, *csrc = nullptr;
    const int8_t* sign = nullptr;                            // +1 x rows / -1 z rows (permuted)
    const int32_t* perm = nullptr;                           // permuted position -> KKT index
    const int32_t *lp = nullptr, *li = nullptr;              // L column pointers / rows
    const int32_t *up_ptr = nullptr, *up_i = nullptr, *up_p2 = nullptr;   // up-looking schedule
    const int32_t *a_src = nullptr, *b_src = nullptr;        // user -> reordered A values / rows
    // ---- CTA-parallel factorisation (use_groups): the elimination order splits into
    // independent leaf groups (subtrees below the top chain) and one dense root block of
    // the last W columns (rows / columns >= s).  Groups: thread per group, dense panel;
    // root: blocked right-looking LDL' by the CTA, diagonal blocks kept as inverses.
    int use_groups = 0;
    int s = 0, W = 0, ngroups = 0;
    int panel_total = 0, root_off = 0, inbox_total = 0;
    const int32_t* g_info = nullptr;    // per group 8 ints: cols_off, w, r, panel_off, inbox_off, vin_off, rows_off, 0
    const int32_t* g_cols = nullptr;    // group columns (permuted indices, ascending)
    const int32_t* g_rows = nullptr;    // root-local indices of each group's off rows (ascending)
    int nbsc = 0;
    const int32_t *bsc_slot = nullptr, *bsc_src = nullptr;   // K value -> panel slot (src coded as csrc)
    int nbdg = 0;
    const int32_t *bdg_slot = nullptr, *bdg_col = nullptr;   // diagonal slots (static regularisation)
    int nrg = 0;
    const int32_t *rg_tgt = nullptr, *rg_ptr = nullptr, *rg_idx = nullptr;   // root entry <- inbox slots
    const int32_t *rv_ptr = nullptr, *rv_idx = nullptr;      // root row <- vector-inbox slots (W + 1)
};

// Per-instance data (device pointers, instance-major) and settings.
struct BatchData {
    const double *V = nullptr, *q = nullptr, *b = nullptr;
    double *dr = nullptr, *dc = nullptr;      // device_setup: written by the kernel
    const double *c_obj = nullptr, *norm_q = nullptr, *norm_b = nullptr;
    double* out_cobj = nullptr;
    int device_setup = 0, equilibrate = 1;
    double *best_x = nullptr, *best_z = nullptr, *best_s = nullptr;
    double *out_x = nullptr, *out_z = nullptr, *out_s = nullptr, *out_res = nullptr;
    int32_t* out_status = nullptr;
    double* workspace = nullptr;     // used when use_smem == 0
    int64_t ws_stride = 0;
    int use_smem = 1;
    double eps_feas = 1e-8, eps_inf = 1e-8;
    int max_iter = 200;
    double delta_s = 1e-8, delta_d = 0.0, beta = 1e-6, backtrack = 0.8, step_scale = 0.99;
    double refine_abs = 1e-12, refine_rel = 1e-12;
    int refine_max = 10;
};

size_t batch_smem_doubles(const BatchPattern& pt);
int batch_launch(const BatchPattern& pt, const BatchData& bd, int count, cudaStream_t stream, int smem_bytes);

}  // namespace cipm
