// Host-side symbolic analysis of the quasi-definite KKT matrix
//     K = [ P   A' ]
//         [ A  -H  ]
// run once per sparsity pattern (reference: kkt/system.py:87-148 pattern,
// :188-240 symbolic_factor, kkt/ordering.py:15-53 ordering, kkt/ldl.py:20-34).
//
// Output is a *supernodal* description consumed by the sm_100a numeric
// factorisation and triangular solves: supernodes are contiguous column ranges
// of the (postordered) permuted matrix with a shared sorted row list; each panel
// is stored dense column-major (rows x width) in one flat value array.
#pragma once
#include <cstdint>
#include <vector>

namespace cipm {

struct SymbolicOptions {
    int ordering = 0;          // 0 = exact minimum degree (reference order), 1 = natural,
                               // 2 = nested dissection (level-structure separators, MD leaves)
    int64_t nd_leaf = 256;     // nested dissection: parts up to this size are ordered by MD
    int64_t auto_min_dim = 20000;   // ordering 3 (auto): below this, the reference's MD
    double nd_max_fill = 1.25;      // ... above it ND if nnz(L) <= this x MD's
    double nd_max_flops = 1.5;      // ... and factor flops <= this x MD's
    int64_t md_work_budget_per_nnz = 50;   // exact MD abandoned for AMD past this work / (nnz + dim)
    int relax_small = 8;       // always merge a child into its parent up to this width
    int relax_mid = 32;        // ... up to this width if zero fraction <= relax_mid_frac
    double relax_mid_frac = 0.3;
    int relax_big = 64;        // ... up to this width if zero fraction <= relax_big_frac
    double relax_big_frac = 0.05;
    int tail_width = 64;       // supernodes at least this wide go to the dense tail path
    int tail_offrows = 512;    // ... or with at least this many off-diagonal rows
    int mid_panel = 512;       // panels (w*r) at least this large, or inboxes of 2x this, and
                               // their ancestors are factored by whole CTAs (mid tier)
    int chain_merge_max = 256;    // merge the single-child chain below a root into one dense
                                  // supernode of at most this many columns (0: off)
};

struct Symbolic {
    int64_t n = 0, m = 0, dim = 0;
    // permutation: position k of the factor holds original KKT index perm[k]
    std::vector<int32_t> perm, iperm;
    std::vector<int32_t> md_perm;          // raw fill-reducing order (before postordering)
    int ordering_used = 0;                 // 0 MD (or AMD past the work budget), 1 natural, 2 ND, 4 AMD
    std::vector<int8_t> sign;              // +1 x rows, -1 z rows (permuted order)
    // supernodes
    int32_t nsuper = 0;
    std::vector<int32_t> sn_col;           // nsuper+1: first column, width = sn_col[J+1]-sn_col[J]
    std::vector<int64_t> sn_rptr;          // nsuper+1: into sn_rows
    std::vector<int32_t> sn_rows;          // sorted permuted row indices (first w = own columns)
    std::vector<int64_t> sn_loff;          // nsuper+1: panel offsets in the value array
    std::vector<int32_t> sn_parent;        // -1 for roots
    std::vector<int32_t> sn_nchild;
    std::vector<int32_t> col2sn;           // dim
    // update lists (left-looking): updates into J come from (src, p0, p1)
    std::vector<int64_t> upd_ptr;          // nsuper+1
    std::vector<int32_t> upd_src, upd_p0, upd_p1;
    // push/pull "inbox" maps (see ldl.cu):
    //  factor — supernode K's packed lower contribution block C_K = L_off D L_off'
    //  (column-major over b' then a' >= b', offset cb_off[K]) is scattered to
    //  inbox positions push_pos[cb_off[K] + t]; supernode J gathers its inbox rows
    //  irow_ptr[sn_rptr[J] + tr] .. (+1) sorted by (target column, source K), each
    //  entry subtracting from panel offset inbox_tgt[e] (= tc * r_J + tr).
    std::vector<int64_t> cb_off;           // nsuper+1 (packed lower (r-w)(r-w+1)/2 per supernode)
    std::vector<int64_t> push_pos;         // cb_off[nsuper]
    std::vector<int64_t> irow_ptr;         // sn_rows.size()+1
    std::vector<int32_t> inbox_tgt;        // cb_off[nsuper]
    //  solves — supernode K's off-row contributions v (offset cv_off[K] = sum (r-w))
    //  go to vpush_pos[cv_off[K] + a]; column j of the factor gathers vcol_ptr[j]..
    std::vector<int64_t> cv_off;           // nsuper+1
    std::vector<int64_t> vpush_pos;        // cv_off[nsuper]
    std::vector<int64_t> vcol_ptr;         // dim+1
    // schedule
    std::vector<int32_t> order;            // topological order: non-tail by level, then tail by level
    std::vector<int32_t> level;            // per supernode, 0 = leaf
    int32_t height = 0;
    std::vector<int8_t> is_tail;           // dense tail supernode (multi-CTA path, dense.cu)
    std::vector<int8_t> is_mid;            // mid tier: one CTA per supernode in the factorisation
    int32_t n_main = 0;                    // order[0 .. n_main) are the non-tail supernodes
    int32_t n_warp = 0;                    // order[0 .. n_warp) are the warp-tier supernodes
    int64_t max_panel_main = 0;            // largest non-tail panel (shared-memory sizing)
    int64_t max_panel_warp = 0;            // largest warp-tier panel
    // continuation scheduling: a task finishing supernode K increments its parent's
    // same-tier counter; the task that completes it continues with the parent
    std::vector<int8_t> tier;              // 0 warp, 1 CTA, 2 dense tail
    std::vector<int32_t> desc32;           // 8 per supernode: c0, w, r, parent, need_solve, need_fac, tier, -
    std::vector<int64_t> desc64;           // 8 per supernode: loff, cv_off, vlo, vhi, ilo, ihi, cb_off, rptr
    std::vector<int32_t> need;             // 2 per supernode: need_solve, need_fac
    std::vector<int32_t> start_solve;      // non-tail supernodes with no children (forward sweep seeds)
    std::vector<int32_t> start_fac_warp;   // warp-tier supernodes with no warp-tier children
    std::vector<int32_t> start_fac_cta;    // CTA-tier supernodes with no CTA-tier children
    std::vector<uint8_t> vin_col;          // vector-inbox entry -> local column in its supernode
    // Within each target supernode's inbox region, the entries pushed by tiny
    // leaves come first (grouped by column), then the rest (grouped by column):
    // column j's tiny entries are [vt_lo[j], vt_hi[j]), its other entries
    // [vn_lo[j], vn_hi[j]).  The forward sweep folds the tiny entries into the
    // right-hand side in one parallel pass (tfold_cols: columns with any), so the
    // persistent kernel gathers only [desc64 vlo, vhi) = the non-tiny part.
    std::vector<int64_t> vt_lo, vt_hi, vn_lo, vn_hi;   // dim
    std::vector<int32_t> tfold_cols;
    std::vector<int32_t> tiny;             // leaves with w <= 4, r <= 16: one lane each (factor, solves)
    std::vector<int32_t> bwd_order;        // backward tickets (reversed): non-tail, non-tiny, topological
    // scatter maps into the panel value array (int64 positions)
    std::vector<int64_t> map_p;            // P CSR nnz; -1 for strictly-lower entries
    std::vector<int64_t> map_a;            // A CSR nnz (entry (n+r, j) of K stored at L(col j? ...))
    std::vector<int64_t> map_diag;         // dim, original index order: diagonal slot of K_ii
    std::vector<int64_t> map_hblk;         // sum_b d_b(d_b+1)/2: upper entries (rl<=cl) per block
    // statistics
    int64_t nnz_l = 0;                     // true strict-lower nnz of L
    int64_t nnz_storage = 0;               // dense panel elements
    double flops = 0.0;                    // 2 * sum_j c_j^2 with c_j strict-lower count
    int64_t max_width = 0, max_rows = 0, max_panel = 0;
    int64_t n_updates = 0;
};

// Pattern inputs: P full CSR (n x n), A CSR (m x n); lin = zero_dim + nonneg_dim;
// blocks (offset, dim) in K's z-row coordinates for every SOC/exp/pow/PSD cone.
int analyze(int64_t n, int64_t m,
            const int64_t* p_rowptr, const int64_t* p_colidx,
            const int64_t* a_rowptr, const int64_t* a_colidx,
            int64_t lin, int64_t nblocks, const int64_t* blk_off, const int64_t* blk_dim,
            const SymbolicOptions& opt, Symbolic& out);

}  // namespace cipm
