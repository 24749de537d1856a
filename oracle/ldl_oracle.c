/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's
 * sequential sparse kernels, used as the parity checker and the CPU baseline.
 * Never linked into the product path (paper_2412_19027_b200/).
 *
 * Restated from (file:line in /root/reference/pkg/src/conic_ipm):
 *   oracle_min_degree     kkt/ordering.py:15-53   exact-degree greedy MD,
 *                                                 explicit elimination graph,
 *                                                 (degree, index) heap order
 *   oracle_ldl_symbolic   kkt/ldl.py:20-34        etree + column counts
 *   oracle_ldl_numeric_*  kkt/ldl.py:37-88        up-looking LDL' with the signed
 *                                                 dynamic-regularisation bump
 *   oracle_ldl_solve_*    kkt/ldl.py:91-104       L, D, L' sweeps in place
 *   oracle_symm_matvec    kkt/ldl.py:107-121      K x from the upper triangle
 *
 * The float32 numeric variant reproduces the reference's numba typing bit for
 * bit: the pivot accumulator runs in float32, the regularisation bound and the
 * running max |D| in float64 (verified against numba ldl_numeric on a mixed
 * KKT; see tests/test_oracle.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef int64_t i64;

/* ---------------- min-degree ordering ---------------- */

typedef struct { i64 *v; i64 n, cap; } vec_t;

static void vpush(vec_t *a, i64 x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 4;
        a->v = (i64 *)realloc(a->v, (size_t)a->cap * sizeof(i64));
    }
    a->v[a->n++] = x;
}

static void vremove(vec_t *a, i64 x) {
    for (i64 k = 0; k < a->n; ++k)
        if (a->v[k] == x) { a->v[k] = a->v[--a->n]; return; }
}

/* binary min-heap of (deg, node) pairs, lexicographic order = Python heapq on tuples */
typedef struct { i64 *d, *u; i64 n, cap; } heap_t;

static int hless(const heap_t *h, i64 a, i64 b) {
    return h->d[a] < h->d[b] || (h->d[a] == h->d[b] && h->u[a] < h->u[b]);
}
static void hswap(heap_t *h, i64 a, i64 b) {
    i64 t = h->d[a]; h->d[a] = h->d[b]; h->d[b] = t;
    t = h->u[a]; h->u[a] = h->u[b]; h->u[b] = t;
}
static void hpush(heap_t *h, i64 deg, i64 node) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->d = (i64 *)realloc(h->d, (size_t)h->cap * sizeof(i64));
        h->u = (i64 *)realloc(h->u, (size_t)h->cap * sizeof(i64));
    }
    i64 k = h->n++;
    h->d[k] = deg; h->u[k] = node;
    while (k > 0) {
        i64 p = (k - 1) / 2;
        if (!hless(h, k, p)) break;
        hswap(h, k, p); k = p;
    }
}
static void hpop(heap_t *h, i64 *deg, i64 *node) {
    *deg = h->d[0]; *node = h->u[0];
    h->n--;
    if (h->n == 0) return;
    h->d[0] = h->d[h->n]; h->u[0] = h->u[h->n];
    i64 k = 0;
    for (;;) {
        i64 l = 2 * k + 1, r = l + 1, s = k;
        if (l < h->n && hless(h, l, s)) s = l;
        if (r < h->n && hless(h, r, s)) s = r;
        if (s == k) break;
        hswap(h, k, s); k = s;
    }
}

/* perm[k] = k-th eliminated node.  Pattern may be any triangle; diagonal ignored. */
int oracle_min_degree(i64 n, const i64 *rowptr, const i64 *colidx, i64 *perm) {
    vec_t *adj = (vec_t *)calloc((size_t)n, sizeof(vec_t));
    i64 *mark = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    char *alive = (char *)malloc((size_t)(n > 0 ? n : 1));
    i64 *nbrs = (i64 *)malloc((size_t)(n > 0 ? n : 1) * sizeof(i64));
    if (!adj || !mark || !alive || !nbrs) return -1;
    for (i64 i = 0; i < n; ++i) { mark[i] = -1; alive[i] = 1; }
    /* symmetric adjacency without duplicates: stamp-based dedupe per row */
    for (i64 i = 0; i < n; ++i)
        for (i64 p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            i64 j = colidx[p];
            if (i != j) { vpush(&adj[i], j); vpush(&adj[j], i); }
        }
    for (i64 i = 0; i < n; ++i) {           /* dedupe */
        i64 w = 0;
        for (i64 k = 0; k < adj[i].n; ++k) {
            i64 j = adj[i].v[k];
            if (mark[j] != i) { mark[j] = i; adj[i].v[w++] = j; }
        }
        adj[i].n = w;
    }
    for (i64 i = 0; i < n; ++i) mark[i] = -1;
    heap_t h = {0};
    for (i64 i = 0; i < n; ++i) hpush(&h, adj[i].n, i);
    i64 k = 0, stamp = 0;
    while (k < n) {
        i64 deg, v;
        hpop(&h, &deg, &v);
        if (!alive[v] || deg != adj[v].n) continue;
        perm[k++] = v;
        alive[v] = 0;
        i64 nn = 0;
        for (i64 t = 0; t < adj[v].n; ++t)
            if (alive[adj[v].v[t]]) nbrs[nn++] = adj[v].v[t];
        for (i64 t = 0; t < nn; ++t) vremove(&adj[nbrs[t]], v);
        for (i64 a = 0; a < nn; ++a) {
            i64 u = nbrs[a];
            ++stamp;
            /* stamps must be unique per (u) pass: use a fresh stamp each time */
            for (i64 t = 0; t < adj[u].n; ++t) mark[adj[u].v[t]] = stamp;
            for (i64 b = a + 1; b < nn; ++b) {
                i64 w = nbrs[b];
                if (mark[w] != stamp) {
                    vpush(&adj[u], w);
                    vpush(&adj[w], u);
                    mark[w] = stamp;
                }
            }
        }
        for (i64 t = 0; t < nn; ++t) hpush(&h, adj[nbrs[t]].n, nbrs[t]);
        free(adj[v].v); adj[v].v = NULL; adj[v].n = adj[v].cap = 0;
    }
    for (i64 i = 0; i < n; ++i) free(adj[i].v);
    free(adj); free(mark); free(alive); free(nbrs); free(h.d); free(h.u);
    return 0;
}

/* ---------------- LDL' ---------------- */

void oracle_ldl_symbolic(i64 n, const i64 *cp, const i64 *ci, i64 *parent, i64 *lnz, i64 *flag) {
    for (i64 j = 0; j < n; ++j) {
        parent[j] = -1; flag[j] = j; lnz[j] = 0;
        for (i64 p = cp[j]; p < cp[j + 1]; ++p) {
            i64 i = ci[p];
            while (flag[i] != j) {
                if (parent[i] == -1) parent[i] = j;
                lnz[i]++;
                flag[i] = j;
                i = parent[i];
            }
        }
    }
}

#define LDL_NUMERIC(NAME, T)                                                          \
i64 NAME(i64 n, const i64 *cp, const i64 *ci, const T *cx, const i64 *lp,              \
         const i64 *parent, i64 *lnz_count, i64 *li, T *lx, T *d, T *y, i64 *pattern,    \
         i64 *flag, const int8_t *signs, T delta_s, T delta_d) {                         \
    i64 n_bumped = 0;                                                                     \
    double run_max = 0.0;                                                                 \
    for (i64 j = 0; j < n; ++j) {                                                         \
        y[j] = 0;                                                                         \
        i64 top = n;                                                                      \
        flag[j] = j;                                                                      \
        lnz_count[j] = 0;                                                                 \
        for (i64 p = cp[j]; p < cp[j + 1]; ++p) {                                         \
            i64 i = ci[p];                                                                \
            y[i] += cx[p];                                                                \
            i64 len = 0;                                                                  \
            while (flag[i] != j) { pattern[len++] = i; flag[i] = j; i = parent[i]; }      \
            while (len > 0) pattern[--top] = pattern[--len];                              \
        }                                                                                 \
        T djf = y[j];                                                         \
        y[j] = 0;                                                                         \
        for (i64 t = top; t < n; ++t) {                                                   \
            i64 i = pattern[t];                                                           \
            T yi = y[i];                                                                  \
            y[i] = 0;                                                                     \
            i64 p2 = lp[i] + lnz_count[i];                                                \
            for (i64 p = lp[i]; p < p2; ++p) y[li[p]] -= lx[p] * yi;                      \
            T l_ji = yi / d[i];                                                           \
            djf -= l_ji * yi;                                                 \
            li[p2] = j;                                                                   \
            lx[p2] = l_ji;                                                                \
            lnz_count[i]++;                                                               \
        }                                                                                 \
        double dj = (double)djf; double bound = (double)delta_s + (double)delta_d * run_max;                       \
        if (fabs(dj) < bound) { dj = signs[j] > 0 ? bound : -bound; n_bumped++; }         \
        if (dj == 0.0) return -1;                                                         \
        d[j] = (T)dj;                                                                     \
        if (fabs(dj) > run_max) run_max = fabs(dj);                                       \
    }                                                                                     \
    return n_bumped;                                                                      \
}

LDL_NUMERIC(oracle_ldl_numeric_f64, double)
LDL_NUMERIC(oracle_ldl_numeric_f32, float)

#define LDL_SOLVE(NAME, T)                                                               \
void NAME(i64 n, const i64 *lp, const i64 *li, const T *lx, const T *d, T *x) {          \
    for (i64 j = 0; j < n; ++j) {                                                        \
        T xj = x[j];                                                                     \
        for (i64 p = lp[j]; p < lp[j + 1]; ++p) x[li[p]] -= lx[p] * xj;                  \
    }                                                                                    \
    for (i64 j = 0; j < n; ++j) x[j] /= d[j];                                            \
    for (i64 j = n - 1; j >= 0; --j) {                                                   \
        T xj = x[j];                                                                     \
        for (i64 p = lp[j]; p < lp[j + 1]; ++p) xj -= lx[p] * x[li[p]];                  \
        x[j] = xj;                                                                       \
    }                                                                                    \
}

LDL_SOLVE(oracle_ldl_solve_f64, double)
LDL_SOLVE(oracle_ldl_solve_f32, float)

void oracle_symm_matvec(i64 n, const i64 *rowptr, const i64 *colidx, const double *vals,
                        const double *x, double *out) {
    for (i64 i = 0; i < n; ++i) out[i] = 0.0;
    for (i64 i = 0; i < n; ++i) {
        double xi = x[i], acc = 0.0;
        for (i64 p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            i64 j = colidx[p];
            double v = vals[p];
            acc += v * x[j];
            if (j != i) out[j] += v * xi;
        }
        out[i] += acc;
    }
}
