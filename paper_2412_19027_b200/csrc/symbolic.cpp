// Host symbolic analysis for the supernodal LDL' (see symbolic.hpp).
//
// Ordering: the exact-external-degree greedy minimum degree of the reference
// (kkt/ordering.py:15-53: explicit elimination graph, (degree, index) heap
// order) so the elimination tree matches the CPU solver's; the permutation is
// then postordered, which is an equivalent reordering (same fill, same tree).
// A dense-tail shortcut keeps it fast: once the minimum-degree node touches
// every remaining node, the remainder is a clique and the reference order of
// a clique with equal degrees is ascending index.
#include "symbolic.hpp"

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <numeric>
#include <queue>
#include <thread>
#include <chrono>
#include <cstdio>
#include <utility>

namespace cipm {
namespace {

struct Graph {
    std::vector<int64_t> ptr;
    std::vector<int32_t> idx;
};

// symmetric adjacency (no self loops, deduplicated) of the KKT pattern
Graph kkt_graph(int64_t n, int64_t m, const int64_t* prp, const int64_t* pci, const int64_t* arp,
                const int64_t* aci, int64_t nblocks, const int64_t* boff, const int64_t* bdim) {
    const int64_t dim = n + m;
    std::vector<int64_t> deg(dim + 1, 0);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = prp[i]; p < prp[i + 1]; ++p)
            if (pci[p] != i) { deg[i]++; deg[pci[p]]++; }
    for (int64_t r = 0; r < m; ++r)
        for (int64_t p = arp[r]; p < arp[r + 1]; ++p) { deg[aci[p]]++; deg[n + r]++; }
    for (int64_t b = 0; b < nblocks; ++b)
        for (int64_t a = 0; a < bdim[b]; ++a) deg[n + boff[b] + a] += 2 * (bdim[b] - 1);
    std::vector<int64_t> ptr(dim + 1, 0);
    for (int64_t i = 0; i < dim; ++i) ptr[i + 1] = ptr[i] + deg[i];
    std::vector<int32_t> idx(ptr[dim]);
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    auto add = [&](int64_t u, int64_t v) { idx[fill[u]++] = (int32_t)v; };
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = prp[i]; p < prp[i + 1]; ++p)
            if (pci[p] != i) { add(i, pci[p]); add(pci[p], i); }
    for (int64_t r = 0; r < m; ++r)
        for (int64_t p = arp[r]; p < arp[r + 1]; ++p) { add(aci[p], n + r); add(n + r, aci[p]); }
    for (int64_t b = 0; b < nblocks; ++b)
        for (int64_t a = 0; a < bdim[b]; ++a)
            for (int64_t c = 0; c < bdim[b]; ++c)
                if (a != c) { add(n + boff[b] + a, n + boff[b] + c); add(n + boff[b] + c, n + boff[b] + a); }
    Graph g;
    g.ptr.assign(dim + 1, 0);
    g.idx.reserve(idx.size());
    for (int64_t i = 0; i < dim; ++i) {
        auto b = idx.begin() + ptr[i], e = idx.begin() + ptr[i + 1];
        std::sort(b, e);
        auto u = std::unique(b, e);
        g.idx.insert(g.idx.end(), b, u);
        g.ptr[i + 1] = (int64_t)g.idx.size();
    }
    return g;
}

// exact minimum degree (the reference's order); `budget` > 0 caps the elimination-
// graph work (adjacency entries touched): past it the order is abandoned and an
// empty vector returned (the caller switches to the quotient-graph AMD below)
std::vector<int32_t> minimum_degree(const Graph& g, int64_t dim, int64_t budget = 0) {
    std::vector<std::vector<int32_t>> adj(dim);
    int64_t work = 0;
    for (int64_t i = 0; i < dim; ++i) adj[i].assign(g.idx.begin() + g.ptr[i], g.idx.begin() + g.ptr[i + 1]);
    std::vector<char> alive(dim, 1);
    std::vector<int64_t> mark(dim, -1);
    using Item = std::pair<int64_t, int32_t>;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    for (int64_t i = 0; i < dim; ++i) heap.emplace((int64_t)adj[i].size(), (int32_t)i);
    std::vector<int32_t> perm;
    perm.reserve(dim);
    std::vector<int32_t> nbrs;
    int64_t remaining = dim, stamp = 0;
    while ((int64_t)perm.size() < dim) {
        Item it = heap.top();
        heap.pop();
        int32_t v = it.second;
        if (!alive[v] || it.first != (int64_t)adj[v].size()) continue;
        if (it.first == remaining - 1 && remaining > 2) {
            // v touches every remaining node: after eliminating it the rest is a
            // clique with equal degrees, eliminated in ascending index order.
            perm.push_back(v);
            alive[v] = 0;
            for (int64_t i = 0; i < dim; ++i)
                if (alive[i]) perm.push_back((int32_t)i);
            break;
        }
        perm.push_back(v);
        alive[v] = 0;
        remaining--;
        nbrs.clear();
        for (int32_t u : adj[v])
            if (alive[u]) nbrs.push_back(u);
        for (int32_t u : nbrs) {
            auto& au = adj[u];
            for (size_t t = 0; t < au.size(); ++t)
                if (au[t] == v) { au[t] = au.back(); au.pop_back(); break; }
        }
        if (budget > 0) {
            work += (int64_t)nbrs.size() * (int64_t)nbrs.size();
            for (int32_t u : nbrs) work += (int64_t)adj[u].size();
            if (work > budget) return {};
        }
        for (size_t a = 0; a < nbrs.size(); ++a) {
            int32_t u = nbrs[a];
            ++stamp;
            for (int32_t x : adj[u]) mark[x] = stamp;
            for (size_t b = a + 1; b < nbrs.size(); ++b) {
                int32_t w = nbrs[b];
                if (mark[w] != stamp) {
                    adj[u].push_back(w);
                    adj[w].push_back(u);
                }
            }
        }
        for (int32_t u : nbrs) heap.emplace((int64_t)adj[u].size(), u);
        std::vector<int32_t>().swap(adj[v]);
    }
    return perm;
}

// Approximate minimum degree on the quotient graph (ordering = 4, and the
// fallback of the exact order when its elimination graph grows too large — e.g.
// C4's block-simplex rows: the exact order forms every fill clique explicitly).
// Eliminated variables become elements; a variable keeps its element list and
// its remaining variable neighbours, so the work is bounded by the quotient
// graph instead of the filled graph.  Per pivot p (the classic scheme):
//  * L_p = A_p  U  (U_{e in E_p} L_e) \ {p}; the elements of E_p are absorbed;
//  * |L_e \ L_p| for every element touching L_p (weights by supervariable size),
//    elements with L_e subset of L_p absorbed as well (aggressive absorption);
//  * approximate external degree of i in L_p:
//      min(d_i + |L_p \ i|, |A_i| + |L_p \ i| + sum_{e in E_i \ p} |L_e \ L_p|, n_left);
//  * indistinguishable variables (same E_i, same A_i) merged into supervariables,
//    eliminated together.
std::vector<int32_t> approx_min_degree(const Graph& g, int64_t dim) {
    std::vector<std::vector<int32_t>> vars(dim), elems(dim), Le(dim);
    std::vector<int32_t> nv(dim, 1), snext(dim, -1), stail(dim);
    std::vector<int8_t> state(dim, 0);             // 0 variable, 1 element, 2 absorbed element
    std::vector<int64_t> deg(dim), w(dim, 0), wmark(dim, 0), mark(dim, 0);
    std::iota(stail.begin(), stail.end(), 0);
    using Item = std::pair<int64_t, int32_t>;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    for (int64_t i = 0; i < dim; ++i) {
        vars[i].assign(g.idx.begin() + g.ptr[i], g.idx.begin() + g.ptr[i + 1]);
        deg[i] = (int64_t)vars[i].size();
        heap.emplace(deg[i], (int32_t)i);
    }
    std::vector<int32_t> order, Lp;
    order.reserve(dim);
    int64_t nel = 0, tag = 0, wtag = 0;
    while (nel < dim && !heap.empty()) {
        const Item it = heap.top();
        heap.pop();
        const int32_t p = it.second;
        if (state[p] != 0 || nv[p] == 0 || it.first != deg[p]) continue;
        // L_p
        ++tag;
        mark[p] = tag;
        Lp.clear();
        for (int32_t v : vars[p])
            if (state[v] == 0 && nv[v] > 0 && mark[v] != tag) { mark[v] = tag; Lp.push_back(v); }
        for (int32_t e : elems[p]) {
            if (state[e] != 1) continue;
            for (int32_t v : Le[e])
                if (state[v] == 0 && nv[v] > 0 && mark[v] != tag) { mark[v] = tag; Lp.push_back(v); }
            state[e] = 2;
            std::vector<int32_t>().swap(Le[e]);
        }
        for (int32_t v = p; v >= 0; v = snext[v]) order.push_back(v);
        nel += nv[p];
        state[p] = 1;
        std::vector<int32_t>().swap(vars[p]);
        std::vector<int32_t>().swap(elems[p]);
        int64_t dLp = 0;
        for (int32_t v : Lp) dLp += nv[v];
        Le[p] = Lp;
        // |L_e \ L_p| of the other elements touching L_p
        ++wtag;
        for (int32_t i : Lp)
            for (int32_t e : elems[i]) {
                if (state[e] != 1 || e == p) continue;
                if (wmark[e] != wtag) {
                    wmark[e] = wtag;
                    int64_t sz = 0;
                    auto& L = Le[e];
                    size_t k = 0;
                    for (int32_t v : L)
                        if (state[v] == 0 && nv[v] > 0) { L[k++] = v; sz += nv[v]; }
                    L.resize(k);
                    w[e] = sz;
                }
                w[e] -= nv[i];
            }
        for (int32_t i : Lp)          // aggressive absorption: L_e inside L_p
            for (int32_t e : elems[i])
                if (state[e] == 1 && e != p && wmark[e] == wtag && w[e] <= 0) {
                    state[e] = 2;
                    std::vector<int32_t>().swap(Le[e]);
                }
        // update the variables of L_p
        const int64_t left = dim - nel;
        for (int32_t i : Lp) {
            auto& E = elems[i];
            size_t k = 0;
            int64_t ext = 0;
            for (int32_t e : E)
                if (state[e] == 1 && e != p) { E[k++] = e; ext += std::max<int64_t>(w[e], 0); }
            E.resize(k);
            E.push_back(p);
            auto& A = vars[i];
            k = 0;
            int64_t a = 0;
            for (int32_t v : A)
                if (state[v] == 0 && nv[v] > 0 && mark[v] != tag) { A[k++] = v; a += nv[v]; }
            A.resize(k);
            const int64_t lp_ext = dLp - nv[i];
            int64_t d = std::min(deg[i] + lp_ext, a + lp_ext + ext);
            deg[i] = std::max<int64_t>(0, std::min(d, left - nv[i]));
        }
        // supervariables: identical (E_i, A_i) among L_p
        std::vector<std::pair<uint64_t, int32_t>> hs;
        hs.reserve(Lp.size());
        for (int32_t i : Lp) {
            uint64_t h = 1469598103934665603ull;
            std::sort(elems[i].begin(), elems[i].end());
            std::sort(vars[i].begin(), vars[i].end());
            for (int32_t e : elems[i]) h = (h ^ (uint64_t)(e + 1)) * 1099511628211ull;
            h = (h ^ 0x9e3779b97f4a7c15ull) * 1099511628211ull;
            for (int32_t v : vars[i]) h = (h ^ (uint64_t)(v + 1)) * 1099511628211ull;
            hs.emplace_back(h, i);
        }
        std::sort(hs.begin(), hs.end());
        for (size_t a = 0; a < hs.size();) {
            size_t b = a;
            while (b < hs.size() && hs[b].first == hs[a].first) ++b;
            for (size_t x = a; x < b; ++x) {
                const int32_t i = hs[x].second;
                if (nv[i] == 0) continue;
                for (size_t y = x + 1; y < b; ++y) {
                    const int32_t j = hs[y].second;
                    if (nv[j] == 0 || elems[i] != elems[j] || vars[i] != vars[j]) continue;
                    nv[i] += nv[j];
                    deg[i] = std::max<int64_t>(0, deg[i] - nv[j]);
                    nv[j] = 0;
                    snext[stail[i]] = j;
                    stail[i] = stail[j];
                    std::vector<int32_t>().swap(vars[j]);
                    std::vector<int32_t>().swap(elems[j]);
                }
            }
            a = b;
        }
        for (int32_t i : Lp)
            if (nv[i] > 0) heap.emplace(deg[i], i);
    }
    return order;
}

// Nested dissection by BFS level-structure vertex separators (ordering = 2).
// Each part: a pseudo-peripheral start (repeated BFS), BFS levels, the level
// nearest the weighted middle with the fewest nodes inside a balance window as
// the separator, trimmed to the nodes adjacent to the far side; parts at most
// `leaf` nodes are ordered by the exact minimum degree above on their induced
// subgraph.  Separators are numbered after both halves, so the elimination
// tree's height is O(log n) separators instead of MD's long chains on banded
// problems (FP64 results are ordering-independent; the solution-
// level parity contract allows it).
struct NdWork {
    const Graph& g;
    std::vector<int32_t> part;     // part id per node (-1 = already ordered)
    std::vector<int32_t> level;
    std::vector<int32_t> queue;
    std::vector<int32_t> loc;      // node -> local index (leaf subgraph)
    std::vector<int32_t> out;      // the order, separators last within a part
    int32_t next_id = 1;
    int64_t leaf;
    explicit NdWork(const Graph& gg, int64_t dim, int64_t lf)
        : g(gg), part(dim, 0), level(dim, -1), queue(dim), loc(dim, -1), leaf(lf) {}

    // BFS from s inside part id; fills queue[0..cnt), level[]; returns cnt, sets last level
    int64_t bfs(int32_t s, int32_t id, int32_t& maxlev) {
        int64_t head = 0, tail = 0;
        queue[tail++] = s;
        level[s] = 0;
        maxlev = 0;
        while (head < tail) {
            int32_t v = queue[head++];
            for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
                int32_t u = g.idx[p];
                if (part[u] == id && level[u] < 0) {
                    level[u] = level[v] + 1;
                    maxlev = std::max(maxlev, level[u]);
                    queue[tail++] = u;
                }
            }
        }
        return tail;
    }
    void clear_levels(int64_t cnt) {
        for (int64_t k = 0; k < cnt; ++k) level[queue[k]] = -1;
    }

    void order_leaf(const std::vector<int32_t>& nodes) {
        const int64_t k = (int64_t)nodes.size();
        for (int64_t i = 0; i < k; ++i) loc[nodes[i]] = (int32_t)i;
        const int32_t id = part[nodes[0]];
        Graph sg;
        sg.ptr.assign(k + 1, 0);
        for (int64_t i = 0; i < k; ++i) {
            int32_t v = nodes[i];
            for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p)
                if (part[g.idx[p]] == id) sg.idx.push_back(loc[g.idx[p]]);
            sg.ptr[i + 1] = (int64_t)sg.idx.size();
        }
        std::vector<int32_t> pl = minimum_degree(sg, k);
        for (int32_t i : pl) out.push_back(nodes[i]);
        for (int32_t v : nodes) { part[v] = -1; loc[v] = -1; }
    }

    // minimum vertex cover of the edges between BFS levels sl and sl+1 of the part
    // (queue[0..cnt) holds the part's nodes with their levels); cover[k] marks queue[k]
    void min_cover_between_levels(int64_t cnt, int32_t id, int32_t sl, std::vector<char>& cover) {
        min_cover_between_levels(queue, cnt, id, sl, cover);
    }
    void min_cover_between_levels(const std::vector<int32_t>& q, int64_t cnt, int32_t id, int32_t sl,
                                  std::vector<char>& cover) {
        cover.assign(cnt, 0);
        // U = level sl nodes with an edge to sl+1, V = level sl+1 nodes with an edge to sl
        std::vector<int32_t> U, V;
        for (int64_t k = 0; k < cnt; ++k) {
            const int32_t v = q[k];
            if (level[v] != sl && level[v] != sl + 1) continue;
            const int32_t other = level[v] == sl ? sl + 1 : sl;
            bool touches = false;
            for (int64_t p = g.ptr[v]; p < g.ptr[v + 1] && !touches; ++p) {
                const int32_t u = g.idx[p];
                touches = part[u] == id && level[u] == other;
            }
            if (!touches) continue;
            loc[v] = (int32_t)(level[v] == sl ? U.size() : V.size());
            (level[v] == sl ? U : V).push_back(v);
        }
        const int32_t nu = (int32_t)U.size(), nv = (int32_t)V.size();
        std::vector<int32_t> mu(nu, -1), mv(nv, -1), dist(nu);
        auto nbrs = [&](int32_t ui, auto&& f) {
            const int32_t v = U[ui];
            for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
                const int32_t w = g.idx[p];
                if (part[w] == id && level[w] == sl + 1 && loc[w] >= 0) f(loc[w]);
            }
        };
        // Hopcroft-Karp
        std::vector<int32_t> bfsq(nu);
        for (;;) {
            int64_t h = 0, t = 0;
            bool found = false;
            for (int32_t ui = 0; ui < nu; ++ui) {
                dist[ui] = mu[ui] < 0 ? 0 : -1;
                if (mu[ui] < 0) bfsq[t++] = ui;
            }
            while (h < t) {
                const int32_t ui = bfsq[h++];
                nbrs(ui, [&](int32_t vi) {
                    const int32_t u2 = mv[vi];
                    if (u2 < 0) found = true;
                    else if (dist[u2] < 0) { dist[u2] = dist[ui] + 1; bfsq[t++] = u2; }
                });
            }
            if (!found) break;
            std::function<bool(int32_t)> dfs = [&](int32_t ui) -> bool {
                const int32_t v = U[ui];
                for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
                    const int32_t w = g.idx[p];
                    if (!(part[w] == id && level[w] == sl + 1 && loc[w] >= 0)) continue;
                    const int32_t vi = loc[w], u2 = mv[vi];
                    if (u2 < 0 || (dist[u2] == dist[ui] + 1 && dfs(u2))) {
                        mu[ui] = vi;
                        mv[vi] = ui;
                        return true;
                    }
                }
                dist[ui] = -1;
                return false;
            };
            for (int32_t ui = 0; ui < nu; ++ui)
                if (mu[ui] < 0) dfs(ui);
        }
        // Koenig: Z = reachable from unmatched U by alternating paths; cover = (U \ Z) + (V & Z)
        std::vector<char> zu(nu, 0), zv(nv, 0);
        std::vector<int32_t> st;
        for (int32_t ui = 0; ui < nu; ++ui)
            if (mu[ui] < 0) { zu[ui] = 1; st.push_back(ui); }
        while (!st.empty()) {
            const int32_t ui = st.back();
            st.pop_back();
            nbrs(ui, [&](int32_t vi) {
                if (zv[vi] || mu[ui] == vi) return;
                zv[vi] = 1;
                const int32_t u2 = mv[vi];
                if (u2 >= 0 && !zu[u2]) { zu[u2] = 1; st.push_back(u2); }
            });
        }
        std::vector<char> inS(0);
        for (int64_t k = 0; k < cnt; ++k) {
            const int32_t v = q[k];
            if (loc[v] < 0) continue;
            if (level[v] == sl) cover[k] = zu[loc[v]] ? 0 : 1;
            else if (level[v] == sl + 1) cover[k] = zv[loc[v]] ? 1 : 0;
        }
        for (int32_t v : U) loc[v] = -1;
        for (int32_t v : V) loc[v] = -1;
    }

    // order the part `id` whose nodes are `nodes` (appends to out)
    void dissect(std::vector<int32_t> nodes) {
        struct Item { std::vector<int32_t> nodes; int stage; std::vector<int32_t> sep; };
        std::vector<Item> stack;
        stack.push_back({std::move(nodes), 0, {}});
        while (!stack.empty()) {
            Item& it = stack.back();
            if (it.stage == 1) {            // both halves ordered: the separator goes last
                for (int32_t v : it.sep) { out.push_back(v); part[v] = -1; }
                stack.pop_back();
                continue;
            }
            std::vector<int32_t> cur = std::move(it.nodes);
            const int32_t id = part[cur[0]];
            if ((int64_t)cur.size() <= leaf) {
                stack.pop_back();
                order_leaf(cur);
                continue;
            }
            // connected components, all found in one pass; each is ordered on its own
            int32_t s = cur[0], maxlev = 0;
            int64_t cnt = bfs(s, id, maxlev);
            if (cnt < (int64_t)cur.size()) {
                std::vector<std::vector<int32_t>> comps;
                comps.emplace_back(queue.begin(), queue.begin() + cnt);
                for (int32_t v : cur) {
                    if (level[v] >= 0) continue;
                    int32_t ml = 0;
                    const int64_t c2 = bfs(v, id, ml);
                    comps.emplace_back(queue.begin(), queue.begin() + c2);
                }
                for (int32_t v : cur) level[v] = -1;
                stack.pop_back();
                for (auto& comp : comps) {
                    const int32_t nid = next_id++;
                    for (int32_t v : comp) part[v] = nid;
                    stack.push_back({std::move(comp), 0, {}});
                }
                continue;
            }
            for (int sweep = 0; sweep < 3; ++sweep) {
                int32_t best = -1;
                int64_t bdeg = INT64_MAX;
                for (int64_t k = cnt - 1; k >= 0 && level[queue[k]] == maxlev; --k) {
                    int32_t v = queue[k];
                    int64_t dg = g.ptr[v + 1] - g.ptr[v];
                    if (dg < bdeg) { bdeg = dg; best = v; }
                }
                clear_levels(cnt);
                int32_t ml2 = 0;
                cnt = bfs(best, id, ml2);
                if (ml2 <= maxlev) { maxlev = ml2; s = best; break; }
                maxlev = ml2;
                s = best;
            }
            // level sizes; separator level: fewest nodes within the balance window
            std::vector<int64_t> lsz(maxlev + 2, 0);
            for (int64_t k = 0; k < cnt; ++k) lsz[level[queue[k]]]++;
            int64_t below = 0, bestsz = INT64_MAX;
            int32_t sl = -1;
            const int64_t tot = cnt;
            for (int32_t l = 1; l < maxlev; ++l) {
                below += lsz[l - 1];
                const int64_t above = tot - below - lsz[l];
                const double bal = (double)std::min(below, above) / (double)tot;
                if (bal < 0.3) continue;
                if (lsz[l] < bestsz) { bestsz = lsz[l]; sl = l; }
            }
            if (sl < 0) {
                // no balanced level (e.g. a star): fall back to the middle level
                below = 0;
                for (int32_t l = 0; l <= maxlev; ++l) {
                    if (below + lsz[l] >= tot / 2) { sl = l; break; }
                    below += lsz[l];
                }
                if (sl <= 0 || sl >= maxlev) {
                    clear_levels(cnt);
                    stack.pop_back();
                    order_leaf(cur);       // cannot split: minimum degree on the whole part
                    continue;
                }
            }
            // separator: a minimum vertex cover of the bipartite graph of the edges
            // between levels sl and sl+1 (Koenig: maximum matching, then the cover from
            // the alternating reachability), never larger than the level-sl boundary; the
            // uncovered level-sl nodes join the low side, the uncovered level-(sl+1) nodes
            // the high side (BFS levels only touch adjacent levels, so the cover separates)
            const int32_t lo = next_id++, hi = next_id++;
            std::vector<int32_t> A, B, S;
            std::vector<char> cover;
            min_cover_between_levels(queue, cnt, id, sl, cover);
            for (int64_t k = 0; k < cnt; ++k) {
                int32_t v = queue[k];
                int32_t lv = level[v];
                if (cover[k]) S.push_back(v);
                else if (lv <= sl) A.push_back(v);
                else B.push_back(v);
            }
            clear_levels(cnt);
            const int32_t sid = next_id++;
            for (int32_t v : A) part[v] = lo;
            for (int32_t v : B) part[v] = hi;
            for (int32_t v : S) part[v] = sid;
            it.stage = 1;
            it.sep = std::move(S);
            if (!B.empty()) stack.push_back({std::move(B), 0, {}});
            if (!A.empty()) stack.push_back({std::move(A), 0, {}});
        }
    }
};

std::vector<int32_t> nested_dissection(const Graph& g, int64_t dim, int64_t leaf) {
    NdWork w(g, dim, leaf);
    w.out.reserve(dim);
    // pendant nodes (degree <= 1: e.g. the lasso's y_i hanging off its zero row) are
    // eliminated first — no fill — and kept out of the BFS levels, where every
    // pendant edge would otherwise have to be cut by the separator
    std::vector<int32_t> rest;
    rest.reserve(dim);
    for (int64_t v = 0; v < dim; ++v) {
        if (g.ptr[v + 1] - g.ptr[v] <= 1) {
            w.out.push_back((int32_t)v);
            w.part[v] = -1;
        } else {
            rest.push_back((int32_t)v);
        }
    }
    if (!rest.empty()) w.dissect(std::move(rest));
    return w.out;
}

// upper CSC of the permuted pattern: column c holds rows r < c
void permuted_upper(const Graph& g, const std::vector<int32_t>& iperm, int64_t dim,
                    std::vector<int64_t>& cp, std::vector<int32_t>& ci) {
    cp.assign(dim + 1, 0);
    for (int64_t i = 0; i < dim; ++i)
        for (int64_t p = g.ptr[i]; p < g.ptr[i + 1]; ++p) {
            int32_t pi = iperm[i], pj = iperm[g.idx[p]];
            if (pi < pj) cp[pj + 1]++;
        }
    for (int64_t c = 0; c < dim; ++c) cp[c + 1] += cp[c];
    ci.assign(cp[dim], 0);
    std::vector<int64_t> fill(cp.begin(), cp.end() - 1);
    for (int64_t i = 0; i < dim; ++i)
        for (int64_t p = g.ptr[i]; p < g.ptr[i + 1]; ++p) {
            int32_t pi = iperm[i], pj = iperm[g.idx[p]];
            if (pi < pj) ci[fill[pj]++] = pi;
        }
    for (int64_t c = 0; c < dim; ++c) std::sort(ci.begin() + cp[c], ci.begin() + cp[c + 1]);
}

std::vector<int32_t> etree(const std::vector<int64_t>& cp, const std::vector<int32_t>& ci, int64_t dim) {
    std::vector<int32_t> parent(dim, -1), anc(dim, -1);
    for (int64_t c = 0; c < dim; ++c) {
        for (int64_t p = cp[c]; p < cp[c + 1]; ++p) {
            int32_t r = ci[p];
            while (r != -1 && r < c) {
                int32_t next = anc[r];
                anc[r] = (int32_t)c;
                if (next == -1) { parent[r] = (int32_t)c; break; }
                r = next;
            }
        }
    }
    return parent;
}

// postorder; children are visited in ascending (weight, index) order so the
// child with the largest column count — the chain continuation of a dense
// tail — is numbered immediately before its parent and can join its supernode
std::vector<int32_t> postorder(const std::vector<int32_t>& parent, const std::vector<int64_t>& weight,
                               int64_t dim) {
    std::vector<int32_t> kids(dim);
    std::iota(kids.begin(), kids.end(), 0);
    std::stable_sort(kids.begin(), kids.end(), [&](int32_t a, int32_t b) { return weight[a] > weight[b]; });
    std::vector<int32_t> head(dim, -1), next(dim, -1);
    for (int32_t j : kids) {                        // push heaviest first -> visited last
        if (parent[j] == -1) continue;
        next[j] = head[parent[j]];
        head[parent[j]] = j;
    }
    std::vector<int32_t> post;
    post.reserve(dim);
    std::vector<int32_t> stack;
    for (int64_t r = 0; r < dim; ++r) {
        if (parent[r] != -1) continue;
        stack.push_back((int32_t)r);
        while (!stack.empty()) {
            int32_t t = stack.back();
            int32_t c = head[t];
            if (c == -1) {
                post.push_back(t);
                stack.pop_back();
            } else {
                head[t] = next[c];
                stack.push_back(c);
            }
        }
    }
    return post;
}


// nnz(L) and 2*sum c_j^2 of an ordering (etree + path-walk column counts),
// abandoned (returns false) once nnz exceeds `budget`
bool fill_stats(const Graph& g, const std::vector<int32_t>& perm, int64_t dim, int64_t budget, int64_t& nnz,
                double& flops) {
    std::vector<int32_t> iperm(dim);
    for (int64_t k = 0; k < dim; ++k) iperm[perm[k]] = (int32_t)k;
    std::vector<int64_t> cp;
    std::vector<int32_t> ci;
    permuted_upper(g, iperm, dim, cp, ci);
    std::vector<int32_t> parent = etree(cp, ci, dim);
    std::vector<int64_t> cnt(dim, 0);
    std::vector<int32_t> fl(dim, -1);
    nnz = 0;
    for (int64_t j = 0; j < dim; ++j) {
        fl[j] = (int32_t)j;
        for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
            for (int32_t i = ci[p]; fl[i] != j; i = parent[i]) { cnt[i]++; fl[i] = (int32_t)j; nnz++; }
        if (nnz > budget) return false;
    }
    flops = 0.0;
    for (int64_t j = 0; j < dim; ++j) flops += 2.0 * (double)cnt[j] * (double)cnt[j];
    return true;
}

// ordering 3 (auto): the reference's minimum degree for small systems; for
// large ones minimum degree and nested dissection are computed concurrently
// and nested dissection is kept when its fill and flops stay close to MD's
// (banded problems: same fill, a 4x shallower elimination tree)
std::vector<int32_t> auto_order(const Graph& g, int64_t dim, const SymbolicOptions& opt, int* chosen) {
    if (dim < opt.auto_min_dim) {
        *chosen = 0;
        return minimum_degree(g, dim);
    }
    std::vector<int32_t> md, nd;
    std::thread t([&] { nd = nested_dissection(g, dim, opt.nd_leaf); });
    // the reference's exact order while its elimination graph stays moderate, else AMD
    md = minimum_degree(g, dim, opt.md_work_budget_per_nnz * (int64_t)(g.ptr[dim] + dim));
    const bool amd = (int64_t)md.size() != dim;
    if (amd) md = approx_min_degree(g, dim);
    t.join();
    int64_t nnz_md = 0, nnz_nd = 0;
    double fl_md = 0, fl_nd = 0;
    fill_stats(g, md, dim, INT64_MAX, nnz_md, fl_md);
    const bool ok = fill_stats(g, nd, dim, (int64_t)(opt.nd_max_fill * (double)nnz_md), nnz_nd, fl_nd);
    if (ok && fl_nd <= opt.nd_max_flops * fl_md) {
        *chosen = 2;
        return nd;
    }
    *chosen = amd ? 4 : 0;
    return md;
}
}  // namespace

namespace {
struct SymTimer {
    bool on = getenv("CIPM_SYM_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[symbolic] %-28s %8.3f s\n", what, std::chrono::duration<double>(t - t0).count());
        t0 = t;
    }
};
}  // namespace

int analyze(int64_t n, int64_t m, const int64_t* prp, const int64_t* pci, const int64_t* arp,
            const int64_t* aci, int64_t lin, int64_t nblocks, const int64_t* boff, const int64_t* bdim,
            const SymbolicOptions& opt, Symbolic& S) {
    const int64_t dim = n + m;
    S.n = n;
    S.m = m;
    S.dim = dim;
    Graph g = kkt_graph(n, m, prp, pci, arp, aci, nblocks, boff, bdim);

    SymTimer T;
    std::vector<int32_t> perm;
    S.ordering_used = opt.ordering == 3 ? 0 : opt.ordering;
    if (opt.ordering == 1) {
        perm.resize(dim);
        std::iota(perm.begin(), perm.end(), 0);
    } else if (opt.ordering == 2) {
        perm = nested_dissection(g, dim, opt.nd_leaf);
    } else if (opt.ordering == 3) {
        int chosen = 0;
        perm = auto_order(g, dim, opt, &chosen);
        S.ordering_used = chosen;
    } else if (opt.ordering == 4) {
        perm = approx_min_degree(g, dim);
    } else {
        perm = minimum_degree(g, dim);
    }
    S.md_perm = perm;
    T.mark("ordering");
    std::vector<int32_t> iperm(dim);
    for (int64_t k = 0; k < dim; ++k) iperm[perm[k]] = (int32_t)k;

    std::vector<int64_t> cp;
    std::vector<int32_t> ci;
    permuted_upper(g, iperm, dim, cp, ci);
    std::vector<int32_t> parent = etree(cp, ci, dim);
    std::vector<int64_t> cnt0(dim, 0);
    {
        std::vector<int32_t> fl(dim, -1);
        for (int64_t j = 0; j < dim; ++j) {
            fl[j] = (int32_t)j;
            for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
                for (int32_t i = ci[p]; fl[i] != j; i = parent[i]) { cnt0[i]++; fl[i] = (int32_t)j; }
        }
    }
    // postorder weight: subtree height first (the critical-path child is numbered
    // immediately before its parent, so the top chain is contiguous and can be
    // merged), column count second (a dense tail's continuation joins its supernode)
    std::vector<int64_t> height_col(dim, 1);
    for (int64_t j = 0; j < dim; ++j)
        if (parent[j] != -1) height_col[parent[j]] = std::max(height_col[parent[j]], height_col[j] + 1);
    std::vector<int64_t> pweight(dim);
    for (int64_t j = 0; j < dim; ++j) pweight[j] = (height_col[j] << 32) + cnt0[j];
    std::vector<int32_t> post = postorder(parent, pweight, dim);
    {
        std::vector<int32_t> p2(dim);
        for (int64_t k = 0; k < dim; ++k) p2[k] = perm[post[k]];
        perm.swap(p2);
        for (int64_t k = 0; k < dim; ++k) iperm[perm[k]] = (int32_t)k;
        permuted_upper(g, iperm, dim, cp, ci);
        parent = etree(cp, ci, dim);
    }
    S.perm = perm;
    S.iperm = iperm;
    S.sign.resize(dim);
    for (int64_t k = 0; k < dim; ++k) S.sign[k] = perm[k] < n ? 1 : -1;

    T.mark("etree + postorder");
    // column structures of L (strict lower), row-by-row reach through the etree
    std::vector<int64_t> cnt(dim, 0);
    std::vector<int32_t> flag(dim, -1);
    for (int64_t j = 0; j < dim; ++j) {
        flag[j] = (int32_t)j;
        for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
            for (int32_t i = ci[p]; flag[i] != j; i = parent[i]) { cnt[i]++; flag[i] = (int32_t)j; }
    }
    std::vector<int64_t> lp(dim + 1, 0);
    for (int64_t j = 0; j < dim; ++j) lp[j + 1] = lp[j] + cnt[j];
    std::vector<int32_t> li(lp[dim]);
    {
        std::vector<int64_t> fill(lp.begin(), lp.end() - 1);
        std::fill(flag.begin(), flag.end(), -1);
        for (int64_t j = 0; j < dim; ++j) {
            flag[j] = (int32_t)j;
            for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
                for (int32_t i = ci[p]; flag[i] != j; i = parent[i]) { li[fill[i]++] = (int32_t)j; flag[i] = (int32_t)j; }
        }
    }
    S.nnz_l = lp[dim];
    S.flops = 0.0;
    for (int64_t j = 0; j < dim; ++j) S.flops += 2.0 * (double)cnt[j] * (double)cnt[j];

    T.mark("column structures");
    // fundamental supernodes
    std::vector<int32_t> nchild(dim, 0);
    for (int64_t j = 0; j < dim; ++j)
        if (parent[j] != -1) nchild[parent[j]]++;
    std::vector<int32_t> fstart;
    for (int64_t j = 0; j < dim; ++j) {
        // columns j-1, j share a structure when j is j-1's parent and the counts nest;
        // other subtrees may attach to j (they become children of the supernode)
        bool cont = j > 0 && parent[j - 1] == j && cnt[j - 1] == cnt[j] + 1;
        if (!cont) fstart.push_back((int32_t)j);
    }
    const int64_t nf = (int64_t)fstart.size();
    fstart.push_back((int32_t)dim);
    std::vector<int32_t> fsn(dim);
    for (int64_t s = 0; s < nf; ++s)
        for (int32_t j = fstart[s]; j < fstart[s + 1]; ++j) fsn[j] = (int32_t)s;
    std::vector<int32_t> fparent(nf, -1);
    for (int64_t s = 0; s < nf; ++s) {
        int32_t last = fstart[s + 1] - 1;
        fparent[s] = parent[last] == -1 ? -1 : fsn[parent[last]];
    }
    // relaxed amalgamation, top-down with union-find representatives
    std::vector<int32_t> rep(nf);
    std::iota(rep.begin(), rep.end(), 0);
    std::function<int32_t(int32_t)> find = [&](int32_t x) {
        while (rep[x] != x) { rep[x] = rep[rep[x]]; x = rep[x]; }
        return x;
    };
    std::vector<int64_t> first(nf), width(nf), offr(nf), truenz(nf);
    for (int64_t s = 0; s < nf; ++s) {
        first[s] = fstart[s];
        width[s] = fstart[s + 1] - fstart[s];
        offr[s] = cnt[fstart[s + 1] - 1];                 // rows below the last column
        int64_t t = 0;
        for (int32_t j = fstart[s]; j < fstart[s + 1]; ++j) t += cnt[j] + 1;
        truenz[s] = t;
    }
    for (int64_t s = nf - 2; s >= 0; --s) {
        if (fparent[s] == -1) continue;
        int32_t P = find(fparent[s]);
        if (fstart[s + 1] != first[P]) continue;         // not adjacent
        int64_t w = width[s] + width[P];
        int64_t r = w + offr[P];
        double size = (double)w * (double)r - 0.5 * (double)w * (double)(w - 1);
        double zeros = size - (double)(truenz[s] + truenz[P]);
        double frac = size > 0 ? zeros / size : 0.0;
        bool ok = w <= opt.relax_small || (w <= opt.relax_mid && frac <= opt.relax_mid_frac) ||
                  (w <= opt.relax_big && frac <= opt.relax_big_frac);
        if (!ok) continue;
        rep[s] = P;
        first[P] = first[s];
        width[P] = w;
        truenz[P] += truenz[s];
    }
    // top-chain merge: the single-child chain hanging below each root is one long
    // sequential path through the elimination tree (one dependency hop per
    // supernode in every factorisation and triangular sweep).  Merged into one
    // dense supernode it becomes a dense-tail node (multi-CTA blocked kernels).
    int64_t chain_max = opt.chain_merge_max;
    if (const char* e = getenv("CIPM_CHAIN_MERGE")) chain_max = atoll(e);   // experiments
    if (chain_max > 0) {
        // the child adjacent in postorder (numbered immediately before its parent) is
        // the heaviest one: the critical-path continuation
        std::vector<int32_t> adj(nf, -1);
        for (int64_t s = 0; s < nf; ++s) {
            if (find((int32_t)s) != s || fparent[s] == -1) continue;
            const int32_t P = find(fparent[s]);
            if (first[s] + width[s] == first[P]) adj[P] = (int32_t)s;
        }
        for (int64_t R = 0; R < nf; ++R) {
            if (find((int32_t)R) != R || fparent[R] != -1) continue;
            std::vector<int32_t> chain;
            int32_t cur = (int32_t)R;
            int64_t wsum = width[R];
            while (adj[cur] >= 0) {
                const int32_t ch = adj[cur];
                if (wsum + width[ch] > chain_max) break;
                chain.push_back(ch);
                wsum += width[ch];
                cur = ch;
            }
            if (chain.size() < 2 || wsum < opt.tail_width) continue;
            for (int32_t ch : chain) {
                rep[ch] = (int32_t)R;
                first[R] = first[ch];
                truenz[R] += truenz[ch];
            }
            width[R] = wsum;
        }
    }
    // final supernodes in column order
    std::vector<int32_t> sid(nf, -1);
    int32_t ns = 0;
    for (int64_t s = 0; s < nf; ++s) {
        int32_t r = find((int32_t)s);
        if (sid[r] == -1) sid[r] = -2;  // placeholder
    }
    S.sn_col.clear();
    S.col2sn.assign(dim, -1);
    for (int64_t j = 0; j < dim; ++j) {
        int32_t r = find(fsn[j]);
        if (sid[r] < 0) {
            sid[r] = ns++;
            S.sn_col.push_back((int32_t)j);
        }
        S.col2sn[j] = sid[r];
    }
    S.sn_col.push_back((int32_t)dim);
    S.nsuper = ns;
    T.mark("supernodes + amalgamation");
    // row lists: own columns then union of column structures beyond the last column
    S.sn_rptr.assign(ns + 1, 0);
    S.sn_rows.clear();
    std::fill(flag.begin(), flag.end(), -1);
    std::vector<int32_t> tmp;
    for (int32_t J = 0; J < ns; ++J) {
        int32_t c0 = S.sn_col[J], c1 = S.sn_col[J + 1];
        tmp.clear();
        for (int32_t j = c0; j < c1; ++j)
            for (int64_t p = lp[j]; p < lp[j + 1]; ++p) {
                int32_t r = li[p];
                if (r >= c1 && flag[r] != J) { flag[r] = J; tmp.push_back(r); }
            }
        std::sort(tmp.begin(), tmp.end());
        for (int32_t j = c0; j < c1; ++j) S.sn_rows.push_back(j);
        S.sn_rows.insert(S.sn_rows.end(), tmp.begin(), tmp.end());
        S.sn_rptr[J + 1] = (int64_t)S.sn_rows.size();
    }
    S.sn_loff.assign(ns + 1, 0);
    S.max_width = S.max_rows = 0;
    for (int32_t J = 0; J < ns; ++J) {
        int64_t w = S.sn_col[J + 1] - S.sn_col[J];
        int64_t r = S.sn_rptr[J + 1] - S.sn_rptr[J];
        S.sn_loff[J + 1] = S.sn_loff[J] + ((w * r + 3) & ~int64_t(3));   // 16-byte aligned panels (TMA bulk)
        S.max_width = std::max(S.max_width, w);
        S.max_rows = std::max(S.max_rows, r);
        S.max_panel = std::max(S.max_panel, w * r);
    }
    S.nnz_storage = S.sn_loff[ns] + 4;   // bulk copies may read up to 16 bytes past a panel
    S.sn_parent.assign(ns, -1);
    S.sn_nchild.assign(ns, 0);
    for (int32_t J = 0; J < ns; ++J) {
        int64_t w = S.sn_col[J + 1] - S.sn_col[J];
        int64_t r = S.sn_rptr[J + 1] - S.sn_rptr[J];
        if (r > w) {
            S.sn_parent[J] = S.col2sn[S.sn_rows[S.sn_rptr[J] + w]];
            S.sn_nchild[S.sn_parent[J]]++;
        }
    }
    T.mark("row lists");
    // update lists (K -> J), K ascending inside each J
    std::vector<int64_t> ucount(ns + 1, 0);
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<int64_t> fillp;
        if (pass == 1) {
            S.upd_ptr.assign(ns + 1, 0);
            for (int32_t J = 0; J < ns; ++J) S.upd_ptr[J + 1] = S.upd_ptr[J] + ucount[J];
            S.upd_src.assign(S.upd_ptr[ns], 0);
            S.upd_p0.assign(S.upd_ptr[ns], 0);
            S.upd_p1.assign(S.upd_ptr[ns], 0);
            fillp.assign(S.upd_ptr.begin(), S.upd_ptr.end() - 1);
        }
        for (int32_t K = 0; K < ns; ++K) {
            int64_t w = S.sn_col[K + 1] - S.sn_col[K];
            int64_t r0 = S.sn_rptr[K], r = S.sn_rptr[K + 1] - r0;
            int64_t p = w;
            while (p < r) {
                int32_t J = S.col2sn[S.sn_rows[r0 + p]];
                int64_t q = p;
                while (q < r && S.col2sn[S.sn_rows[r0 + q]] == J) ++q;
                if (pass == 0) {
                    ucount[J]++;
                } else {
                    int64_t t = fillp[J]++;
                    S.upd_src[t] = K;
                    S.upd_p0[t] = (int32_t)p;
                    S.upd_p1[t] = (int32_t)q;
                }
                p = q;
            }
        }
    }
    S.n_updates = S.upd_ptr[ns];
    T.mark("update lists");
    // inbox maps for the push/pull factorisation and forward solve
    {
        S.cb_off.assign(ns + 1, 0);
        S.cv_off.assign(ns + 1, 0);
        for (int32_t K = 0; K < ns; ++K) {
            int64_t w = S.sn_col[K + 1] - S.sn_col[K];
            int64_t o = (S.sn_rptr[K + 1] - S.sn_rptr[K]) - w;
            S.cb_off[K + 1] = S.cb_off[K] + o * (o + 1) / 2;
            S.cv_off[K + 1] = S.cv_off[K] + o;
        }
        const int64_t nrec = S.cb_off[ns];
        const int64_t nrow_all = (int64_t)S.sn_rows.size();
        // pass 1: count entries per (J, tr) bucket (global row slot = sn_rptr[J] + tr)
        std::vector<int64_t> cnt_row(nrow_all + 1, 0);
        std::vector<int32_t> tr_of;   // per K scratch: local row in the target supernode
        std::vector<int64_t> src_of;  // inbox slot -> contribution record
        for (int pass = 0; pass < 2; ++pass) {
            std::vector<int64_t> fillp;
            if (pass == 1) {
                S.irow_ptr.assign(nrow_all + 1, 0);
                for (int64_t t = 0; t < nrow_all; ++t) S.irow_ptr[t + 1] = S.irow_ptr[t] + cnt_row[t];
                S.push_pos.assign(nrec, 0);
                S.inbox_tgt.assign(nrec, 0);
                src_of.assign(nrec, 0);
                fillp.assign(S.irow_ptr.begin(), S.irow_ptr.end() - 1);
            }
            for (int32_t K = 0; K < ns; ++K) {
                const int64_t w = S.sn_col[K + 1] - S.sn_col[K];
                const int64_t r0 = S.sn_rptr[K];
                const int64_t o = (S.sn_rptr[K + 1] - r0) - w;
                if (o == 0) continue;
                const int32_t* offrows = S.sn_rows.data() + r0 + w;
                // target supernode of every off row; the off rows are ascending, so the
                // targets are too, and each target's local rows of offrows[b..) come from
                // ONE merge walk per distinct target (not a search per entry)
                std::vector<int32_t> tJ(o), tloc(o);
                for (int64_t a = 0; a < o; ++a) tJ[a] = S.col2sn[offrows[a]];
                int64_t t = 0;
                int32_t curJ = -1;
                for (int64_t b = 0; b < o; ++b) {
                    const int32_t J = tJ[b];
                    const int32_t c0 = S.sn_col[J];
                    const int32_t* rowsJ = S.sn_rows.data() + S.sn_rptr[J];
                    const int64_t rJ = S.sn_rptr[J + 1] - S.sn_rptr[J];
                    if (J != curJ) {
                        curJ = J;
                        int64_t q = std::lower_bound(rowsJ, rowsJ + rJ, offrows[b]) - rowsJ;
                        for (int64_t a = b; a < o; ++a) {
                            while (q < rJ && rowsJ[q] < offrows[a]) ++q;
                            tloc[a] = (int32_t)q;
                        }
                    }
                    const int32_t tc = offrows[b] - c0;
                    for (int64_t a = b; a < o; ++a, ++t) {
                        const int32_t tr = tloc[a];
                        const int64_t slot = S.sn_rptr[J] + tr;
                        if (pass == 0) {
                            cnt_row[slot]++;
                        } else {
                            const int64_t e = fillp[slot]++;
                            S.push_pos[S.cb_off[K] + t] = e;
                            S.inbox_tgt[e] = (int32_t)(tc * rJ + tr);
                            src_of[e] = S.cb_off[K] + t;
                        }
                    }
                }
            }
        }
        // within each row bucket: order by target column, ties by arrival (source K
        // ascending) — one sort of packed (target, arrival) keys per bucket
        {
            std::vector<uint64_t> key;
            std::vector<int64_t> src;
            for (int64_t t = 0; t < nrow_all; ++t) {
                const int64_t lo = S.irow_ptr[t], hi = S.irow_ptr[t + 1];
                if (hi - lo < 2) continue;
                const int64_t nb = hi - lo;
                key.resize(nb);
                for (int64_t k = 0; k < nb; ++k) key[k] = ((uint64_t)(uint32_t)S.inbox_tgt[lo + k] << 32) | (uint64_t)k;
                bool sorted = true;
                for (int64_t k = 1; k < nb && sorted; ++k) sorted = key[k - 1] <= key[k];
                if (sorted) continue;
                std::sort(key.begin(), key.end());
                src.resize(nb);
                for (int64_t k = 0; k < nb; ++k) src[k] = src_of[lo + (int64_t)(key[k] & 0xffffffffu)];
                for (int64_t k = 0; k < nb; ++k) {
                    S.inbox_tgt[lo + k] = (int32_t)(key[k] >> 32);
                    S.push_pos[src[k]] = lo + k;
                }
            }
        }
        // vector inbox: bucket by target column, source K ascending
        S.vcol_ptr.assign(dim + 1, 0);
        for (int32_t K = 0; K < ns; ++K) {
            const int64_t w = S.sn_col[K + 1] - S.sn_col[K];
            for (int64_t p = S.sn_rptr[K] + w; p < S.sn_rptr[K + 1]; ++p) S.vcol_ptr[S.sn_rows[p] + 1]++;
        }
        for (int64_t j = 0; j < dim; ++j) S.vcol_ptr[j + 1] += S.vcol_ptr[j];
        S.vpush_pos.assign(S.cv_off[ns], 0);
        std::vector<int64_t> vf(S.vcol_ptr.begin(), S.vcol_ptr.end() - 1);
        for (int32_t K = 0; K < ns; ++K) {
            const int64_t w = S.sn_col[K + 1] - S.sn_col[K];
            int64_t a = 0;
            for (int64_t p = S.sn_rptr[K] + w; p < S.sn_rptr[K + 1]; ++p, ++a)
                S.vpush_pos[S.cv_off[K] + a] = vf[S.sn_rows[p]]++;
        }
    }
    T.mark("inbox maps");
    // levels and topological order
    S.level.assign(ns, 0);
    for (int32_t J = 0; J < ns; ++J)
        if (S.sn_parent[J] != -1) S.level[S.sn_parent[J]] = std::max(S.level[S.sn_parent[J]], S.level[J] + 1);
    S.height = 0;
    for (int32_t J = 0; J < ns; ++J) S.height = std::max(S.height, S.level[J] + 1);
    // dense tail: supernodes whose panel or contribution block is large enough
    // for the multi-CTA tensor-core path (dense.cu), plus all their ancestors.
    // The complement is closed under descendants, so the persistent kernels
    // finish it before the tail starts.
    S.is_tail.assign(ns, 0);
    const int64_t tail_w = std::min<int64_t>(opt.tail_width, 64);   // the persistent kernels hold w < 64 columns
    int64_t tail_off = opt.tail_offrows;
    if (const char* e = getenv("CIPM_TAIL_OFFROWS")) tail_off = atoll(e);   // experiments
    for (int32_t J = 0; J < ns; ++J) {
        int64_t w = S.sn_col[J + 1] - S.sn_col[J];
        int64_t o = (S.sn_rptr[J + 1] - S.sn_rptr[J]) - w;
        if (w >= tail_w || o >= tail_off) S.is_tail[J] = 1;
    }
    for (int32_t J = 0; J < ns; ++J)       // parents have larger indices (postorder)
        if (S.is_tail[J] && S.sn_parent[J] >= 0) S.is_tail[S.sn_parent[J]] = 1;
    // mid tier: large panels / inboxes and all their (non-tail) ancestors
    S.is_mid.assign(ns, 0);
    for (int32_t J = 0; J < ns; ++J) {
        if (S.is_tail[J]) continue;
        const int64_t w = S.sn_col[J + 1] - S.sn_col[J];
        const int64_t r = S.sn_rptr[J + 1] - S.sn_rptr[J];
        const int64_t inbox = S.irow_ptr[S.sn_rptr[J + 1]] - S.irow_ptr[S.sn_rptr[J]];
        if (w * r >= opt.mid_panel || inbox >= 2 * (int64_t)opt.mid_panel) S.is_mid[J] = 1;
    }
    for (int32_t J = 0; J < ns; ++J)
        if (S.is_mid[J] && S.sn_parent[J] >= 0 && !S.is_tail[S.sn_parent[J]]) S.is_mid[S.sn_parent[J]] = 1;
    auto tier = [&](int32_t J) { return S.is_tail[J] ? 2 : (S.is_mid[J] ? 1 : 0); };
    S.order.resize(ns);
    std::iota(S.order.begin(), S.order.end(), 0);
    std::stable_sort(S.order.begin(), S.order.end(), [&](int32_t a, int32_t b) {
        if (tier(a) != tier(b)) return tier(a) < tier(b);
        return S.level[a] < S.level[b];
    });
    S.n_main = 0;
    S.n_warp = 0;
    for (int32_t J = 0; J < ns; ++J) {
        S.n_main += S.is_tail[J] ? 0 : 1;
        S.n_warp += tier(J) == 0 ? 1 : 0;
    }
    S.max_panel_warp = 0;
    for (int32_t J = 0; J < ns; ++J)
        if (tier(J) == 0)
            S.max_panel_warp = std::max<int64_t>(S.max_panel_warp,
                                                 (S.sn_col[J + 1] - S.sn_col[J]) * (S.sn_rptr[J + 1] - S.sn_rptr[J]));
    S.max_panel_main = 0;
    for (int32_t J = 0; J < ns; ++J)
        if (!S.is_tail[J])
            S.max_panel_main = std::max<int64_t>(S.max_panel_main,
                                                 (S.sn_col[J + 1] - S.sn_col[J]) * (S.sn_rptr[J + 1] - S.sn_rptr[J]));

    T.mark("levels + tiers");
    // scatter maps: K(i,j) (original indices) -> panel position
    auto pos = [&](int64_t i, int64_t j) -> int64_t {
        int32_t a = iperm[i], b = iperm[j];
        int32_t row = std::max(a, b), col = std::min(a, b);
        int32_t J = S.col2sn[col];
        const int32_t* rows = S.sn_rows.data() + S.sn_rptr[J];
        int64_t r = S.sn_rptr[J + 1] - S.sn_rptr[J];
        int64_t lr = std::lower_bound(rows, rows + r, row) - rows;
        return S.sn_loff[J] + (int64_t)(col - S.sn_col[J]) * r + lr;
    };
    S.map_p.assign(prp[n], -1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = prp[i]; p < prp[i + 1]; ++p)
            if (pci[p] >= i) S.map_p[p] = pos(i, pci[p]);
    S.map_a.assign(arp[m], 0);
    for (int64_t r = 0; r < m; ++r)
        for (int64_t p = arp[r]; p < arp[r + 1]; ++p) S.map_a[p] = pos(aci[p], n + r);
    S.map_diag.assign(dim, 0);
    for (int64_t i = 0; i < dim; ++i) S.map_diag[i] = pos(i, i);
    S.map_hblk.clear();
    for (int64_t b = 0; b < nblocks; ++b)
        for (int64_t rl = 0; rl < bdim[b]; ++rl)
            for (int64_t cl = rl; cl < bdim[b]; ++cl)
                S.map_hblk.push_back(pos(n + boff[b] + rl, n + boff[b] + cl));
    T.mark("scatter maps");
    // continuation scheduling (ldl.cu): per-supernode descriptors, same-tier child
    // counts, start lists (supernodes without same-tier children), inbox column ids
    {
        const int32_t BIG = 0x3fffffff;
        S.tier.assign(ns, 0);
        for (int32_t J = 0; J < ns; ++J) S.tier[J] = S.is_tail[J] ? 2 : (S.is_mid[J] ? 1 : 0);
        // tiny leaves (no children, w <= 4, r <= 16): one thread each, in separate
        // launches before (factor, forward) / after (backward) the persistent kernels,
        // so they are excluded from the continuation child counts
        std::vector<char> tiny(ns, 0);
        S.tiny.clear();
        for (int32_t J = 0; J < ns; ++J) {
            const int64_t w = S.sn_col[J + 1] - S.sn_col[J], r = S.sn_rptr[J + 1] - S.sn_rptr[J];
            if (S.tier[J] == 0 && S.sn_nchild[J] == 0 && w <= 4 && r <= 16) {
                tiny[J] = 1;
                S.tiny.push_back(J);
            }
        }
        // vector inbox re-laid per target supernode: tiny sources first, then the rest
        {
            std::vector<int64_t> tc(dim, 0), nc(dim, 0);
            for (int32_t K = 0; K < ns; ++K) {
                const int64_t w = S.sn_col[K + 1] - S.sn_col[K];
                for (int64_t p = S.sn_rptr[K] + w; p < S.sn_rptr[K + 1]; ++p) (tiny[K] ? tc : nc)[S.sn_rows[p]]++;
            }
            S.vt_lo.assign(dim, 0);
            S.vt_hi.assign(dim, 0);
            S.vn_lo.assign(dim, 0);
            S.vn_hi.assign(dim, 0);
            S.tfold_cols.clear();
            for (int32_t J = 0; J < ns; ++J) {
                const int64_t c0 = S.sn_col[J], c1 = S.sn_col[J + 1];
                int64_t t = S.vcol_ptr[c0], tot_t = 0;
                for (int64_t j = c0; j < c1; ++j) tot_t += tc[j];
                int64_t u = S.vcol_ptr[c0] + tot_t;
                for (int64_t j = c0; j < c1; ++j) {
                    S.vt_lo[j] = t;
                    t += tc[j];
                    S.vt_hi[j] = t;
                    S.vn_lo[j] = u;
                    u += nc[j];
                    S.vn_hi[j] = u;
                    if (tc[j] > 0) S.tfold_cols.push_back((int32_t)j);
                }
            }
            std::vector<int64_t> tf(S.vt_lo), nf(S.vn_lo);
            for (int32_t K = 0; K < ns; ++K) {
                const int64_t w = S.sn_col[K + 1] - S.sn_col[K];
                int64_t a = 0;
                for (int64_t p = S.sn_rptr[K] + w; p < S.sn_rptr[K + 1]; ++p, ++a) {
                    const int32_t j = S.sn_rows[p];
                    S.vpush_pos[S.cv_off[K] + a] = tiny[K] ? tf[j]++ : nf[j]++;
                }
            }
        }
        std::vector<int32_t> need_fac(ns, 0), need_solve(ns, 0);
        for (int32_t J = 0; J < ns; ++J) {
            const int32_t P = S.sn_parent[J];
            if (P < 0 || tiny[J]) continue;
            if (S.tier[P] != 2) need_solve[P]++;
            if (S.tier[P] == S.tier[J] && S.tier[P] != 2) need_fac[P]++;
        }
        S.desc32.assign((size_t)ns * 8, 0);
        S.desc64.assign((size_t)ns * 8, 0);
        for (int32_t J = 0; J < ns; ++J) {
            int32_t* d = &S.desc32[(size_t)J * 8];
            d[0] = S.sn_col[J];
            d[1] = S.sn_col[J + 1] - S.sn_col[J];
            d[2] = (int32_t)(S.sn_rptr[J + 1] - S.sn_rptr[J]);
            d[3] = S.sn_parent[J];
            d[4] = S.tier[J] == 2 ? BIG : need_solve[J];
            d[5] = S.tier[J] == 2 ? BIG : need_fac[J];
            d[6] = S.tier[J];
            int64_t* e = &S.desc64[(size_t)J * 8];
            e[0] = S.sn_loff[J];
            e[1] = S.cv_off[J];
            e[2] = S.vn_lo[S.sn_col[J]];            // non-tiny part of the vector inbox
            e[3] = S.vcol_ptr[S.sn_col[J + 1]];
            e[4] = S.irow_ptr[S.sn_rptr[J]];
            e[5] = S.irow_ptr[S.sn_rptr[J + 1]];
            e[6] = S.cb_off[J];
            e[7] = S.sn_rptr[J];
        }
        S.need.assign((size_t)ns * 2, 0);
        for (int32_t J = 0; J < ns; ++J) {
            S.need[2 * (size_t)J] = S.desc32[(size_t)J * 8 + 4];
            S.need[2 * (size_t)J + 1] = S.desc32[(size_t)J * 8 + 5];
        }
        S.start_solve.clear();
        S.start_fac_warp.clear();
        S.start_fac_cta.clear();
        for (int32_t J = 0; J < ns; ++J) {
            if (S.tier[J] == 2 || tiny[J]) continue;
            if (need_solve[J] == 0) S.start_solve.push_back(J);
            if (need_fac[J] == 0) (S.tier[J] == 0 ? S.start_fac_warp : S.start_fac_cta).push_back(J);
        }
        // backward sweep order: non-tail, non-tiny supernodes, topological (children first)
        S.bwd_order.clear();
        for (int32_t k = 0; k < S.n_main; ++k)
            if (!tiny[S.order[k]]) S.bwd_order.push_back(S.order[k]);
        S.vin_col.assign((size_t)S.vcol_ptr[dim], 0);
        for (int64_t j = 0; j < dim; ++j) {
            const int32_t J = S.col2sn[j];
            for (int64_t e = S.vt_lo[j]; e < S.vt_hi[j]; ++e) S.vin_col[e] = (uint8_t)(j - S.sn_col[J]);
            for (int64_t e = S.vn_lo[j]; e < S.vn_hi[j]; ++e) S.vin_col[e] = (uint8_t)(j - S.sn_col[J]);
        }
    }
    (void)lin;
    return 0;
}

}  // namespace cipm
