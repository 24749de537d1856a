"""CPU tests of the native boundary: the library loads, exports every symbol of
include/cipm.h, and the host symbolic analysis is correct (no GPU needed)."""
import os
import re

import numpy as np
import pytest

from golden_io import instance_names, load_instance, problem_from_doc
import supernodal_model as SM
from oracle import OracleSolver
from oracle import cones as C
from paper_2412_19027_b200 import model, native
from paper_2412_19027_b200.settings import SolverSettings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "cipm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void)\s+(cipm_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = native.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(native.exported_symbols())
    assert L.cipm_version() >= 100


def _scaled(name):
    prob = problem_from_doc(load_instance(name))
    r, _ = model.reorder_cones(prob)
    s, _ = model.equilibrate(r)
    return prob, s


@pytest.mark.parametrize("name", [n for n in instance_names() if not n.startswith("dual_inf")])
def test_min_degree_matches_reference_order(name):
    prob, s = _scaled(name)
    sym = native.SymbolicAnalysis(s.P, s.A, native.Layout(s.cones))
    o = OracleSolver(prob, SolverSettings())
    np.testing.assert_array_equal(sym.array("md_perm"), o.kkt.perm)
    assert sym.info()["nnz_l"] == o.kkt.nnz_l


@pytest.mark.parametrize("ordering", [0, 2])
@pytest.mark.parametrize("name", ["lp_20x40", "socp_10", "psd_4x3", "exppow_20_8", "mpc_s0", "lasso_40x160"])
def test_supernodal_structure_reconstructs_kkt(name, ordering):
    _, s = _scaled(name)
    lay = native.Layout(s.cones)
    sym = native.SymbolicAnalysis(s.P, s.A, lay, ordering=ordering, nd_leaf=8)
    olay = C.ConeLayout.from_specs(s.cones)
    s0, z0 = C.unit_start(olay)
    sc = C.update_scaling(olay, s0, z0, 1.0)
    diag, blocks = sc.kkt_blocks()
    rng = np.random.default_rng(0)
    diag = diag.copy()
    diag[lay.zero_dim:] *= rng.uniform(0.1, 10, lay.nonneg_dim)
    hb = np.concatenate([b[np.triu_indices(b.shape[0])] for _, b in blocks]) if blocks else np.zeros(0)
    n = s.n
    reg = 1e-3
    vals = SM.assemble(sym, n, s.P, s.A, diag, hb, reg)
    perm = sym.array("perm")
    dim = len(perm)
    L, D = SM.factor(sym, vals, np.where(perm < n, 1, -1), 1e-14)
    L2, D2 = SM.factor_inbox(sym, vals, np.where(perm < n, 1, -1), 1e-14)
    assert np.allclose(L, L2, rtol=1e-9, atol=1e-12) and np.allclose(D, D2, rtol=1e-9, atol=1e-12)
    Ld = SM.dense_factor(sym, L2, D2)
    K = np.zeros((dim, dim))
    K[:n, :n] = s.P.toarray()
    A = s.A.toarray()
    K[n:, :n] = A
    K[:n, n:] = A.T
    H = sc.dense().copy()
    H[np.arange(len(diag)), np.arange(len(diag))] = diag
    K[n:, n:] = -H
    K += np.diag(np.where(np.arange(dim) < n, reg, -reg))
    Kp = K[np.ix_(perm, perm)]
    assert np.abs(Ld @ np.diag(D) @ Ld.T - Kp).max() < 1e-10 * max(1.0, np.abs(Kp).max())


def test_symbolic_invariants():
    _, s = _scaled("lp_150x300")
    sym = native.SymbolicAnalysis(s.P, s.A, native.Layout(s.cones))
    col, rptr, rows = sym.array("sn_col"), sym.array("sn_rptr"), sym.array("sn_rows")
    par = sym.array("sn_parent")
    order = sym.array("order")
    ns = len(col) - 1
    pos = np.empty(ns, dtype=np.int64)
    pos[order] = np.arange(ns)
    for J in range(ns):
        w = col[J + 1] - col[J]
        rj = rows[rptr[J]:rptr[J + 1]]
        assert np.array_equal(rj[:w], np.arange(col[J], col[J + 1]))
        assert np.all(np.diff(rj) > 0)
        if par[J] >= 0:
            assert pos[par[J]] > pos[J]          # topological order
            assert col[par[J]] <= rj[w] < col[par[J] + 1]
    # every scatter position is unique
    mp = sym.array("map_p")
    allpos = np.concatenate([mp[mp >= 0], sym.array("map_a"), sym.array("map_diag"), sym.array("map_hblk")])
    # P diagonal and map_diag coincide for x rows; everything else is unique
    assert len(np.unique(np.concatenate([sym.array("map_a"), sym.array("map_diag")]))) == \
        len(sym.array("map_a")) + len(sym.array("map_diag"))
    assert allpos.max() < sym.info()["nnz_storage"]


def test_min_degree_entry_point_on_arrow():
    # 5x5 arrow (dense last row/col): MD eliminates the leaves first, spike last (SPEC kkt-solver example)
    import scipy.sparse as sp
    a = np.eye(5)
    a[4, :] = 1
    a[:, 4] = 1
    m = sp.csr_matrix(a)
    perm = native.min_degree(m.indptr, m.indices)
    assert perm[-1] == 4 or perm[-2] == 4


def test_nested_dissection_is_a_shallow_permutation():
    """ND (ordering 2) is a permutation; on a banded SOCP it keeps MD's fill within
    the auto rule's bounds and cuts the supernodal tree height; auto picks it."""
    from paper_2412_19027_b200 import generators as G
    prob = G.gen_socp(3000, seed=0)
    r, _ = model.reorder_cones(prob)
    lay = native.Layout(r.cones)
    md = native.SymbolicAnalysis(r.P, r.A, lay, ordering=0)
    nd = native.SymbolicAnalysis(r.P, r.A, lay, ordering=2)
    auto = native.SymbolicAnalysis(r.P, r.A, lay, ordering=3)
    dim = r.n + r.m
    assert np.array_equal(np.sort(nd.array("md_perm")), np.arange(dim))
    imd, ind = md.info(), nd.info()
    assert ind["ordering"] == 2 and imd["ordering"] == 0
    assert ind["nnz_l"] <= 1.25 * imd["nnz_l"]
    assert ind["height"] < imd["height"]
    assert auto.info()["ordering"] == 2
    assert np.array_equal(auto.array("perm"), nd.array("perm"))


def test_auto_ordering_keeps_reference_md_when_small_or_fill_heavy():
    prob, s = _scaled("lp_150x300")
    sym = native.SymbolicAnalysis(s.P, s.A, native.Layout(s.cones), ordering=3)
    assert sym.info()["ordering"] == 0
    o = OracleSolver(prob, SolverSettings())
    np.testing.assert_array_equal(sym.array("md_perm"), o.kkt.perm)


@pytest.mark.parametrize("name", ["lasso_40x160", "lp_150x300", "socp_10", "mpc_s0"])
def test_vector_inbox_tiny_first_layout(name):
    """Each supernode's vector inbox holds the tiny leaves' entries first, then the
    rest, both grouped by column; every push position is used exactly once and a
    tiny source lands in its column's tiny range (the fold pass sums exactly those)."""
    _, s = _scaled(name)
    sym = native.SymbolicAnalysis(s.P, s.A, native.Layout(s.cones))
    col, rptr, rows = sym.array("sn_col"), sym.array("sn_rptr"), sym.array("sn_rows")
    vcp, cvo, vpp = sym.array("vcol_ptr"), sym.array("cv_off"), sym.array("vpush_pos")
    tlo, thi, nlo, nhi = (sym.array(k) for k in ("vt_lo", "vt_hi", "vn_lo", "vn_hi"))
    tiny = set(sym.array("tiny").tolist())
    ns = len(col) - 1
    assert np.array_equal(np.sort(vpp), np.arange(vcp[-1]))          # a permutation of the inbox slots
    for J in range(ns):
        c0, c1 = col[J], col[J + 1]
        lo, hi = vcp[c0], vcp[c1]
        t_tot = int(np.sum(thi[c0:c1] - tlo[c0:c1]))
        assert tlo[c0] == lo and nlo[c0] == lo + t_tot and nhi[c1 - 1] == hi
        assert np.all(tlo[c0 + 1:c1] == thi[c0:c1 - 1]) and np.all(nlo[c0 + 1:c1] == nhi[c0:c1 - 1])
    fold = set(sym.array("tfold_cols").tolist())
    assert fold == {j for j in range(len(tlo)) if thi[j] > tlo[j]}
    for K in range(ns):
        w = col[K + 1] - col[K]
        for a, p in enumerate(range(rptr[K] + w, rptr[K + 1])):
            j, pos = rows[p], vpp[cvo[K] + a]
            if K in tiny:
                assert tlo[j] <= pos < thi[j]
            else:
                assert nlo[j] <= pos < nhi[j]


def test_amd_ordering_valid_and_competitive():
    """Ordering 4 (quotient-graph approximate minimum degree, the fallback of the exact
    order on large systems): a permutation of the KKT rows whose fill stays within 10 %
    of the reference's exact minimum degree on a generator instance."""
    from paper_2412_19027_b200 import generators as G
    from paper_2412_19027_b200.model import reorder_cones
    from paper_2412_19027_b200.native import Layout, SymbolicAnalysis
    for prob in (G.gen_socp(300, seed=2), G.gen_lp(150, 300, seed=4), G.gen_exppow(200, 80, seed=1)):
        r, _ = reorder_cones(prob)
        lay = Layout(r.cones)
        amd = SymbolicAnalysis(r.P, r.A, lay, ordering=4)
        md = SymbolicAnalysis(r.P, r.A, lay, ordering=0)
        perm = amd.array("md_perm")
        assert sorted(perm.tolist()) == list(range(r.n + r.m))
        assert amd.info()["ordering"] == 4
        assert amd.info()["nnz_l"] <= 1.10 * md.info()["nnz_l"], (amd.info()["nnz_l"], md.info()["nnz_l"])
        amd.close()
        md.close()
