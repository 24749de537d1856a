"""CPU-only: tier / panel statistics of a config's supernodal symbolic analysis.

    python tools/sym_stats.py c2_lasso
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.model import reorder_cones  # noqa: E402
from paper_2412_19027_b200.native import Layout, SymbolicAnalysis  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_lasso"
    prob = G.build(cfg)
    rp, _ = reorder_cones(prob)
    sym = SymbolicAnalysis(rp.P, rp.A, Layout(rp.cones), ordering=int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    info = sym.info()
    col = sym.array("sn_col")
    rptr = sym.array("sn_rptr")
    tier = sym.array("tier")
    lvl = sym.array("level")
    tiny = sym.array("tiny")
    w = np.diff(col)
    r = np.diff(rptr)
    print(cfg, {k: info[k] for k in info})
    istiny = np.zeros(len(w), bool)
    istiny[tiny] = True
    for t, name in ((0, "warp"), (1, "cta"), (2, "tail")):
        sel = (tier == t) & ~istiny
        if not sel.any():
            continue
        fl = (w[sel] * (r[sel] - w[sel]) ** 2).sum() + (w[sel] ** 2 * r[sel]).sum()
        print(f"{name:5s} n={sel.sum():7d} w max {w[sel].max():5d} mean {w[sel].mean():7.1f}  r max {r[sel].max():5d} "
              f"mean {r[sel].mean():7.1f} panel max {(w[sel]*r[sel]).max():8d}  ~flops {fl:.3g}  levels "
              f"{lvl[sel].min()}..{lvl[sel].max()}")
    print(f"tiny  n={istiny.sum()}")
    tl = np.where(tier == 2)[0]
    for J in tl[:20]:
        print("  tail", J, "w", w[J], "r", r[J], "level", lvl[J])
    ct = np.where((tier == 1))[0]
    order = np.argsort(-(w[ct] * r[ct]))
    for J in ct[order[:15]]:
        print("  cta", J, "w", w[J], "r", r[J], "level", lvl[J])


if __name__ == "__main__":
    main()
