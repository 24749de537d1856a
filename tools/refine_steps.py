"""Refinement steps per refined solve (affine incl. col2, combined), per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402

for cfg in sys.argv[1:] or ["c1_lp", "c2_lasso", "c3_socp", "c5a_psd"]:
    s = Solver(G.build(cfg), SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"]))
    s.last_refine_steps = []
    r = s.solve()
    st = s.last_refine_steps
    print(cfg, r.status, r.iterations, "affine", [a for a, _ in st], "combined", [b for _, b in st],
          "ordering", s.symbolic.info()["ordering"], flush=True)
    s.close()
