"""Solve one config with verbose output and per-iteration refinement steps."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_socp"
scale = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
prob = G.build(cfg, **scale)
s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"], verbose=True))
r = s.solve()
print(cfg, r.status, r.iterations, r.obj_primal, "refine steps", s.last_refine_steps)
s.close()
