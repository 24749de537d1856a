"""One warm solve of a config, for ncu captures:

    ncu --set full -k regex:forward_kernel -s 4 -c 1 -o gpurun_out/prof python tools/profile_run.py c2_lasso
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_lasso"
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = G.build(cfg)
s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"]))
for _ in range(solves):
    r = s.solve()
print(cfg, r.status, r.iterations, r.solve_seconds)
s.close()
