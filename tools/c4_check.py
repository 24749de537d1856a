"""C4 (exp + pow cones) on the GPU: reduced scale vs the oracle numbers, then full scale."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402

scale = sys.argv[1] if len(sys.argv) > 1 else "fifth"
ne, npw = (10_000, 4_000) if scale == "fifth" else (50_000, 20_000)
prob = G.gen_exppow(ne, npw, seed=0)
t0 = time.perf_counter()
s = Solver(prob, SolverSettings(eps_feas=1e-8))
setup = time.perf_counter() - t0
info = s.symbolic.info()
t1 = time.perf_counter()
r = s.solve()
solve = time.perf_counter() - t1
r2 = s.solve()
print(json.dumps(dict(scale=scale, status=r.status, it=r.iterations, gp=r.obj_primal, gd=r.obj_dual, setup=setup,
                      solve=solve, solve2=r2.solve_seconds, info=info)))
