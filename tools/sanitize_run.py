"""Small solves for compute-sanitizer (memcheck / initcheck / racecheck):

    compute-sanitizer --tool initcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
cases = {
    "lp_tail": (G.gen_lp(200, 400, seed=1), "full"),
    "lp_tail_mixed": (G.gen_lp(200, 400, seed=1), "mixed"),
    "socp": (G.gen_socp(60, seed=1), "full"),
    "psd": (G.gen_psd(40, side=4, seed=1), "full"),
    "exppow": (G.gen_exppow(60, 20, seed=1), "full"),
    "lasso_nd": (G.gen_lasso(200, 800, seed=1), "mixed"),
    "psd_side20": (G.gen_psd(2, side=20, seed=1), "full"),
}
if which in ("all", "batch"):
    from paper_2412_19027_b200.batch import BatchSolver
    bs = BatchSolver(G.build_instances("c5b_mpc", 0, 4), SolverSettings(eps_feas=1e-8))
    out = bs.solve()
    bs.close()
    print("batch", [r.status for r in out], [r.iterations for r in out], flush=True)
for name, (prob, prec) in cases.items():
    if which != "all" and which != name:
        continue
    s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=prec))
    r = s.solve()
    s.close()
    print(name, r.status, r.iterations, flush=True)
