"""GPU probe: host-side time split of the public-API path (update_data + solve)
for one config, with cProfile's top entries.

    python tools/e2e_probe.py c2_lasso
"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_lasso"
    prob = G.build(cfg)
    s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"]))
    s.solve()
    q, b = np.ascontiguousarray(prob.q), np.ascontiguousarray(prob.b)
    for _ in range(6):
        t0 = time.perf_counter()
        s.update_data(q=q, b=b)
        t1 = time.perf_counter()
        r = s.solve()
        t2 = time.perf_counter()
        print(f"update_data {1e3 * (t1 - t0):.2f} ms, solve {1e3 * (t2 - t1):.2f} ms, iterations {r.iterations}")
    pr = cProfile.Profile()
    pr.enable()
    s.update_data(q=q, b=b)
    s.solve()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)


if __name__ == "__main__":
    main()
