"""GPU probe: host-side time split of the batched public-API path (C5b):
update_data, the device run, the result copy, and building every SolveResult.

    python tools/batch_e2e_probe.py [count]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.batch import BatchSolver  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    probs = G.build_instances("c5b_mpc", 0, count)
    bs = BatchSolver(probs, SolverSettings(eps_feas=1e-8))
    bs.solve()
    q, b = np.stack([p.q for p in probs]), np.stack([p.b for p in probs])
    for _ in range(6):
        t0 = time.perf_counter()
        bs.update_data(q=q, b=b)
        t1 = time.perf_counter()
        bs.run()
        t2 = time.perf_counter()
        out = bs.results()
        t3 = time.perf_counter()
        objs = list(out)
        t4 = time.perf_counter()
        print(f"update_data {1e3 * (t1 - t0):.2f} ms, run {1e3 * (t2 - t1):.2f} ms (kernel {bs.last_kernel_ms:.2f}),"
              f" results {1e3 * (t3 - t2):.2f} ms, build {len(objs)} SolveResult {1e3 * (t4 - t3):.2f} ms,"
              f" iterations {int(out.iterations.sum())}")
    bs.close()


if __name__ == "__main__":
    main()
