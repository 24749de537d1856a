"""Per-instance golden results of the C5b batch (2048 MPC QPs, seeds 0..2047)
from the UNMODIFIED reference solver.

Run in the build container (``/root/reference`` is not on the GPU box):

    python tests/golden/make_mpc.py            # writes tests/golden/mpc2048.json

Each worker process solves a contiguous slice of the seeds with
``conic_ipm.solve`` (one core each, the reference's ``bench --jobs`` mode,
``bench.py:98-113``) and records status, iterations and both objectives.
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
N = 2048


def run(rng):
    lo, hi = rng
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[k] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, REPO)
    import conic_ipm as ref
    from paper_2412_19027_b200 import generators as G
    from bench import _to_reference
    out = []
    st = ref.SolverSettings(eps_feas=1e-8)
    for seed in range(lo, hi):
        r = ref.solve(_to_reference(ref, G.gen_mpc(seed=seed)), st)
        out.append((seed, str(r.status.value if hasattr(r.status, "value") else r.status), int(r.iterations),
                    float(r.obj_primal), float(r.obj_dual)))
    return out


def main():
    jobs = os.cpu_count() or 1
    step = (N + jobs - 1) // jobs
    ranges = [(lo, min(N, lo + step)) for lo in range(0, N, step)]
    rows = []
    with mp.get_context("spawn").Pool(len(ranges)) as pool:
        for part in pool.imap_unordered(run, ranges):
            rows.extend(part)
    rows.sort()
    doc = dict(config="c5b_mpc", generator="gen_mpc(seed=k)", eps_feas=1e-8, precision="full",
               status=[r[1] for r in rows], iterations=[r[2] for r in rows],
               obj_primal=[r[3] for r in rows], obj_dual=[r[4] for r in rows])
    json.dump(doc, open(os.path.join(HERE, "mpc2048.json"), "w"))
    print("instances", len(rows), "statuses", sorted(set(doc["status"])), "iterations", sum(doc["iterations"]))


if __name__ == "__main__":
    main()
