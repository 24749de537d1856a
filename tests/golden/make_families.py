"""Golden fixtures for the CLI families, JSON I/O and metrics, from the UNMODIFIED
reference (run in the build container: python tests/golden/make_families.py).

* families: sha256 of the reference's canonical problem JSON (io.problem_to_dict)
  for small instances of every family -> our families.py must reproduce them;
* metrics: the reference's metrics_from_records on a seeded random record table;
* suite: the reference's `bench` records (virtual clock) for a small suite.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from conic_ipm import bench as rb  # noqa: E402
from conic_ipm import io as rio  # noqa: E402
from conic_ipm.generators import GenSpec  # noqa: E402

SPECS = [("portfolio", 12, 0, 0, 0), ("portfolio", 30, 3, 0, 0), ("huber", 8, 0, 0, 0), ("huber", 15, 2, 0, 0),
         ("entropy", 6, 0, 0, 0), ("entropy", 16, 1, 0, 0), ("multistage", 24, 1, 2, 2),
         ("multistage", 30, 0, 3, 3)]


def main():
    fam = []
    for family, n, seed, k, periods in SPECS:
        spec = GenSpec(family=family, n=n, seed=seed, k=k, periods=periods)
        doc = rio.problem_to_dict(spec.build(), name=spec.name, seed=seed)
        text = json.dumps(doc, sort_keys=True)
        fam.append({"family": family, "n": n, "seed": seed, "k": k, "periods": periods, "name": spec.name,
                    "sha256": hashlib.sha256(text.encode()).hexdigest()})
    rng = np.random.default_rng(7)
    recs = []
    for p in range(9):
        for cfg in ("full", "mixed", "other"):
            t = float(rng.uniform(0.0, 5.0)) if rng.random() > 0.1 else 0.0
            recs.append(rb.BenchRecord(problem=f"p{p}", config=cfg, status="optimal", total_seconds=t,
                                       setup_seconds=0.0, solve_seconds=t, iterations=int(rng.integers(5, 30)),
                                       norm_rp=1e-9, norm_rd=1e-9, gap=1e-9))
    metrics = {"csv": rb.records_to_csv(recs), "metrics": rb.metrics_from_records(recs)}
    specs = [GenSpec(family=f, n=n, seed=s) for f in ("portfolio", "huber", "entropy") for n in (6, 10) for s in (0, 1)]
    records = rb.run_suite(specs, [rb.BUILTIN_CONFIGS["full"]], time_limit=60.0, clock=rb.VIRTUAL)
    suite = {"families": ["portfolio", "huber", "entropy"], "sizes": [6, 10], "seeds": [0, 1],
             "csv": rb.records_to_csv(records)}
    json.dump({"families": fam, "metrics": metrics, "suite": suite}, open(os.path.join(HERE, "families.json"), "w"),
              indent=1)
    print("wrote families.json:", len(fam), "instances,", len(records), "suite records")


if __name__ == "__main__":
    main()
