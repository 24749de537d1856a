"""Re-solve a config-shape case several times (fresh Solver each) and report
status / iterations / objective bits: flags nondeterminism."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402

DOC = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                  "configs.json")))
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ordering = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ref = DOC[name]
prob = G.GENERATORS[ref["gen"]](seed=0, **ref["kwargs"])
for k in range(reps):
    s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=ref["precision"]), ordering=ordering)
    r1 = s.solve()
    r2 = s.solve()
    import hashlib
    hp = hashlib.md5(s.symbolic.array("perm").tobytes()).hexdigest()[:8]
    he = hashlib.md5(s._equil.d_row.tobytes() + s._equil.d_col.tobytes()).hexdigest()[:8] \
        if s._equil.d_row is not None else "?"
    print(name, k, r1.status, r1.iterations, r1.obj_primal.hex(), "| same solver again:", r2.status, r2.iterations,
          "perm", hp, "equil", he, flush=True)
    s.close()
