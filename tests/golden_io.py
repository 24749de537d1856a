"""Load golden fixtures (written by tests/golden/make_golden.py) into ProblemData."""
from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_2412_19027_b200.csr import CsrMatrix
from paper_2412_19027_b200.model import ConeSpec, ProblemData

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _csr(d):
    return CsrMatrix(d["nrows"], d["ncols"], np.array(d["rowptr"], dtype=np.int64),
                     np.array(d["colidx"], dtype=np.int64), np.array(d["values"]))


def cone_from_doc(c):
    return ConeSpec(c["kind"], c["dim"], c.get("alpha"), c.get("side"))


def problem_from_doc(doc) -> ProblemData:
    p = doc["problem"]
    return ProblemData(_csr(p["P"]), _csr(p["A"]), np.array(p["q"]), np.array(p["b"]),
                       [cone_from_doc(c) for c in p["cones"]])


def instance_names():
    return sorted(os.path.basename(f)[:-5] for f in glob.glob(os.path.join(GOLDEN, "instances", "*.json")))


def load_instance(name):
    with open(os.path.join(GOLDEN, "instances", name + ".json")) as f:
        return json.load(f)


def load_kernels():
    with open(os.path.join(GOLDEN, "kernels.json")) as f:
        return json.load(f)
