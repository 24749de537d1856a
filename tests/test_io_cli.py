"""JSON problem I/O, the benchmark families, metrics and the CLI (
reference io.py, generators.py, metrics.py, bench.py, cli.py), pinned against
fixtures the unmodified reference produced (tests/golden/families.json, written by
tests/golden/make_families.py)."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from golden_io import instance_names, load_instance, problem_from_doc
from paper_2412_19027_b200 import io as pio
from paper_2412_19027_b200.benchsuite import BenchRecord, metrics_from_records, records_from_csv, records_to_csv
from paper_2412_19027_b200.families import GenSpec
from paper_2412_19027_b200.metrics import normalized_geomeans, perf_profiles, shifted_geomean

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = json.load(open(os.path.join(ROOT, "tests", "golden", "families.json")))


def _cli(*args, check=None):
    r = subprocess.run([sys.executable, "-m", "paper_2412_19027_b200", *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=600)
    if check is not None:
        assert r.returncode == check, (r.returncode, r.stderr[-2000:])
    return r


@pytest.mark.parametrize("case", FIX["families"], ids=lambda c: c["name"])
def test_families_match_reference_instances(case):
    """Same seed, same draw order, same matrices: the canonical problem JSON hashes equal."""
    spec = GenSpec(family=case["family"], n=case["n"], seed=case["seed"], k=case["k"], periods=case["periods"])
    assert spec.name == case["name"]
    doc = pio.problem_to_dict(spec.build(), name=spec.name, seed=case["seed"])
    assert hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest() == case["sha256"]


@pytest.mark.parametrize("name", instance_names()[:12])
def test_json_round_trip_bitwise(name, tmp_path):
    prob = problem_from_doc(load_instance(name))
    path = tmp_path / "p.json"
    pio.write_problem(prob, path, name=name, seed=3)
    back, meta = pio.read_problem(path)
    assert meta == {"name": name, "seed": 3}
    for a, b in ((prob.P, back.P), (prob.A, back.A)):
        np.testing.assert_array_equal(a.rowptr, b.rowptr)
        np.testing.assert_array_equal(a.colidx, b.colidx)
        assert a.values.tobytes() == b.values.tobytes()
    assert prob.q.tobytes() == back.q.tobytes() and prob.b.tobytes() == back.b.tobytes()
    assert [(c.kind, c.dim, c.alpha, c.side) for c in prob.cones] == \
        [(c.kind, c.dim, c.alpha, c.side) for c in back.cones]


def test_json_validation_errors(tmp_path):
    from paper_2412_19027_b200.exceptions import ValidationError
    bad = tmp_path / "bad.json"
    bad.write_text('{"n": 1')
    with pytest.raises(ValidationError, match="invalid JSON"):
        pio.read_problem(bad)
    with pytest.raises(ValidationError, match="power cone needs 'alpha'"):
        pio.problem_from_dict({"n": 1, "m": 3, "q": [0.0], "b": [0.0, 0.0, 0.0],
                               "P": {"rowptr": [0, 0], "colidx": [], "values": []},
                               "A": {"rowptr": [0, 1, 2, 3], "colidx": [0, 0, 0], "values": [1.0, 1.0, 1.0]},
                               "cones": [{"type": "pow", "dim": 3}]})
    with pytest.raises(ValidationError, match="unknown cone type"):
        pio.problem_from_dict({"n": 0, "m": 0, "q": [], "b": [], "P": {"rowptr": [0], "colidx": [], "values": []},
                               "A": {"rowptr": [0], "colidx": [], "values": []},
                               "cones": [{"type": "cube", "dim": 1}]})


def test_metrics_match_reference():
    recs = records_from_csv(FIX["metrics"]["csv"])
    assert records_to_csv(recs) == FIX["metrics"]["csv"]
    got = json.loads(json.dumps(metrics_from_records(recs)))
    want = FIX["metrics"]["metrics"]
    assert got.keys() == want.keys()
    assert got["geomean"] == pytest.approx(want["geomean"], rel=1e-15)
    assert got["normalized"] == pytest.approx(want["normalized"], rel=1e-15)
    assert got["relative_profile"]["tau"] == pytest.approx(want["relative_profile"]["tau"], rel=1e-15)
    assert got["relative_profile"]["fraction"] == want["relative_profile"]["fraction"]
    assert got["absolute_profile"]["fraction"] == want["absolute_profile"]["fraction"]


def test_metrics_known_values():
    assert shifted_geomean([1.0, 3.0]) == pytest.approx(np.sqrt(2.0 * 4.0) - 1.0)
    times = {("a", "x"): 1.0, ("a", "y"): 2.0, ("b", "x"): 4.0, ("b", "y"): 2.0}
    prof = perf_profiles(times)
    assert prof.ratios[("a", "y")] == 2.0 and prof.ratios[("b", "x")] == 2.0
    assert prof.rel["x"][0] == 0.5 and prof.rel["x"][-1] == 1.0
    g = normalized_geomeans(times)
    assert min(g["normalized"].values()) == 1.0
    with pytest.raises(ValueError):
        shifted_geomean([])


def test_cli_gen_and_errors(tmp_path):
    out = tmp_path / "e.json"
    r = _cli("gen", "--family", "entropy", "--n", "6", "--seed", "1", "--out", str(out), check=0)
    assert json.loads(r.stdout)["name"] == "entropy_n6_s1"
    prob, meta = pio.read_problem(out)
    assert meta["name"] == "entropy_n6_s1" and prob.n == 12
    bad = tmp_path / "bad.json"
    bad.write_text("[1, 2]")
    assert _cli("solve", str(bad)).returncode == 2
    assert _cli("bench", "--families", "nope").returncode == 2
    csv_path = tmp_path / "r.csv"
    csv_path.write_text(FIX["metrics"]["csv"])
    r = _cli("metrics", "--csv", str(csv_path), check=0)
    assert json.loads(r.stdout)["geomean"] == pytest.approx(FIX["metrics"]["metrics"]["geomean"], rel=1e-15)


@pytest.mark.gpu
def test_gpu_cli_solve_golden(gpu, tmp_path):
    """`solve` on a problem file: status and objective of the reference's result, exit 0."""
    doc = load_instance("socp_40")
    path = tmp_path / "p.json"
    pio.write_problem(problem_from_doc(doc), path)
    r = _cli("solve", str(path), "--eps-feas", str(doc["settings"]["eps_feas"]), check=0)
    res = json.loads(r.stdout)
    assert res["status"] == doc["result"]["status"]
    assert abs(res["obj_primal"] - doc["result"]["obj_primal"]) <= 1e-6 * max(1.0, abs(doc["result"]["obj_primal"]))


@pytest.mark.gpu
def test_gpu_cli_bench_virtual_clock(gpu, tmp_path):
    """`bench` with the virtual clock: the CSV is bit-reproducible run to run (SPEC AC10)
    and every record matches the reference suite's status and iterations (±1)."""
    s = FIX["suite"]
    args = ["bench", "--families", ",".join(s["families"]), "--sizes", ",".join(map(str, s["sizes"])),
            "--seeds", ",".join(map(str, s["seeds"])), "--clock", "virtual"]
    a = _cli(*args, check=0).stdout
    b = _cli(*args, check=0).stdout
    assert a == b
    got, want = records_from_csv(a), records_from_csv(s["csv"])
    assert [r.problem for r in got] == [r.problem for r in want]
    for g, w in zip(got, want):
        assert g.status == w.status, (g.problem, g.status, w.status)
        assert abs(g.iterations - w.iterations) <= 1, (g.problem, g.iterations, w.iterations)
