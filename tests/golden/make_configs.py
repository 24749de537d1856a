"""Config-shape golden results from the UNMODIFIED reference solver.

The BASELINE configs at full size (C1, C2, C3, C5a) and reduced scale (C2,
C3, C5a at 1/10; C4 at 1/5 -- its full size takes the reference's Python setup
hours): status, iterations, objectives and
final residual norms of ``conic_ipm.solve`` on the same seeded generator
instances the bench uses.  Run in the build container (``/root/reference`` is
not on the GPU box):

    python tests/golden/make_configs.py          # writes tests/golden/configs.json

Each case runs in its own process (numba/threads pinned to one core).
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

# name -> (generator, kwargs, precision); C4 at 1/5 scale is the survey's probe size
CASES = {
    "c1_lp_full": ("lp", dict(n=2000, m=4000), "full"),
    "c2_lasso_tenth": ("lasso", dict(nf=5_000, mr=20_000), "mixed"),
    "c3_socp_tenth": ("socp", dict(ncones=10_000), "full"),
    "c4_exppow_fifth": ("exppow", dict(n_exp=10_000, n_pow=4_000), "full"),
    "c5a_psd_tenth": ("psd", dict(ncones=1_000, side=6), "full"),
    # the BASELINE sizes themselves (reference setup + solve: minutes each); C4 at
    # full size is not here: the reference's pure-Python minimum degree on its
    # 415k-row KKT pattern runs for hours
    "c2_lasso_full": ("lasso", dict(nf=50_000, mr=200_000), "mixed"),
    "c3_socp_full": ("socp", dict(ncones=100_000), "full"),
    "c5a_psd_full": ("psd", dict(ncones=10_000, side=6), "full"),
}


def run(name):
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[k] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, REPO)
    import conic_ipm as ref
    from paper_2412_19027_b200 import generators as G
    from bench import _to_reference
    gen, kw, prec = CASES[name]
    p = G.GENERATORS[gen](seed=0, **kw)
    r = ref.solve(_to_reference(ref, p), ref.SolverSettings(eps_feas=1e-8, precision=prec))
    return name, dict(gen=gen, kwargs=kw, precision=prec, eps_feas=1e-8, status=str(r.status.value
                      if hasattr(r.status, "value") else r.status), iterations=int(r.iterations),
                      obj_primal=float(r.obj_primal), obj_dual=float(r.obj_dual), norm_rp=float(r.norm_rp),
                      norm_rd=float(r.norm_rd), gap=float(r.gap), setup_seconds=float(r.setup_seconds),
                      solve_seconds=float(r.solve_seconds))


def main():
    names = sys.argv[1:] or list(CASES)
    out_path = os.path.join(HERE, "configs.json")
    doc = json.load(open(out_path)) if os.path.exists(out_path) else {}
    with mp.get_context("spawn").Pool(len(names)) as pool:
        for name, res in pool.imap_unordered(run, names):
            doc[name] = res
            print(name, res["status"], res["iterations"], res["obj_primal"], flush=True)
            json.dump(doc, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
