"""GPU probe: time the factorisation and triangular solves of one config at a
fixed iterate (after a few IPM iterations), with CUDA events per launch.

    python tools/solve_probe.py c2_lasso [iters]
"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.native import pdbl  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_lasso"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    prob = G.build(cfg)
    st = SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"], max_iter=iters)
    s = Solver(prob, st)
    s.solve()                         # leaves a factor of the last iteration
    ctx = s._ctx
    dim = s.n + s.m
    rhs = np.random.default_rng(0).standard_normal(dim)
    x = np.zeros(dim)
    steps = ctypes.c_int(0)
    res = ctypes.c_double(0)
    out = {}
    for rep in range(3):
        ctx.call("cipm_profile", 1)
        ctx.call("cipm_factor")
        ctx.call("cipm_sync")
        ctx.call("cipm_kkt_solve", pdbl(rhs), pdbl(x), ctypes.byref(steps), ctypes.byref(res))
        kst = np.zeros(5)
        ctx.call("cipm_kernel_stats", pdbl(kst))
        out[rep] = dict(factor_ms=kst[0] / max(1, kst[1]), solve_pair_ms=kst[2] / max(1, kst[3]),
                        refine_steps=steps.value, residual=res.value)
    print(json.dumps(dict(config=cfg, env={k: v for k, v in os.environ.items() if k.startswith("CIPM_")},
                          runs=out)))
    s.close()




def trace_main():
    """python tools/solve_probe.py --trace c2_lasso: per-task timeline of one
    factorisation and one forward sweep (writes gpurun_out/trace_<cfg>.npz)."""
    cfg = sys.argv[2]
    prob = G.build(cfg)
    st = SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"], max_iter=3)
    s = Solver(prob, st)
    s.solve()
    ctx = s._ctx
    dim = s.n + s.m
    rhs = np.random.default_rng(0).standard_normal(dim)
    x = np.zeros(dim)
    steps, res = ctypes.c_int(0), ctypes.c_double(0)
    ctx.call("cipm_factor")
    ctx.call("cipm_kkt_solve", pdbl(rhs), pdbl(x), ctypes.byref(steps), ctypes.byref(res))
    ctx.call("cipm_trace", 1, None)
    ctx.call("cipm_factor")
    ctx.call("cipm_kkt_solve", pdbl(rhs), pdbl(x), ctypes.byref(steps), ctypes.byref(res))
    ns = s.symbolic.info()["nsuper"]
    out = np.zeros(12 * ns, dtype=np.int64)
    ctx.call("cipm_trace", 0, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", f"trace_{cfg}.npz"), fwd=out[:6 * ns].reshape(ns, 6),
             fac=out[6 * ns:].reshape(ns, 6),
             order=s.symbolic.array("order"), sn_col=s.symbolic.array("sn_col"),
             sn_rptr=s.symbolic.array("sn_rptr"), sn_parent=s.symbolic.array("sn_parent"))
    print("trace written", ns)


def host_main():
    """python tools/solve_probe.py --host c2_lasso: per-entry-point wall time of one solve
    (CIPM_HOST_PROFILE=1 synchronises after every C call)."""
    os.environ["CIPM_HOST_PROFILE"] = "1"
    from paper_2412_19027_b200 import native
    native.DeviceContext.host_profile = True
    cfg = sys.argv[2]
    prob = G.build(cfg)
    s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"]))
    s.solve()
    s._ctx.profile = {}
    t0 = time.perf_counter()
    r = s.solve()
    wall = time.perf_counter() - t0
    prof = s._ctx.profile
    tot = sum(v[0] for v in prof.values())
    print(f"{cfg}: wall {wall*1e3:.2f} ms, in C calls {tot*1e3:.2f} ms, iterations {r.iterations}")
    for k, (t, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:24s} {n:4d} calls {t*1e3:9.3f} ms  {t*1e3/max(1,n):8.3f} ms/call")
    s.close()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--host":
    host_main()
    sys.exit(0)

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--trace":
    trace_main()
    sys.exit(0)


if __name__ == "__main__":
    main()
