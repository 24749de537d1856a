"""GPU probe: live per-kernel durations and the gaps between kernels of one warm
solve (torch.profiler / CUPTI, not serialised like ncu).

    python tools/cupti_timeline.py c2_lasso [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2412_19027_b200 import generators as G  # noqa: E402
from paper_2412_19027_b200.settings import SolverSettings  # noqa: E402
from paper_2412_19027_b200.solver import Solver  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2_lasso"
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    prob = G.build(cfg)
    s = Solver(prob, SolverSettings(eps_feas=1e-8, precision=G.CONFIGS[cfg]["precision"]))
    s.solve()
    s.solve()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = s.solve()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda t: t[0])
    t0, t1 = ks[0][0], ks[-1][1]
    busy = {}
    for a, b, n in ks:
        k = n.split("(")[0][:60]
        d = busy.setdefault(k, [0, 0.0])
        d[0] += 1
        d[1] += b - a
    span = t1 - t0
    tot = sum(v[1] for v in busy.values())
    print(f"{cfg}: {r.iterations} iterations, span {span / 1e3:.2f} ms, kernel time {tot / 1e3:.2f} ms, "
          f"{len(ks)} kernels, idle {100 * (1 - tot / span):.1f} %")
    for k, (c, t) in sorted(busy.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"  {k:60s} {c:6d} {t / 1e3:8.3f} ms {t / c:8.2f} us/launch {100 * t / span:5.1f} %")
    if out_path:
        with open(out_path, "w") as f:
            json.dump([(a - t0, b - t0, n) for a, b, n in ks], f)
    s.close()


if __name__ == "__main__":
    main()
