"""Summarise a cipm_trace timeline (gpurun_out/trace_<cfg>.npz from solve_probe --trace)."""
import sys

import numpy as np

d = np.load(sys.argv[1])
fac, fwd = d["fac"], d["fwd"]
w = np.diff(d["sn_col"])
r = np.diff(d["sn_rptr"])
for name, t in (("factor", fac), ("forward", fwd)):
    valid = t[:, 5] > 0
    if not valid.any():
        continue
    t0 = t[valid, 0].min()
    print(f"{name}: span {(t[valid, 5].max() - t0) / 1e3:.1f} us over {valid.sum()} tasks")
    big = valid & (w * r > 507)
    small = valid & ~big
    for lab, sel in (("cta-ish", big), ("warp", small)):
        if not sel.any():
            continue
        f = t[sel]
        ph = [np.mean(f[:, k + 1] - f[:, k]) / 1e3 for k in range(1, 5)]
        print(f"  {lab:8s} n={sel.sum():6d} phases(us) " + " ".join(f"{p:6.2f}" for p in ph) +
              f"  total {np.mean(f[:, 5] - f[:, 0]) / 1e3:6.2f}  first {(f[:, 0].min() - t0) / 1e3:7.1f}"
              f"  last {(f[:, 5].max() - t0) / 1e3:7.1f}")
