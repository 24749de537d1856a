#!/bin/bash
# C2 factor / forward critical-path trace + bench value only (fast iteration)
O=gpurun_out/${1:-t}; mkdir -p $O
timeout 300 python tools/solve_probe.py --trace c2_lasso > $O/trace.log 2>&1; mv gpurun_out/trace_c2_lasso.npz $O/ 2>/dev/null
timeout 300 python tools/solve_probe.py c2_lasso 3 2>&1 | tail -1
timeout 300 python tools/solve_probe.py --host c2_lasso 2>&1 | head -4
