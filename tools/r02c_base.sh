#!/bin/bash
# baseline timings on a fresh box (session 3 of round 2)
O=gpurun_out/${1:-base}; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
timeout 300 python tools/e2e_probe.py c2_lasso > $O/e2e_c2.txt 2>&1; echo "e2e rc=$?"
timeout 300 python tools/solve_probe.py c2_lasso 6 > $O/probe_c2.txt 2>&1; echo "probe rc=$?"
timeout 300 python tools/solve_probe.py --host c2_lasso > $O/host_c2.txt 2>&1; echo "host rc=$?"
timeout 600 python bench.py --config c5b_mpc --steps 3 --warmup 3 --no-cpu-baseline > $O/c5b.json 2> $O/c5b.err; echo "c5b rc=$?"
timeout 600 python bench.py --config c1_lp --steps 3 --warmup 3 --no-cpu-baseline > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
