#!/bin/bash
# full GPU pass: tests, bench lines (default + batched), launch list, ncu capture of the top kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?; tail -c 600 gpurun_out/bench_default.json
timeout 600 python bench.py --config c5b_mpc --steps 3 --warmup 3 > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err; echo c5b=$?; tail -c 800 gpurun_out/bench_c5b.json; tail -3 gpurun_out/bench_c5b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backward_kernel|factor_kernel|factor_cta_kernel" -s 8 -c 4 -o gpurun_out/prof_c2_full python tools/solve_probe.py c2_lasso 3 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
