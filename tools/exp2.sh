#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputests.log
for c in c2_lasso c3_socp c5a_psd; do timeout 300 python tools/solve_probe.py $c 3 2>&1 | tail -1; done
timeout 300 python tools/solve_probe.py --trace c2_lasso
for c in c2_lasso c1_lp c3_socp c5a_psd; do timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; python -c "import json;d=json.load(open(\"gpurun_out/bench_$c.json\"));print(d[\"value\"],d[\"ms_per_step\"],d[\"config\"][\"status\"],d[\"config\"][\"iterations_per_solve\"],d[\"roofline\"][\"factor_ms_avg\"],d[\"roofline\"][\"solve_ms_avg_per_pair\"])"; done
