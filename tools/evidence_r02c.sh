#!/bin/bash
# round-2 (session 3) final evidence pass, one fresh box: GPU tests, smoke, bench lines of
# every config with the reference CPU baselines, the reference arm for C2, the C2 launch
# list, the ncu sweep-traffic capture, the CUPTI timeline and the e2e host probes
O=gpurun_out/ev10; mkdir -p $O gpurun_out/ncu
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/gputests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c2_lasso.json 2> $O/bench_c2_lasso.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c5b_mpc --steps 3 --warmup 3 > $O/bench_c5b_mpc.json 2> $O/bench_c5b_mpc.err; echo "c5b rc=$?"
for c in c1_lp c3_socp c5a_psd c4_exppow; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_c2_lasso.json 2> $O/ref_c2_lasso.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/launches_c2.csv 30 > $O/launches_c2_summary.txt 2>&1
bash tools/ncu_sweeps.sh c2_lasso > $O/ncu_sweeps.txt 2>&1; echo "ncu sweeps rc=$?"
rm -f gpurun_out/ncu/sw_c2_lasso.ncu-rep
timeout 600 python tools/cupti_timeline.py c2_lasso $O/timeline_c2.json > $O/timeline_c2.txt 2>&1; echo "timeline rc=$?"
timeout 600 python tools/batch_e2e_probe.py > $O/batch_e2e_probe.txt 2>&1; echo "batch probe rc=$?"
timeout 300 python tools/e2e_probe.py c2_lasso > $O/e2e_probe_c2.txt 2>&1; echo "e2e probe rc=$?"
