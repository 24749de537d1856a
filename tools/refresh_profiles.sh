#!/bin/bash
# Round-end evidence pass on one B200: GPU tests, bench lines per config (with the
# reference CPU baseline), the C2 launch list and ncu --set full captures of the
# top kernels.  Everything lands in gpurun_out/r/ (copied to profiles/ by hand).
O=gpurun_out/r; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $O/gputests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gputests.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --config c5b_mpc --steps 3 --warmup 3 > $O/bench_c5b.json 2> $O/bench_c5b.err; echo "c5b rc=$?"
for c in c1_lp c3_socp c5a_psd; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config c4_exppow --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c4_exppow.json 2> $O/bench_c4_exppow.err; echo "c4 rc=$?"
timeout 600 python tools/refine_steps.py > $O/refine_steps.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/launches_c2.csv 30 > $O/launches_c2_summary.txt 2>&1
mkdir -p gpurun_out/ncu
bash tools/ncu_kernels.sh > $O/ncu_kernels.log 2>&1; echo "ncu rc=$?"
