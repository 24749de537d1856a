#!/bin/bash
# bench lines only (every config, reference CPU baseline on the host cores) + GPU tests
O=gpurun_out/rb; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $O/gputests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gputests.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --config c5b_mpc --steps 3 --warmup 3 > $O/bench_c5b.json 2> $O/bench_c5b.err; echo "c5b rc=$?"
for c in c1_lp c3_socp c5a_psd; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config c4_exppow --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c4_exppow.json 2> $O/bench_c4_exppow.err; echo "c4 rc=$?"
CIPM_PHASES=1 timeout 200 python tools/solve_probe.py c2_lasso 2 2>&1 | grep phases | tail -1 > $O/phases_c2.txt
