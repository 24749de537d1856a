#!/bin/bash
# in-place base image + correctly rounded reciprocal on the pivot chains: parity, benches, diag microbench
O=gpurun_out/${1:-rcp}; mkdir -p $O
./tools/micro/diag_bench > $O/diag_div.txt 2>&1; ./tools/micro/diag_bench_rcp > $O/diag_rcp.txt 2>&1; cat $O/diag_div.txt $O/diag_rcp.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c2_lasso c1_lp c3_socp c5a_psd c4_exppow; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/$c.json 2> $O/$c.err; echo "$c rc=$?"
python -c "import json;d=json.load(open('$O/$c.json'));print('$c',d['value'],d['e2e']['value'],d['config']['iterations_per_solve'],d['config']['status'],d['roofline'].get('factor_ms_avg'),d['roofline'].get('solve_ms_avg_per_pair'))"
done
