#!/bin/bash
# GPU tests + per-config bench lines (value, ms/step, status, iters, factor ms, solve-pair ms, e2e)
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
for c in ${CONFIGS:-c2_lasso c1_lp c3_socp c5a_psd}; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$c',round(d['value'],2),round(d['ms_per_step'],2),d['config']['status'],d['config']['iterations_per_solve'],round(d['roofline']['factor_ms_avg'],3),round(d['roofline']['solve_ms_avg_per_pair'],3),'e2e',round(d['e2e']['value'],2))"; done
