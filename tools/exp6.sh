#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -1
for m in 0 256 512 1024; do
  echo "== chain merge $m"
  CIPM_CHAIN_MERGE=$m timeout 300 python bench.py --config c2_lasso --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['config']['status'],d['config']['iterations_per_solve'],d['roofline']['factor_ms_avg'],d['roofline']['solve_ms_avg_per_pair'])"
done
for c in c1_lp c3_socp c5a_psd; do timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$c',d['value'],d['ms_per_step'],d['config']['status'],d['config']['iterations_per_solve'],d['roofline']['factor_ms_avg'],d['roofline']['solve_ms_avg_per_pair'])"; done
