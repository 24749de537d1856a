#!/bin/bash
timeout 300 python tools/solve_probe.py c1_lp 3 2>&1 | tail -1
CIPM_SOLVE_SLICE=4 timeout 300 python tools/solve_probe.py c1_lp 3 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --config c1_lp --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['status'],d['config']['iterations_per_solve'],d['ms_per_step'])"; done
CIPM_SOLVE_SLICE=4 timeout 300 python bench.py --config c1_lp --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('noslice',d['config']['status'],d['config']['iterations_per_solve'],d['ms_per_step'])"
