#!/bin/bash
O=gpurun_out/${1:-pin}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_batch.py tests/test_gpu_configs.py -m gpu -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python tools/batch_e2e_probe.py > $O/probe.txt 2>&1; echo "probe rc=$?"; cat $O/probe.txt | tail -6
timeout 300 python tools/e2e_probe.py c2_lasso > $O/e2e_c2.txt 2>&1; echo "e2e rc=$?"; head -6 $O/e2e_c2.txt
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c5b_mpc --steps 3 --warmup 3 --no-cpu-baseline > $O/c5b.json 2> $O/c5b.err; echo "c5b rc=$?"
for f in c2 c5b; do python -c "import json;d=json.load(open('$O/$f.json'));print('$f',d['value'],d['e2e']['value'],d['e2e']['d2h_bytes_per_step'])"; done
