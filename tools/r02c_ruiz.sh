#!/bin/bash
O=gpurun_out/${1:-ruiz}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_configs.py -m gpu -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 300 python tools/e2e_probe.py c2_lasso > $O/e2e_c2.txt 2>&1; echo "e2e rc=$?"; head -6 $O/e2e_c2.txt
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
python -c "import json;d=json.load(open('$O/c2.json'));print('c2',d['value'],d['e2e']['value'])"
