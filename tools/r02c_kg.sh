#!/bin/bash
O=gpurun_out/${1:-kg}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
python -c "import json;d=json.load(open('$O/c2.json'));print('c2',d['value'],d['e2e']['value'])"
timeout 600 python bench.py --config c1_lp --steps 3 --warmup 3 --no-cpu-baseline > $O/c1.json 2> $O/c1.err; echo "c1 rc=$?"
python -c "import json;d=json.load(open('$O/c1.json'));print('c1',d['value'],d['e2e']['value'])"
timeout 600 python tools/cupti_timeline.py c2_lasso $O/tl_c2.json > $O/tl_c2.txt 2>&1; echo "tl rc=$?"
