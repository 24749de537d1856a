#!/bin/bash
O=gpurun_out/${1:-rec}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_batch.py -m gpu -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
timeout 300 python tools/e2e_probe.py c2_lasso > $O/e2e_c2.txt 2>&1; echo "e2e rc=$?"
