#!/bin/bash
O=gpurun_out/${1:-batch}; mkdir -p $O
timeout 600 python tools/batch_e2e_probe.py > $O/probe.txt 2>&1; echo "probe rc=$?"; cat $O/probe.txt | tail -3
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --config c5b_mpc --steps 3 --warmup 3 --no-cpu-baseline > $O/c5b.json 2> $O/c5b.err; echo "c5b rc=$?"
