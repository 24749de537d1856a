#!/bin/bash
# experiment: batch tests, solve-kernel grid sweep, ncu full of the C2 solve kernels
timeout 600 python -m pytest tests/test_batch.py -m gpu -x -q --timeout 300 > gpurun_out/batch_tests.log 2>&1; echo batch_tests=$?; tail -15 gpurun_out/batch_tests.log
for sb in 0 64 148 296 592; do
  if [ $sb = 0 ]; then unset CIPM_SOLVE_BLOCKS; else export CIPM_SOLVE_BLOCKS=$sb; fi
  timeout 300 python tools/solve_probe.py c2_lasso 3 2>&1 | tail -1
done
unset CIPM_SOLVE_BLOCKS
for fb in 148 296 592; do CIPM_FACTOR_BLOCKS=$fb timeout 300 python tools/solve_probe.py c2_lasso 3 2>&1 | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backward_kernel|factor_kernel" -s 6 -c 3 -o gpurun_out/prof_c2b python tools/solve_probe.py c2_lasso 3 > gpurun_out/ncu_c2b.log 2>&1; echo ncu=$?
