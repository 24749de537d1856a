#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 2>&1 | tail -8
CIPM_SOLVE_SLICE=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 2>&1 | tail -4
