#!/bin/bash
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/initcheck.log 2>&1; echo initcheck=$?; grep -E "ERROR SUMMARY|Uninitialized|at 0x|in .*cipm" gpurun_out/initcheck.log | head -30
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/memcheck.log 2>&1; echo memcheck=$?; grep -E "ERROR SUMMARY|Invalid|at 0x" gpurun_out/memcheck.log | head -20
tail -6 gpurun_out/memcheck.log
