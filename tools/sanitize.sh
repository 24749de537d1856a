#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small solves (all tiers, cones, batch).
# CIPM_NO_GRAPHS=1: kernels launched eagerly (the sanitizer does not follow conditional graph nodes)
O=gpurun_out/san; mkdir -p $O
python tools/sanitize_run.py > $O/plain.log 2>&1; echo "plain rc=$? $(tail -1 $O/plain.log)"
for tool in memcheck racecheck synccheck; do
  CIPM_NO_GRAPHS=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/$tool.log | tail -2 | tr '\n' ' ')"
done
