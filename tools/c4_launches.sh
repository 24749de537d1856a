#!/bin/bash
# C4 launch list of one factor + refined solve at a fixed iterate (per-kernel shares)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/solve_probe.py c4_exppow 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c4.csv 25
