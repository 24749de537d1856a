#!/bin/bash
# per-kernel launch summary (ncu, cold/serialised) of one solve probe: $1 = config
cfg=$1; O=gpurun_out/lp; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$cfg.csv python tools/solve_probe.py $cfg 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_$cfg.csv 16
