#!/bin/bash
# ncu source-level stall profile of the persistent sweep kernels of one config ($1)
cfg=${1:-c3_socp}; O=gpurun_out/ncu; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:forward_kernel|backward_kernel" -s 2 -c 2 -o /tmp/fs_$cfg python tools/solve_probe.py $cfg 2 > $O/fs_$cfg.log 2>&1
ncu -i /tmp/fs_$cfg.ncu-rep --page source --csv --print-source cuda,sass > /tmp/fs_${cfg}_cuda.csv 2>>$O/fs_$cfg.log
ncu -i /tmp/fs_$cfg.ncu-rep --page details --csv > $O/fs_${cfg}_details.csv 2>>$O/fs_$cfg.log
python tools/ncu_lines.py /tmp/fs_${cfg}_cuda.csv 40 > $O/fs_${cfg}_lines.txt
