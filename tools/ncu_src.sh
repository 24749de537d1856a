#!/bin/bash
# ncu source-level (CUDA line) export for selected kernels of one solve probe.
#   tools/ncu_src.sh <config> <kernel-regex> <count> <tag>
cfg=$1; rx=$2; cnt=${3:-1}; tag=${4:-src}
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -c $cnt -o /tmp/$tag python tools/solve_probe.py $cfg 2 > gpurun_out/ncu/${tag}.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu/${tag}_cuda.csv 2>>gpurun_out/ncu/${tag}.log
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/ncu/${tag}_raw.csv 2>>gpurun_out/ncu/${tag}.log
ls -la gpurun_out/ncu/${tag}*
