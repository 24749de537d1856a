#!/bin/bash
# ncu source-level capture of the batched IPM kernel (C5b, 2048 instances)
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_ipm -c 1 -o /tmp/bsrc python bench.py --config c5b_mpc --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu/bsrc.log 2>&1
ncu -i /tmp/bsrc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu/bsrc_cuda.csv 2>>gpurun_out/ncu/bsrc.log
ncu -i /tmp/bsrc.ncu-rep --page raw --csv > gpurun_out/ncu/bsrc_raw.csv 2>>gpurun_out/ncu/bsrc.log
python tools/ncu_lines.py gpurun_out/ncu/bsrc_cuda.csv 45 > gpurun_out/ncu/bsrc_lines.txt
rm -f gpurun_out/ncu/bsrc_cuda.csv
