#!/bin/bash
# one ncu --set full capture of every sweep kernel of a refinement step (config $1), raw CSV out
cfg=${1:-c2_lasso}; O=gpurun_out/ncu; mkdir -p $O
rx="fwd_tiny_kernel|tiny_fold_kernel|forward_kernel|root_solve|tail_fwd|tail_bwd|backward_kernel|bwd_tiny_kernel|scatter_add_perm"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 40 -c 9 -o /tmp/sw_$cfg python tools/solve_probe.py $cfg 3 > $O/sw_$cfg.log 2>&1
ncu -i /tmp/sw_$cfg.ncu-rep --page raw --csv > $O/sw_${cfg}_raw.csv 2>>$O/sw_$cfg.log
cp /tmp/sw_$cfg.ncu-rep $O/ 2>/dev/null
python tools/ncu_traffic.py $O/sw_${cfg}_raw.csv $cfg $O/ncu_traffic.json | head -5
