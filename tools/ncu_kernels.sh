#!/bin/bash
# one ncu --set full capture per kernel class; only the raw-metric CSVs come back
mkdir -p gpurun_out/ncu
cap() {  # name regex skip count cmd...
  local name=$1 rx=$2 sk=$3 cnt=$4; shift 4
  timeout 900 ncu --set full --clock-control none -k regex:"$rx" -s $sk -c $cnt -o /tmp/$name "$@" > /dev/null 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/ncu/$name.csv 2>/dev/null
  echo "$name $(wc -l < gpurun_out/ncu/$name.csv)"
}
cap c2_vec "resid_n|resid_m|kkt_res_n|nn_update_scaling|nn_combined_ds|mu_candidates" 20 6 python bench.py --config c2_lasso --steps 1 --warmup 1 --no-cpu-baseline
cap c2_solve "forward_kernel|backward_kernel|factor_kernel|factor_cta_kernel" 4 4 python tools/solve_probe.py c2_lasso 3
cap c3_soc "soc_" 10 6 python bench.py --config c3_socp --steps 1 --warmup 0 --no-cpu-baseline
cap c5a_psd "psd_" 10 6 python bench.py --config c5a_psd --steps 1 --warmup 0 --no-cpu-baseline
cap c4_nsym "nsym_" 10 6 python tools/c4_check.py fifth
cap c1_gemm "tail_gemm|tail_diag" 30 6 python tools/solve_probe.py c1_lp 2
cap c1_tailsolve "tail_fwd|tail_bwd" 40 6 python tools/solve_probe.py c1_lp 2
cap c3_solve "forward_kernel|backward_kernel|factor_cta_kernel" 4 3 python tools/solve_probe.py c3_socp 3
cap c5b_batch "batch_ipm" 0 1 python bench.py --config c5b_mpc --steps 1 --warmup 0 --no-cpu-baseline
du -sh gpurun_out/ncu
