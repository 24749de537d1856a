#!/bin/bash
O=gpurun_out/${1:-tl}; mkdir -p $O
for c in c2_lasso c1_lp c3_socp; do
timeout 600 python tools/cupti_timeline.py $c $O/tl_$c.json > $O/tl_$c.txt 2>&1; echo "$c rc=$?"; head -45 $O/tl_$c.txt
done
