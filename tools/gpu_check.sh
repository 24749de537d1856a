#!/bin/bash
# quick GPU iteration: tests (optional -k filter), C2 bench line, sweep phases and trace
O=gpurun_out/${1:-q}; K=${2:-}; mkdir -p $O
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -k "$K" > $O/gputests.log 2>&1
else timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 > $O/gputests.log 2>&1; fi
echo "tests rc=$?"; tail -3 $O/gputests.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python - $O/bench.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("value",round(d["value"],1),d["unit"],"ms/step",round(d["ms_per_step"],2),"e2e",round(d["e2e"]["value"],1),
          "frac",round(d["roofline"]["frac"],4),"pair_ms",round(d["roofline"].get("solve_ms_avg_per_pair",0),4),
          "factor_ms",round(d["roofline"].get("factor_ms_avg",0),4),"status",d["config"].get("status"),d["config"].get("iterations_per_solve"))
except Exception as e: print("bench parse failed",e)
PY
CIPM_PHASES=1 timeout 300 python tools/solve_probe.py c2_lasso 3 2>&1 | grep phases | tail -1
timeout 300 python tools/solve_probe.py --trace c2_lasso > $O/trace.log 2>&1; mv gpurun_out/trace_c2_lasso.npz $O/ 2>/dev/null
timeout 300 python tools/solve_probe.py --host c2_lasso 2>&1 | head -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_probe.csv python tools/solve_probe.py c2_lasso 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_probe.csv 25 > $O/launches_probe.txt 2>&1; head -30 $O/launches_probe.txt
