#!/bin/bash
# sweep-pair / factor time of one config with an env toggle A/B: $1 config, $2 "VAR=val"
probe() { timeout 300 python tools/solve_probe.py $1 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["runs"]["2"]; print("factor_ms %.3f pair_ms %.4f steps %d" % (r["factor_ms"], r["solve_pair_ms"], r["refine_steps"]))'; }
for cfg in $1; do
  echo "$cfg default   $(probe $cfg)"
  echo "$cfg $2 $(env $2 bash -c "$(declare -f probe); probe $cfg")"
done
