O=gpurun_out/rt; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 > $O/gputests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gputests.log; grep "^FAILED" $O/gputests.log | head -3
probe() { timeout 300 python tools/solve_probe.py $1 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["runs"]["2"]; print("factor_ms %.3f pair_ms %.4f steps %d" % (r["factor_ms"], r["solve_pair_ms"], r["refine_steps"]))'; }
for c in c2_lasso c3_socp; do echo "$c $(probe $c)"; done
timeout 600 python bench.py --no-cpu-baseline > $O/b2.json 2>&1; python -c "
import json; d=json.loads(open('$O/b2.json').read().strip().splitlines()[-1]); print('c2 value', d['value'], 'e2e', d['e2e']['value'], d['config']['status'])"
bash tools/ncu_fwdsrc.sh c3_socp
