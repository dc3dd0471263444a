cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1
for c in C2 C5 C3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), d['phases_ms']['pass_launch_ms'])" >> gpurun_out/b4.log; done
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4', round(d['ms_per_step'],2), d['phases_ms']['pass_launch_ms'])" >> gpurun_out/b4.log
rm -f gpurun_out/dpp.log; bash tools/probe/dp_prof.sh
