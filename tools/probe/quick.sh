# quick perf check: C2 bench line (device + e2e) and one lone 1080p run
timeout 150 python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']; print('C2', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), {k: round(p[k],3) for k in ('scan','carve_after_scan','carve_dp_Mcyc','carve_select_Mcyc','pass_launch_ms','scan_fallbacks')})"
python tools/probe/single_run.py 1 10 | head -1
