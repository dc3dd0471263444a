#!/bin/bash
# screened-scan check: GPU tests, config benches, scan loop overhead, window kernel launch times
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/t5.log
rm -f gpurun_out/b5.log
for c in C2 C5 C3 C4 C1; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']; print('$c', round(d['ms_per_step'],2), 'scan', round(p['scan'],2), 'windows', p['scan_windows'], 'fallbacks', p['scan_fallbacks'])" >> gpurun_out/b5.log; done
timeout 300 python tools/probe/scan_overhead.py >> gpurun_out/b5.log 2>&1
SCPL_HOST_LOOPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:window_stats_scan --csv --log-file gpurun_out/ws_new.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
