#!/bin/bash
# quick scan iteration: scan / config parity tests, scan-only and full timings, window kernel launch times
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seams.py -m gpu -x -q -k "config_clip or scan or buffer or stream" 2>&1 | tail -3 > gpurun_out/t5.log
rm -f gpurun_out/b5.log
for c in C2 C5 C3; do timeout 300 python tools/probe/scan_alone.py $c 5 2>&1 | grep -v "^  \|run lengths" >> gpurun_out/b5.log; done
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']; print('C4', round(d['ms_per_step'],2), 'scan', round(p['scan'],2), 'windows', p['scan_windows'], 'fallbacks', p['scan_fallbacks'])" >> gpurun_out/b5.log
SCPL_HOST_LOOPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:window_stats_scan --csv --log-file gpurun_out/ws_new.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
