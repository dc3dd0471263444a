#!/bin/bash
# A/B: scan windows per loop-body execution (SCPL_SCAN_UNROLL)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
out=gpurun_out/scan_unroll_ab.log; rm -f $out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seams.py -m gpu -x -q -k "config_clip or scan or buffer or stream or weights" 2>&1 | tail -2 >> $out
run() { timeout 300 env $2 python bench.py --config $1 --steps ${3:-20} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 [$2]', round(d['ms_per_step'],2), 'scan', round(d['phases_ms']['scan'],2))" >> $out; }
for rep in 1 2; do
  for v in "SCPL_SCAN_UNROLL=1" "SCPL_SCAN_UNROLL=2" "SCPL_SCAN_UNROLL=3"; do
    run C2 $v; run C5 $v; run C3 $v; run C4 $v 5
  done
done
