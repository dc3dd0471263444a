#!/bin/bash
# A/B: carve iterations per loop-body execution (SCPL_CARVE_UNROLL)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
out=gpurun_out/unroll_ab.log; rm -f $out
SCPL_CARVE_UNROLL=4 timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_clip_golden or size_cases or small_clips" 2>&1 | tail -2 >> $out
run() { timeout 300 env $2 python bench.py --config $1 --steps ${3:-20} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 [$2]', round(d['ms_per_step'],2))" >> $out; }
for rep in 1 2; do
  for v in "SCPL_CARVE_UNROLL=1" "SCPL_CARVE_UNROLL=2" "SCPL_CARVE_UNROLL=4"; do
    run C2 $v; run C5 $v; run C3 $v; run C4 $v 5
  done
done
for u in 1 2 4; do timeout 120 env SCPL_CARVE_UNROLL=$u python tools/probe/single_run.py 2>&1 | head -1 >> $out; done
