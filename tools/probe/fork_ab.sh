#!/bin/bash
# A/B: the carve loop's condition kernel on a side branch after the pass (SCPL_CHECK_FORK=1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
out=gpurun_out/fork_ab.log; rm -f $out
SCPL_CHECK_FORK=1 timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_clip_golden or size_cases or small_clips" 2>&1 | tail -2 >> $out
run() { timeout 300 env $2 python bench.py --config $1 --steps ${3:-20} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 [$2]', round(d['ms_per_step'],2))" >> $out; }
for rep in 1 2; do
  for v in "SCPL_CHECK_FORK=0" "SCPL_CHECK_FORK=1"; do
    run C2 $v; run C5 $v; run C3 $v; run C4 $v 5
  done
done
timeout 120 env SCPL_CHECK_FORK=1 python tools/probe/single_run.py >> $out 2>&1
timeout 120 env SCPL_CHECK_FORK=0 python tools/probe/single_run.py >> $out 2>&1
