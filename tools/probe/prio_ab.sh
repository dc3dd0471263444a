#!/bin/bash
# A/B of the carve groups' priority order now that graph kernel nodes carry their stream's priority
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
out=gpurun_out/prio_ab.log; rm -f $out
run() { timeout 300 env $2 python bench.py --config $1 --steps ${3:-20} --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 [$2]', round(d['ms_per_step'],2))" >> $out; }
for rep in 1 2; do
  for v in "X=1" "SCPL_PRIO_LATE=1" "SCPL_GRAPH_PRIO=0"; do
    run C2 $v; run C5 $v; run C4 $v 5
  done
done
sort $out
