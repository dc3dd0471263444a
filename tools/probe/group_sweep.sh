#!/bin/bash
# C2 / C5 device ms per step under group-size caps (SCPL_GROUP_MAX) and minimums
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
for v in "" "SCPL_GROUP_MAX=2" "SCPL_GROUP_MAX=4" "SCPL_GROUP_MAX=6" "SCPL_GROUP_MAX=8"; do
  for c in C2 C5; do
    ms=$(env $v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])['ms_per_step'],2))")
    echo "$c [${v:-default}] $ms ms" >> gpurun_out/gs.log
  done
done
