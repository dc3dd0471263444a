#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
for sp in 8 12 16 24; do
  for c in C4 C2 C5; do
    st=5; [ $c = C4 ] && st=3
    r=$(SCPL_SPEC=$sp timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), 'scan', round(d['phases_ms']['scan'],2), 'windows', d['phases_ms']['scan_windows'])")
    echo "$c spec $sp: $r" >> gpurun_out/sp.log
  done
done
