#!/bin/bash
# bench a config under env variants: tools/probe/variants.sh C2 "" "SCPL_PRIO_LATE=1" ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
cfg=$1; shift
for v in "$@"; do
  r=$(env $v timeout 600 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phases_ms']
print(f\"{d['value']:.0f} fps {d['ms_per_step']:.2f} ms scan {p['scan']:.2f} after {p['carve_after_scan']:.2f} launch {p['pass_launch_ms']*1e3:.0f}us\")" 2>&1)
  echo "$cfg [${v:-default}] $r"
done
