#!/bin/bash
# A/B of the scan speculation length on one box, interleaved (device-resident ms per step)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
out=gpurun_out/spec_ab.log; rm -f $out
run() { timeout 300 python bench.py --config $1 --steps ${2:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']; print('$1 spec=${SCPL_SPEC:-8}', round(d['ms_per_step'],2), 'scan', round(p['scan'],2), 'windows', p['scan_windows'])" >> $out; }
for rep in 1 2; do
  for spec in 8 16 12; do
    export SCPL_SPEC=$spec
    for c in C2 C5 C3; do run $c; done
    run C4 4
  done
done
