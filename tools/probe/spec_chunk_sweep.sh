#!/bin/bash
# device-resident ms per step under scan speculation lengths (SCPL_SPEC) and chunk lengths (SCPL_CHUNK)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
out=gpurun_out/spec_chunk.log; rm -f $out
run() { timeout 300 python bench.py --config $1 --steps ${2:-8} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']; print('$1 spec=${SCPL_SPEC:-8} chunk=${SCPL_CHUNK:-16}', round(d['ms_per_step'],2), 'scan', round(p['scan'],2), 'windows', p['scan_windows'])" >> $out; }
for spec in 8 12 16 24; do
  export SCPL_SPEC=$spec
  for c in C2 C5 C3; do run $c; done
  run C4 3
done
export SCPL_SPEC=8
for ch in 32 64 300; do
  export SCPL_CHUNK=$ch
  for c in C2 C5 C3; do run $c; done
done
