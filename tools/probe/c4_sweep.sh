#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
for v in "" "SCPL_LANES=4" "SCPL_LANES=12" "SCPL_LANES=16" "SCPL_GROUP_MIN=4" "SCPL_GROUP_MIN=16" "SCPL_GROUP_MAX=8" "SCPL_LANES=16,SCPL_GROUP_MIN=16"; do
  python tools/probe/c4_batch.py --clips 64 --steps 3 "$v" >> gpurun_out/c4s.log 2>&1
done
