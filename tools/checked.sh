#!/bin/bash
# The checked build (libscpl_checked.so: device-side invariant checks that trap, see
# SCPL_DCHECK in scpl_common.cuh) over small clips and the stress set, every DP window variant,
# graph and host-driven loops.  (compute-sanitizer is closed on the GPU pool: runs under it
# have left GPUs needing a reset, so the invariants are checked by the kernels themselves.)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/checked.txt
: > $out
for kc in 3 4 6; do
  for loops in 0 1; do
    env=(SCPL_CHECKED=1 SCPL_CARVE_KC=$kc)
    [ $loops = 1 ] && env+=(SCPL_HOST_LOOPS=1)
    timeout 600 env "${env[@]}" python tools/probe/checked_case.py > gpurun_out/checked_kc${kc}_l${loops}.log 2>&1
    echo "small clips kc=$kc host_loops=$loops rc=$? :: $(grep -E 'CHECKED CASE|SCPL_DCHECK' gpurun_out/checked_kc${kc}_l${loops}.log | head -3 | tr '\n' ' ')" >> $out
  done
done
timeout 1200 env SCPL_CHECKED=1 python tools/probe/stress.py ${REPS:-5} --batch 16 > gpurun_out/checked_stress.log 2>&1
echo "stress (checked build) rc=$? :: $(tail -1 gpurun_out/checked_stress.log)" >> $out
cat $out
