#!/bin/bash
# DP phase breakdown (SCPL_CARVE_PROF build, made on the box): lone 1080p run and C5
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
SCPL_EXTRA_NVCC_FLAGS=-DSCPL_CARVE_PROF python -m paper_1903_03180_b200.build_ext --force > gpurun_out/dpp_build.log 2>&1
for kc in 3 4 6; do
  echo "== lone run kc$kc" >> gpurun_out/dpp.log
  SCPL_CARVE_KC=$kc SCPL_PROF=1 timeout 120 python tools/probe/single_run.py 4 1 2>&1 | grep -E "carve prof|carve ts|ms/call" | tail -3 >> gpurun_out/dpp.log
done
echo "== C5" >> gpurun_out/dpp.log
SCPL_PROF=1 timeout 200 python tools/probe/clip_timeline.py C5 2>&1 | grep -E "carve prof|carve ts" | tail -4 >> gpurun_out/dpp.log
