cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
for v in "SCPL_FUSED=1" "SCPL_FUSED="; do
  echo "== single run 4 frames $v" >> gpurun_out/fp.log
  env $v timeout -s KILL 120 python tools/probe/single_run.py 4 5 >> gpurun_out/fp.log 2>&1
  echo "== single run prof $v" >> gpurun_out/fp.log
  env $v SCPL_PROF=1 timeout -s KILL 120 python tools/probe/single_run.py 4 1 2>&1 | grep -E "carve prof|carve prod|carve ts|ms/call" | tail -4 >> gpurun_out/fp.log
done
echo "== C5 prof" >> gpurun_out/fp.log
SCPL_FUSED=1 SCPL_PROF=1 timeout -s KILL 200 python tools/probe/clip_timeline.py C5 2>&1 | grep -E "carve prod|carve ts|carve prof" | tail -6 >> gpurun_out/fp.log
