cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
for d in 0 1 4 8; do
  echo "== FDBG $d" >> gpurun_out/fd.log
  SCPL_FDBG=$d SCPL_PROF=1 timeout -s KILL 120 python tools/probe/single_run.py 4 1 2>&1 | grep -E "carve prod|carve ts|ms/call" | tail -3 >> gpurun_out/fd.log
done
