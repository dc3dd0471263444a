#!/bin/bash
# per-launch duration + DRAM bytes of the streaming kernels over one C2 step (graph loops: the
# uniform / replay / codes launches are plain launches); ncu numbers are cold-cache, serialised
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"replay_rows_vec|uniform_vec|codes_kernel" --csv --log-file gpurun_out/sk_${1:-C2}.csv \
  python bench.py --config ${1:-C2} --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/sk_${1:-C2}.log 2>&1
