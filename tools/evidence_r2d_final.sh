#!/bin/bash
# Round-2 evidence on the final commit (fourth session): bench lines, configs, launch lists
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=r2d
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench_C2.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 --warmup 4 --no-cpu-baseline > gpurun_out/${R}_bench_C4.log 2>&1
timeout 1200 bash tools/probe/all_configs.sh > gpurun_out/${R}_configs.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/${R}_ncu_bench.log 2>&1
SCPL_HOST_LOOPS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches_C2_hostloops.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/${R}_ncu_hl.log 2>&1
timeout 300 python tools/probe/scan_overhead.py > gpurun_out/${R}_scan_overhead.txt 2>&1
echo done > gpurun_out/${R}_final.done
