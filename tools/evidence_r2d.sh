#!/bin/bash
# Round-2 evidence, fourth session (r2d): benches, configs, launch lists, the window kernel's
# full capture + stall lines, streaming-kernel table
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
SCPL_HOST_LOOPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:window_stats_scan -s 3 -c 1 \
  -o gpurun_out/${R}_full_window_stats_scan -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${R}_full_ws.log 2>&1
SCPL_HOST_LOOPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:uniform_vec -s 3 -c 1 \
  -o gpurun_out/${R}_full_uniform_vec -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${R}_full_uv.log 2>&1
SCPL_HOST_LOOPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:carve_pass_kernel -s 12 -c 1 \
  -o gpurun_out/${R}_full_carve_pass_kernel -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${R}_full_carve.log 2>&1
bash tools/probe/stream_kernels.sh C2
timeout 600 python tools/probe/c4_var.py 12 > gpurun_out/${R}_c4_steps.txt 2>&1
echo done > gpurun_out/${R}_evidence.done
