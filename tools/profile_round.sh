#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box, one GPU): launch list of one C2 step with
# host-driven loops (every kernel visible), and a full-set capture of each main kernel.
set -x
OUT=${OUT:-gpurun_out}
export SCPL_HOST_LOOPS=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
for k in carve_pass codes_kernel window_stats_scan carve_compact carve_dirty replay_rows uniform_kernel; do
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -o $OUT/full_$k \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$k.log 2>&1
done
