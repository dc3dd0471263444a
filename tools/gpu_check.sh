#!/bin/bash
# build locally, then run the GPU tests + a short bench on the box; prints test summary and phases
set -e
cd /root/repo
python -m paper_1903_03180_b200.build_ext > /tmp/build.log 2>&1 || { grep -E "error" -A3 /tmp/build.log | head -20; exit 1; }
grep -E "error" /tmp/build.log && exit 1
STEPS=${STEPS:-5}
/usr/local/graft/bin/gpurun --timeout ${TIMEOUT:-900} -- "timeout -s KILL 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/t.log; timeout -s KILL 300 python bench.py --no-cpu-baseline ${BENCH_ARGS:---no-e2e} --steps $STEPS --warmup 3 > gpurun_out/b.log 2>&1; ${EXTRA_CMD:-true}" > /tmp/gpurun.log 2>&1 || true
tail -2 /tmp/gpurun.log
cat gpurun_out/t.log
grep -o "\"phases_ms\": {[^}]*}" gpurun_out/b.log || tail -5 gpurun_out/b.log
grep -o "\"ms_per_step\": [0-9.]*\|\"e2e\": {[^}]*}" gpurun_out/b.log
