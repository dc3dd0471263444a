#!/bin/bash
# One GPU-box session: tests, then short benches (outputs under gpurun_out/).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout ${T_TESTS:-1500} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests.log
for cfg in ${BENCH_CONFIGS:-C2 C4}; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
  echo "bench $cfg rc=$?" >> gpurun_out/bench_$cfg.log
done
