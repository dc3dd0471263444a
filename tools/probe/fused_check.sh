#!/bin/bash
# fused-pass bring-up: small parity first (hard timeouts), then goldens, then benches
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"
mkdir -p gpurun_out
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fc_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fc_smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/fc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fc_tests.log
for cfg in ${BENCH_CONFIGS:-C2 C5}; do
  timeout -s KILL 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_$cfg.log 2>&1
done
