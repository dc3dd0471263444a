#!/bin/bash
# Regenerate the config goldens from the reference itself (build container only; ~35 min on
# 8 cores): C1..C5 with per-pass label hashes, and all 64 C4 clips.  One process per job.
set -e
cd "$(dirname "$0")/.."
export PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 OMP_NUM_THREADS=1
{
  echo "C3"; echo "C2"; echo "C5"; echo "C1"
  for c in $(seq 0 63); do echo "C4 --clip $c"; done
} | xargs -P "${JOBS:-8}" -I{} sh -c 'python tests/golden/make_golden.py {} > "/tmp/gold/$(echo {} | tr " " "_").log" 2>&1'
