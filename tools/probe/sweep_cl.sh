for cl in 4 3 2; do for gm in 4 8; do
 echo "CL=$cl GM=$gm"; SCPL_CARVE_CL=$cl SCPL_GROUP_MIN=$gm timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['phases_ms'])"
done; done
