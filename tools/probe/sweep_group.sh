# carve throughput without scan overlap: every run in one group dispatched after the scan
for cfg in "1000 4" "1000 3" "1000 2" "4 4"; do
  set -- $cfg
  echo "GM=$1 CL=$2"; SCPL_GROUP_MIN=$1 SCPL_CARVE_CL=$2 timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']; print(round(d['ms_per_step'],3), {k: round(p[k],3) for k in ('scan','carve_after_scan','carve_dp_Mcyc','carve_select_Mcyc','pass_launch_ms')})"
done
