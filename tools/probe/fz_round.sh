timeout -s KILL 600 python tools/probe/fused_repro.py > gpurun_out/fr.log 2>&1
for cfg in C5 C2; do timeout -s KILL 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_$cfg.log 2>&1; done
SCPL_HOST_LOOPS=1 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:carve_pass_kernel -s 12 -c 1 -o gpurun_out/fz_pass -f python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/fz_ncu.log 2>&1
