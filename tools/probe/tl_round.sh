cd $GRAFT_REPO_ROOT
SCPL_TIMELINE=1 timeout 300 python tools/probe/clip_timeline.py C2 > gpurun_out/tl_C2.log 2>&1
SCPL_TIMELINE=1 timeout 300 python tools/probe/clip_timeline.py C5 > gpurun_out/tl_C5.log 2>&1
SCPL_TIMELINE=1 timeout 600 python tools/probe/c4_batch.py --child --clips 64 --steps 1 --warmup 1 > gpurun_out/tl_C4.log 2>&1
