"""One 1080p run carved alone (the e2e critical path's last step): device time per call and
phase split; with SCPL_HOST_LOOPS=1 under ncu it gives the per-kernel durations."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200 import pipeline  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
clip, tw, th = config_clip("C2", frames=nfr)
dev = torch.from_numpy(clip).cuda()
cfg = P.RetargetConfig(target_width=tw, mode="buffered")
for _ in range(2 if reps > 1 else 0):
    P.retarget_video_tensor(dev, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    out, m = P.retarget_video_tensor(dev, cfg)
e1.record()
torch.cuda.synchronize()
print(f"{nfr} frame(s): {e0.elapsed_time(e1) / reps:.3f} ms/call, runs {m.runs}, passes {m.dp_passes}")
print(pipeline.last_phase_ms)
