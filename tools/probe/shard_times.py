"""Device time of each rank's share of ONE clip (sharding.py) for N = 1, 2, 4, 8: every rank
scans the whole clip and carves its runs, with no rank waiting on another, so running the
shares one after another on one GPU gives each GPU's compute time of an N-GPU job (the NCCL
output exchange excluded)."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = 5
clip, tw, th = config_clip(name)
dev = torch.from_numpy(clip).cuda()
cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
for N in (1, 2, 4, 8):
    worst = 0.0
    for r in range(N):
        for _ in range(2):
            P.retarget_video_tensor(dev, cfg, shard=(r, N))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            P.retarget_video_tensor(dev, cfg, shard=(r, N))
        e1.record()
        torch.cuda.synchronize()
        worst = max(worst, e0.elapsed_time(e1) / reps)
    print(f"{name} N={N}: slowest rank {worst:.3f} ms -> {clip.shape[0] / worst * 1e3:.0f} frames/s "
          f"(excl. output exchange)", flush=True)
