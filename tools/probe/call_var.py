"""Call-to-call variation: per-call device time and host wall time of one config clip
(scan-only and full) -- looks for rare slow calls."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
clip, tw, th = config_clip(name)
dev = torch.from_numpy(clip).cuda()
T, H, W = clip.shape[:3]
for label, cfg in (("scan only", P.RetargetConfig(target_width=W, target_height=H, mode="buffered")),
                   ("full", P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))):
    for _ in range(2):
        P.retarget_video_tensor(dev, cfg)
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        P.retarget_video_tensor(dev, cfg)
        e1.record()
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    print(name, label, " ".join(f"{d:.1f}/{h:.1f}" for d, h in out), flush=True)
