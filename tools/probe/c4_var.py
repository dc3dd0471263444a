"""Step-to-step variation of the C4 batch (device-resident): per-step device times in one process."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
devs = []
for i in range(64):
    c, tw, th = config_clip("C4", clip=i)
    devs.append(torch.from_numpy(c).cuda())
cfg = P.RetargetConfig(target_width=tw, mode="buffered")
for _ in range(2):
    P.retarget_videos(devs, cfg)
torch.cuda.synchronize()
ts = []
for _ in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.retarget_videos(devs, cfg)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get("LABEL", ""), " ".join(f"{t:.1f}" for t in ts), flush=True)
