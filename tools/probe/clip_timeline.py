"""Per-run carve timeline of one config clip (SCPL_PROF=1 per-pass timestamps, SCPL_TIMELINE=1
group marks): when each run's carve starts, how long its passes and the gaps between them take.

    SCPL_PROF=1 SCPL_TIMELINE=1 python tools/probe/clip_timeline.py C2
"""
import os
import re
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200 import pipeline  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
clip, tw, th = config_clip(name)
dev = torch.from_numpy(clip).cuda()
cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
for _ in range(3):
    out, m = P.retarget_video_tensor(dev, cfg)
torch.cuda.synchronize()
print("RUNS", m.runs)
print("PHASES", pipeline.last_phase_ms, flush=True)
