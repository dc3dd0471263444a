"""End-to-end (pinned host buffers) C2 timeline: H2D chunk marks, scan chunks, groups, D2H marks.

    SCPL_TIMELINE=1 python tools/probe/e2e_timeline.py [C2]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
clip, tw, th = config_clip(name)
host = torch.from_numpy(clip).pin_memory()
cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
out = None
for _ in range(3):
    out, m = P.retarget_video_tensor(host, cfg, out=out) if out is not None else P.retarget_video_tensor(host, cfg)
torch.cuda.synchronize()
