"""The buffer scan of C2 with nothing to carve (targets = source size): its device time alone,
to compare with the scan phase of the full pipeline (where carve clusters share the SMs)."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200 import pipeline  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
clip, tw, th = config_clip(name)
dev = torch.from_numpy(clip).cuda()
T, H, W = clip.shape[:3]
for label, cfg in (("scan only", P.RetargetConfig(target_width=W, target_height=H, mode="buffered")),
                   ("full", P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))):
    for _ in range(2):
        P.retarget_video_tensor(dev, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out, m = P.retarget_video_tensor(dev, cfg)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / reps:.3f} ms/call, runs {len(m.runs)}, passes {m.dp_passes}")
    print("  ", pipeline.last_phase_ms)
print("run lengths", [n for _, n in m.runs])
