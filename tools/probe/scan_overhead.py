"""Per-iteration overhead of the device-side scan loop: scan-only calls on tiny frames (the
window kernel is ~2 us there), smooth frames (long runs) and noise (a breach per window)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200 import pipeline  # noqa: E402

rng = np.random.default_rng(0)
T, H, W = 320, 48, 64
base = rng.integers(0, 255, (H, W, 3), dtype=np.uint8)
smooth = np.stack([base] * T)
smooth[:, 0, 0, 0] = np.arange(T) % 7
noise = rng.integers(0, 255, (T, H, W, 3), dtype=np.uint8)
for label, clip in (("smooth", smooth), ("noise", noise)):
    dev = torch.from_numpy(clip).cuda()
    cfg = P.RetargetConfig(target_width=W, target_height=H, mode="buffered")
    for _ in range(3):
        P.retarget_video_tensor(dev, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        out, m = P.retarget_video_tensor(dev, cfg)
    e1.record()
    torch.cuda.synchronize()
    ph = pipeline.last_phase_ms
    print(f"{label}: {e0.elapsed_time(e1) / reps:.3f} ms/call, runs {len(m.runs)}, windows {ph.get('scan_windows')}, "
          f"scan {ph.get('scan'):.3f} ms -> {1e3 * ph.get('scan') / max(ph.get('scan_windows'), 1):.1f} us per window")
