"""Small clips through every kernel of the path, for the checked build (tools/checked.sh):
a buffered clip carved on both axes, a reaverage clip, raw mode, and a two-clip batch; each
result is checked against the CPU oracle (test infrastructure, not the product)."""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
import paper_1903_03180_b200 as P  # noqa: E402
from oracle import scpl_oracle as O  # noqa: E402

rng = np.random.default_rng(12)
T, h, w = 10, 70, 150
base = np.round(255.0 * np.arange(w) / (w - 1))[None, :, None].repeat(h, 0).repeat(3, 2)
frames = []
for k in range(T):
    img = base.copy()
    img[10:30, 5 + 3 * k:40 + 3 * k] = (200, 30, 90)
    img += rng.normal(0, 4, img.shape)
    frames.append(np.clip(np.rint(img), 0, 255).astype(np.uint8))
ok = True
for cfg, kw in [(dict(target_width=101, target_height=52, mode="buffered"), {}),
                (dict(target_width=120, mode="buffered", reaverage_energy=True), {}),
                (dict(target_width=140, mode="raw"), {})]:
    out, m = P.retarget_video(frames, P.RetargetConfig(**cfg))
    ref = O.retarget_video(frames, **cfg)
    ok &= m.dp_passes == ref.dp_passes and all(np.array_equal(a, b) for a, b in zip(out, ref.frames))
res = P.retarget_videos([frames, frames[::-1]], P.RetargetConfig(target_width=101, mode="buffered"))
for (o, m), fr in zip(res, (frames, frames[::-1])):
    ref = O.retarget_video(fr, target_width=101)
    ok &= m.dp_passes == ref.dp_passes and all(np.array_equal(a, b) for a, b in zip(o, ref.frames))
print("CHECKED CASE", "OK" if ok else "MISMATCH", os.environ.get("SCPL_CARVE_KC", "auto"),
      "host-loops" if os.environ.get("SCPL_HOST_LOOPS") else "graphs", flush=True)
sys.exit(0 if ok else 1)
