"""Repeat the config clips many times and check every output frame against the reference's
golden hashes (catches rare races in the carve's cluster exchange or the scan's screening)."""
import glob
import hashlib
import json
import os
import sys

import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bad_total = 0
for path in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "C*.json"))):
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    dev = torch.from_numpy(clip).cuda()
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered",
                           reaverage_energy=g.get("reaverage", False))
    bad = 0
    for _ in range(reps):
        out, m = P.retarget_video_tensor(dev, cfg)
        host = out.cpu().numpy()
        ok = [list(r) for r in m.runs] == g["runs"] and m.dp_passes == g["dp_passes"]
        ok = ok and all(hashlib.sha256(host[t].tobytes()).hexdigest() == g["frames_sha"][t]
                        for t in range(host.shape[0]))
        bad += not ok
    bad_total += bad
    print(f"{os.path.basename(path)}: {reps - bad}/{reps} identical to the reference", flush=True)
print("ALL OK" if bad_total == 0 else f"MISMATCHES: {bad_total}")
