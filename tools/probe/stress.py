"""Repeat the config clips many times: the first repetition is checked against the reference's
golden hashes, every later one against the first on the device (catches rare races in the
carve's cluster exchange, the scan's screening or the batch scheduler).

    python tools/probe/stress.py [reps] [--batch N]   (--batch: also N C4 clips per batch call)
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("reps", type=int, nargs="?", default=10)
ap.add_argument("--batch", type=int, default=16)
a = ap.parse_args()
G = os.path.join(ROOT, "tests", "golden")


def golden_ok(g, out, m):
    host = out.cpu().numpy()
    return ([list(r) for r in m.runs] == g["runs"] and m.dp_passes == g["dp_passes"]
            and all(hashlib.sha256(host[t].tobytes()).hexdigest() == g["frames_sha"][t] for t in range(host.shape[0])))


bad_total = 0
paths = [os.path.join(G, f) for f in ("C1.json", "C2.json", "C3.json", "C5.json", "C1_rea.json", "C2_f62_rea.json")]
paths += [os.path.join(G, f"C4_clip{i}.json") for i in range(4)]
for path in paths:
    if not os.path.exists(path):
        continue
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    dev = torch.from_numpy(clip).cuda()
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered",
                           reaverage_energy=g.get("reaverage", False))
    first, m0 = P.retarget_video_tensor(dev, cfg)
    bad = 0 if golden_ok(g, first, m0) else 1
    for _ in range(a.reps - 1):
        out, m = P.retarget_video_tensor(dev, cfg)
        bad += not (torch.equal(out, first) and m.runs == m0.runs and m.dp_passes == m0.dp_passes)
    bad_total += bad
    print(f"{os.path.basename(path)}: {a.reps - bad}/{a.reps} identical to the reference", flush=True)
if a.batch:
    gs = [json.load(open(p)) for p in sorted(glob.glob(os.path.join(G, "C4_clip*.json")))[:a.batch]]
    devs = [torch.from_numpy(config_clip("C4", clip=g["clip"])[0]).cuda() for g in gs]
    cfg = P.RetargetConfig(target_width=gs[0]["target_width"], mode="buffered")
    first = P.retarget_videos(devs, cfg)
    bad = sum(not golden_ok(g, o, m) for g, (o, m) in zip(gs, first))
    for _ in range(a.reps - 1):
        res = P.retarget_videos(devs, cfg)
        bad += sum(not (torch.equal(o, o0) and m.dp_passes == m0.dp_passes) for (o, m), (o0, m0) in zip(res, first))
    bad_total += bad
    print(f"C4 batch of {len(gs)} clips: {a.reps * len(gs) - bad}/{a.reps * len(gs)} clip results identical", flush=True)
print("ALL OK" if bad_total == 0 else f"MISMATCHES: {bad_total}")
