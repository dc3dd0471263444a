"""Golden outputs of the REFERENCE for non-default energy weights (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_weights_golden.py

Runs vidcarve.retarget_video (buffered) on tests/cases.weights_clip for every pair of
cases.WEIGHT_CASES and writes weights.json: run boundaries (recorded by wrapping
pipeline._process_run at runtime; the reference source is not modified), dp_passes and the SHA-256 of every
output frame.  Only the JSON travels to the GPU box."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/

import vidcarve  # noqa: E402  (reference, from /root/reference/pkg/src)
from vidcarve import pipeline as vp  # noqa: E402

import cases  # noqa: E402

out = {}
for wm, wg in cases.WEIGHT_CASES:
    frames, tw = cases.weights_clip(wm)
    cfg = vidcarve.RetargetConfig(target_width=tw, mode="buffered", w_motion=wm, w_grad=wg)
    lens = []
    orig = vp._process_run

    def rec(run, *a, **k):  # run lengths, recorded by wrapping the reference's _process_run at runtime
        lens.append(len(run))
        return orig(run, *a, **k)

    vp._process_run = rec
    try:
        res, m = vp.retarget_video(frames, cfg)
    finally:
        vp._process_run = orig
    starts = [sum(lens[:i]) for i in range(len(lens))]
    out[f"{wm}/{wg}"] = {"runs": [[int(s), int(n)] for s, n in zip(starts, lens)], "dp_passes": int(m.dp_passes),
                         "frames": [cases.sha(f) for f in res]}
with open(os.path.join(HERE, "weights.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print("wrote weights.json", {k: (len(v["runs"]), v["dp_passes"]) for k, v in out.items()})
