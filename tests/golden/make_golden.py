"""Generate the golden fixtures by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py small
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py C1 [C2 ...] [--frames N]

`small` writes small.json (energy / DP / labels / batches / buffer / pipeline
outputs for the seeded cases in tests/cases.py) and luma_table.sha256 (the
reference's to_luma over all 2^24 RGB triples). `Cn` runs
vidcarve.retarget_video on the seeded synthetic clip of that BASELINE config
(paper_1903_03180_b200.synth) and records run boundaries, dp_passes, every
batch (size, last-row columns, costs, offsets hash) and every output frame's
SHA-256, plus the SHA-256 of every pass's parent labels (int64). Recording
wraps three reference functions at runtime (pipeline.batch_carve,
pipeline._process_run, batching.label_parents); the reference source is not
modified. /root/reference does not exist on the GPU box: only the JSON
outputs travel.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root
sys.path.insert(0, os.path.dirname(HERE))                   # tests/

import vidcarve  # noqa: E402  (reference, from /root/reference/pkg/src)
from vidcarve import pipeline as vp  # noqa: E402
from vidcarve.batching import batch_carve, label_parents, select_batch  # noqa: E402
from vidcarve.buffering import BufferPolicy, SpatioTemporalBuffer, _asde_from_sums  # noqa: E402
from vidcarve.energy import gradient_energy, motion_energy, to_luma  # noqa: E402
from vidcarve.seams import cumulative_energy  # noqa: E402

import cases  # noqa: E402
from cases import fhex, sha  # noqa: E402


def batch_record(b):
    offs = np.stack([s.offsets for s in b.seams], axis=1).astype(np.int32) if len(b) else np.zeros((0, 0), np.int32)
    return {
        "b": len(b),
        "cols": [int(s.offsets[-1]) for s in b.seams],
        "costs": [fhex(s.cost) for s in b.seams],
        "offsets_sha": sha(offs),
        "source_width": b.source_width,
    }


def small():
    out = {}
    lt = cases.luma_table_frame()
    with open(os.path.join(HERE, "luma_table.sha256"), "w") as f:
        f.write(sha(to_luma(lt)) + "\n")

    en = {}
    for s in cases.ENERGY_SEEDS:
        curr, prev = cases.energy_case(s)
        en[str(s)] = {
            "luma": sha(to_luma(curr)),
            "grad": sha(gradient_energy(to_luma(curr))),
            "motion": sha(motion_energy(curr, prev)),
            "motion_first": sha(motion_energy(curr, None)),
            "motion_w": sha(motion_energy(curr, prev, 0.3, 0.7)),
        }
    out["energy"] = en

    dp = {}
    for s in cases.MAP_SEEDS:
        m = cases.map_case(s)
        t = cumulative_energy(m)
        lab = label_parents(t)
        full = select_batch(t, lab)
        k = max(1, len(full) // 2)
        dp[str(s)] = {
            "ce": sha(t.ce), "back": sha(t.back), "labels": [int(x) for x in lab],
            "batch": batch_record(full), "batch_k": batch_record(select_batch(t, lab, k=k)), "k": k,
        }
    out["dp"] = dp

    cv = {}
    for s in cases.CARVE_SEEDS:
        frame, target, energy = cases.carve_case(s)
        carved, batches = batch_carve(frame, target, energy=energy)
        cv[str(s)] = {"carved": sha(carved), "batches": [batch_record(b) for b in batches]}
    out["carve"] = cv

    st = {}
    for s in cases.STREAM_SEEDS:
        maps = cases.stream_case(s)
        buf = SpatioTemporalBuffer(policy=BufferPolicy())
        runs, asdes = [], []
        for m in maps:
            if len(buf):  # record the candidate ASDE the push will compute (buffering.py:116-118)
                n = len(buf) + 1
                asdes.append(fhex(_asde_from_sums(buf._sum + m, buf._sum_sq + m * m, n)))
            r = buf.push(np.zeros(m.shape, np.uint8), m)
            if r is not None:
                runs.append(len(r))
        runs.append(len(buf.flush()))
        st[str(s)] = {"runs": runs, "asde": asdes}
    out["stream"] = st

    cl = {}
    for name, (ck, cfg) in cases.CLIP_CASES.items():
        frames = cases.small_clip(**ck)
        cfg = dict(cfg)
        pol = BufferPolicy(**{k: cfg.pop(k) for k in ("alpha", "max_len") if k in cfg})
        res, m = vidcarve.retarget_video([f.copy() for f in frames], vidcarve.RetargetConfig(policy=pol, **cfg))
        cl[name] = {"frames": [sha(f) for f in res], "shapes": [list(f.shape) for f in res],
                    "dp_passes": m.dp_passes}
    out["clips"] = cl

    import io
    from vidcarve import bench as vb, media as vm
    md = {}
    for name, data in cases.media_streams():
        try:
            fr = list(vm.read_frames(io.BytesIO(data)))
            md[name] = {"frames": [sha(f) for f in fr], "shapes": [list(f.shape) for f in fr]}
            buf = io.BytesIO()
            vm.write_frames(buf, fr)
            md[name]["written"] = sha(np.frombuffer(buf.getvalue(), np.uint8)) if fr else None
        except Exception as e:  # noqa: BLE001 -- the reference's exception type and message are the fixture
            md[name] = {"error": type(e).__name__, "message": str(e)}
    out["media"] = md
    jt = {}
    for name, (ck, win) in cases.JITTER_CASES.items():
        frames = cases.small_clip(**ck)
        jt[name] = fhex(vb.jitter(frames, window=win).value)
    out["jitter"] = jt
    cb = {}
    for kind in vb.SYNTHETIC_KINDS:
        frames = vb.generate(vb.SyntheticSpec(kind=kind, width=40, height=30, frames=9, seed=2))
        res = vb.compare(frames, {m: vidcarve.RetargetConfig(target_width=30, mode=m) for m in vidcarve.MODES})
        cb[kind] = {m: {"dp_passes": r.dp_passes, "frames_out": r.frames_out, "jitter": f"{r.jitter:.6f}"}
                    for m, r in res.items()}
    out["cli_bench"] = cb
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)


def config(name: str, frames: int | None, clip: int, reaverage: bool = False):
    from paper_1903_03180_b200.synth import config_clip
    arr, tw, th = config_clip(name, frames=frames, clip=clip)
    import vidcarve.batching as vb_mod
    runs, batches, labels = [], [], []
    orig_carve, orig_process, orig_labels = vp.batch_carve, vp._process_run, vb_mod.label_parents

    def rec_labels(tables):  # batch_carve's per-pass parent labels (batching.py:148)
        lab = orig_labels(tables)
        labels.append(sha(np.asarray(lab, dtype=np.int64)))
        return lab

    def rec_carve(*a, **k):
        del labels[:]
        carved, bs = orig_carve(*a, **k)
        assert len(labels) == len(bs)
        recs = [batch_record(b) for b in bs]
        for r, lab in zip(recs, labels):
            r["labels_sha"] = lab
        batches[-1].append(recs)
        return carved, bs

    def rec_process(run, *a, **k):
        runs.append(len(run))
        batches.append([])
        return orig_process(run, *a, **k)

    vp.batch_carve, vp._process_run, vb_mod.label_parents = rec_carve, rec_process, rec_labels
    try:
        t0 = time.time()
        out, m = vp.retarget_video(list(arr), vp.RetargetConfig(target_width=tw, target_height=th, mode="buffered",
                                                                reaverage_energy=reaverage))
        wall = time.time() - t0
    finally:
        vp.batch_carve, vp._process_run, vb_mod.label_parents = orig_carve, orig_process, orig_labels
    starts = np.concatenate([[0], np.cumsum(runs)[:-1]]).tolist()
    rec = {
        "config": name, "clip": clip, "frames": int(arr.shape[0]), "shape": list(arr.shape[1:]),
        "target_width": tw, "target_height": th,
        "runs": [[int(s), int(n)] for s, n in zip(starts, runs)],
        "dp_passes": m.dp_passes, "batches": batches,
        "frames_sha": [sha(f) for f in out], "out_shape": list(out[0].shape),
        "reference_wall_s": wall, "reaverage": reaverage,
    }
    suffix = f"_clip{clip}" if name == "C4" else ""
    suffix += f"_f{frames}" if frames is not None else ""
    suffix += "_rea" if reaverage else ""
    with open(os.path.join(HERE, f"{name}{suffix}.json"), "w") as f:
        json.dump(rec, f, indent=0)
    print(name, suffix, "runs", runs, "dp", m.dp_passes, f"{wall:.1f}s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="+")
    ap.add_argument("--frames", type=int, default=None)
    ap.add_argument("--clip", type=int, default=0)
    ap.add_argument("--reaverage", action="store_true")
    a = ap.parse_args()
    for w in a.what:
        if w == "small":
            small()
        else:
            config(w, a.frames, a.clip, a.reaverage)
