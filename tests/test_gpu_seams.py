"""GPU parity at config scale: every batch the carve chose (seam columns, costs, offsets, parent
labels) on the BASELINE config clips, the 64-clip C4 batch path, and the drop-in API's edge
cases (custom energy functions, dtypes, mixed gray/RGB clips, threads).

The goldens were produced by running the reference itself (tests/golden/make_golden.py); the
seam records come from libscpl's seam-dump parity mode (include/scpl.h, scpl_video_result).
"""
import glob
import json
import os
import threading

import numpy as np
import pytest

from cases import fhex, sha

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    import paper_1903_03180_b200 as P
    return P


def _golden(pattern):
    return sorted(glob.glob(os.path.join(GOLD, pattern)))


def _c4_goldens():
    def idx(p):
        return int(os.path.basename(p)[len("C4_clip"):-len(".json")])
    return sorted((p for p in _golden("C4_clip*.json") if os.path.basename(p)[7:-5].isdigit()), key=idx)


def _dump_rec(b, with_labels):
    """A seam-dump batch in make_golden.py's batch_record format (batching.py:20-36 fields)."""
    offs = b["offsets"].astype(np.int32) if len(b["cols"]) else np.zeros((0, 0), np.int32)
    r = {"b": len(b["cols"]), "cols": [int(c) for c in b["cols"]], "costs": [fhex(c) for c in b["costs"]],
         "offsets_sha": sha(offs), "source_width": int(b["source_width"])}
    if with_labels:
        r["labels_sha"] = sha(b["labels"].astype(np.int64))
    return r


def _axes(g):
    """The carved axes of a run in the reference's phase order (pipeline.py:192-193, 258-262)."""
    h, w = g["shape"][:2]
    order = (1, 0) if g.get("height_first") else (0, 1)
    tw, th = g["target_width"] or w, g["target_height"] or h
    return [ax for ax in order if (ax == 0 and tw < w) or (ax == 1 and th < h)]


def _check_seams(g, seams):
    """Every batch of every run and axis equals the reference's."""
    axes = _axes(g)
    assert len(g["batches"]) == len(g["runs"])
    bad = []
    for r, per_run in enumerate(g["batches"]):
        assert len(per_run) == len(axes), (r, len(per_run), axes)
        for ax, want in zip(axes, per_run):
            got = seams[(r, ax)]
            labels = bool(want) and "labels_sha" in want[0]
            have = [_dump_rec(b, labels) for b in got]
            if have != want:
                k = next((i for i, (a, b) in enumerate(zip(have, want)) if a != b), min(len(have), len(want)))
                bad.append((r, ax, k, len(have), len(want)))
    assert not bad, f"{len(bad)} (run, axis) records differ, first {bad[:3]}"
    assert len(seams) == len(g["runs"]) * len(axes)


@pytest.mark.parametrize("path", [p for p in _golden("C[1235].json")] + _c4_goldens()[:2])
def test_config_seams_golden(P, path):
    """Seam columns, costs, offsets and parent labels of every pass of every run (the
    reference's batch_carve decisions, batching.py:39-73 / seams.py:68-81), bit-exact, on the
    full BASELINE config clips -- through the video path itself (seam-dump mode)."""
    import torch
    from paper_1903_03180_b200.synth import config_clip
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    out, m = P.retarget_video_tensor(torch.from_numpy(clip).cuda(),
                                     P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"),
                                     seam_dump=True)
    assert [list(r) for r in m.runs] == g["runs"]
    assert m.dp_passes == g["dp_passes"]
    _check_seams(g, m.seams)
    host = out.cpu().numpy()
    bad = [t for t in range(host.shape[0]) if sha(host[t]) != g["frames_sha"][t]]
    assert not bad, f"{len(bad)} frames differ, first {bad[:5]}"


def test_c4_batch_all_clips_golden(P):
    """BASELINE C4 as specified: the 64 independent clips in ONE batch call (scpl_retarget_batch,
    every clip's scan in flight at once, runs of all clips sharing carve groups), each clip's
    runs, dp_passes, every output frame and every seam record equal to the reference's."""
    import torch
    from paper_1903_03180_b200.synth import config_clip
    paths = _c4_goldens()
    assert len(paths) >= 16, "C4 goldens missing"
    gs = [json.load(open(p)) for p in paths]
    clips = []
    for g in gs:
        clip, tw, th = config_clip("C4", clip=g["clip"])
        clips.append(torch.from_numpy(clip).cuda())
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
    res = P.retarget_videos(clips, cfg, seam_dump=True)
    assert len(res) == len(gs)
    for g, (out, m) in zip(gs, res):
        assert [list(r) for r in m.runs] == g["runs"], g["clip"]
        assert m.dp_passes == g["dp_passes"], g["clip"]
        _check_seams(g, m.seams)
        host = out.cpu().numpy()
        bad = [t for t in range(host.shape[0]) if sha(host[t]) != g["frames_sha"][t]]
        assert not bad, f"clip {g['clip']}: {len(bad)} frames differ"
    # the same batch without the dump (the bench path) gives the same frames
    res2 = P.retarget_videos(clips, cfg)
    for (a, _), (b, m2), g in zip(res, res2, gs):
        assert torch.equal(a, b) and m2.dp_passes == g["dp_passes"]


def test_c4_batch_host_buffers(P):
    """The batch path with pinned HOST clips (chunked H2D, per-run D2H) and frame lists."""
    import torch
    from paper_1903_03180_b200.synth import config_clip
    paths = _c4_goldens()[:6]
    gs = [json.load(open(p)) for p in paths]
    clips = [torch.from_numpy(config_clip("C4", clip=g["clip"])[0]).pin_memory() for g in gs]
    tw = gs[0]["target_width"]
    res = P.retarget_videos(clips, P.RetargetConfig(target_width=tw, mode="buffered"))
    for g, (out, m) in zip(gs, res):
        assert not out.is_cuda and out.is_pinned()
        assert [list(r) for r in m.runs] == g["runs"] and m.dp_passes == g["dp_passes"]
        host = out.numpy()
        assert all(sha(host[t]) == g["frames_sha"][t] for t in range(host.shape[0])), g["clip"]
    lists = [list(c[:20].numpy()) for c in clips[:3]]
    res3 = P.retarget_videos(lists, P.RetargetConfig(target_width=tw, mode="buffered"))
    for fr, (out, m) in zip(lists, res3):
        ref, m1 = P.retarget_video(fr, P.RetargetConfig(target_width=tw, mode="buffered"))
        assert m.runs == m1.runs and m.dp_passes == m1.dp_passes
        assert all(np.array_equal(a, b) for a, b in zip(out, ref))


def test_batch_matches_single_clip_calls(P):
    """A batch of small mixed-content clips (both axes, reaverage off) equals one call per clip."""
    import torch
    rng = np.random.default_rng(91)
    clips = []
    for k in range(5):
        c = rng.integers(0, 256, size=(23, 40, 56, 3), dtype=np.uint8)
        c[5:15] = c[5]  # a static stretch: a long run
        clips.append(torch.from_numpy(c).cuda())
    cfg = P.RetargetConfig(target_width=41, target_height=33, mode="buffered")
    res = P.retarget_videos(clips, cfg, seam_dump=True)
    for c, (out, m) in zip(clips, res):
        one, m1 = P.retarget_video_tensor(c, cfg, seam_dump=True)
        assert torch.equal(out, one) and m.runs == m1.runs and m.dp_passes == m1.dp_passes
        assert m.seams.keys() == m1.seams.keys()
        for key in m.seams:
            for a, b in zip(m.seams[key], m1.seams[key]):
                assert all(np.array_equal(a[f], b[f]) for f in ("cols", "costs", "offsets", "labels"))


# ------------------------------------------------------------------ buffer scan
def test_buffer_stream_asde_golden(P):
    """Every candidate ASDE the buffer computes (buffering.py:116-118, _asde_from_sums with
    numpy's pairwise mean) equals the reference's bit for bit (hex), not just the decisions."""
    import cases
    small = json.load(open(os.path.join(GOLD, "small.json")))
    for s in cases.STREAM_SEEDS:
        maps = cases.stream_case(s)
        want = small["stream"][str(s)]["asde"]
        buf = P.SpatioTemporalBuffer(policy=P.BufferPolicy())
        got = []
        for m in maps:
            had = len(buf) > 0
            buf.push(np.zeros(m.shape, np.uint8), m)
            if had:
                got.append(fhex(buf.last_candidate_asde))
        assert got == want, s


def _tie_clip(h=60, w=90, T=9):
    """Gray frames whose buffer statistics land EXACTLY on the threshold: flat frames (zero
    gradient) with a brightness step of 85 give e = fl(0.6*85) = 51, std = 25.5 at every pixel,
    so the 2-frame ASDE is 25.5 == phi(2) (buffering.py:119 accepts on <=).  The screened scan
    cannot settle such a window and must fall back to the exact evaluation."""
    lv = [0, 85, 85, 0, 0, 85, 170, 170, 85][:T]
    return [np.full((h, w), v, np.uint8) for v in lv]


def test_scan_fallback_fires_naturally(P):
    from oracle import scpl_oracle as O
    from paper_1903_03180_b200 import pipeline
    frames = _tie_clip()
    cfg = P.RetargetConfig(target_width=70, mode="buffered")
    out, m = P.retarget_video(frames, cfg)
    ph = dict(pipeline.last_phase_ms)
    ref = O.retarget_video(frames, target_width=70)
    assert [tuple(r) for r in m.runs] == [tuple(r) for r in ref.runs]
    assert m.dp_passes == ref.dp_passes
    assert all(np.array_equal(a, b) for a, b in zip(out, ref.frames))
    assert ph["scan_fallbacks"] >= 1, ph  # the exact re-run was needed (and agreed)
    assert abs(O.threshold(2, O.BufferPolicy()) - 25.5) < 1e-12


# ------------------------------------------------------------------ drop-in API edge cases
def test_scan_runs_and_given_runs(P):
    """scan_runs (scan only) gives the reference's runs; carving a subset of them (runs=...)
    writes exactly those runs' frames, equal to the full call's."""
    import torch
    from paper_1903_03180_b200.synth import config_clip
    g = json.load(open(_c4_goldens()[0]))
    clip, tw, th = config_clip("C4", clip=g["clip"])
    dev = torch.from_numpy(clip).cuda()
    cfg = P.RetargetConfig(target_width=tw, mode="buffered")
    runs = P.scan_runs(dev, cfg)
    assert [list(r) for r in runs] == g["runs"]
    sub = [runs[0], runs[2]]
    out = torch.zeros((clip.shape[0],) + tuple(g["out_shape"]), dtype=torch.uint8, device="cuda")
    res, m = P.retarget_video_tensor(dev, cfg, out=out, runs=sub)
    host = res.cpu().numpy()
    for s, n in sub:
        assert all(sha(host[t]) == g["frames_sha"][t] for t in range(s, s + n))
    s1, n1 = runs[1]
    assert not host[s1:s1 + n1].any()  # untouched


def test_custom_energy_fn_matches_reference_loop(P):
    """batch_carve(energy_fn=...) (batching.py:118-146): the caller's energy on each carved
    frame, DP / labels / select / removal on the GPU; compared with the same loop over the
    oracle's primitives."""
    from oracle import scpl_oracle as O
    rng = np.random.default_rng(17)
    frame = rng.integers(0, 256, size=(30, 45, 3), dtype=np.uint8)

    def efn(f):  # a user energy: squared luma gradient along x, float
        lum = O.to_luma(f).astype(np.float64)
        return np.abs(np.diff(lum, axis=1, append=lum[:, -1:])) ** 1.5

    got, batches = P.batch_carve(frame, 31, energy_fn=efn)
    cur, want = frame, []
    while cur.shape[1] > 31:
        ce, back = O.cumulative_energy(efn(cur))
        b = O.select_batch(ce, back, O.label_parents(back), k=cur.shape[1] - 31)
        cur = O.remove_batch(cur, b)
        want.append(b)
    assert np.array_equal(got, cur)
    assert [len(b) for b in batches] == [len(b) for b in want]
    for x, y in zip(batches, want):
        assert [int(s.offsets[-1]) for s in x] == [int(c) for c in y.cols]
        assert [s.cost for s in x] == [float(c) for c in y.costs]


def test_remove_batch_keeps_dtype(P):
    """remove_batch is dtype-generic like the reference (batching.py:100-107)."""
    from oracle import scpl_oracle as O
    t = P.cumulative_energy(np.full((3, 3), 5.0))
    b = P.select_batch(t, P.label_parents(t))
    for arr in (np.array([[10, 20, 30]] * 3), np.arange(27, dtype=np.float64).reshape(3, 3, 3) / 7,
                np.arange(9, dtype=np.int16).reshape(3, 3)):
        got = P.remove_batch(arr, b)
        keep = np.ones(arr.shape[:2], bool)
        for s in b:
            keep[np.arange(3), s.offsets] = False
        want = arr[keep].reshape((3, 3 - len(b)) + arr.shape[2:])
        assert got.dtype == arr.dtype and np.array_equal(got, want)
    assert O is not None


def test_video_dtypes(P):
    """uint8 tensors only on the tensor path; integer frame lists in 0..255 convert exactly and
    keep their dtype; floats / out-of-range values are rejected (never wrapped)."""
    import torch
    rng = np.random.default_rng(3)
    frames = [rng.integers(0, 256, size=(12, 16, 3), dtype=np.uint8) for _ in range(4)]
    cfg = P.RetargetConfig(target_width=11, mode="buffered")
    ref, m0 = P.retarget_video(frames, cfg)
    got, m1 = P.retarget_video([f.astype(np.int64) for f in frames], cfg)
    assert all(g.dtype == np.int64 and np.array_equal(g, r) for g, r in zip(got, ref))
    with pytest.raises(ValueError):
        P.retarget_video([f.astype(np.int64) + 300 for f in frames], cfg)
    with pytest.raises(TypeError):
        P.retarget_video_tensor(torch.from_numpy(np.stack(frames)).float().cuda(), cfg)


def test_mixed_gray_rgb_clip(P):
    """A clip mixing gray and RGB frames (the reference takes each frame's layout on its own,
    energy.py:30-37): same runs, passes and pixels as the oracle; each output keeps its layout."""
    from oracle import scpl_oracle as O
    rng = np.random.default_rng(8)
    frames = []
    for t in range(7):
        f = rng.integers(0, 256, size=(20, 30, 3), dtype=np.uint8)
        frames.append(O.to_luma(f) if t % 3 == 1 else f)
    cfg = P.RetargetConfig(target_width=22, target_height=17, mode="buffered")
    out, m = P.retarget_video(frames, cfg)
    ref = O.retarget_video(frames, target_width=22, target_height=17, literal_replay=True)
    assert [tuple(r) for r in m.runs] == [tuple(r) for r in ref.runs] and m.dp_passes == ref.dp_passes
    for a, b in zip(out, ref.frames):
        assert a.shape == b.shape and np.array_equal(a, b)


def test_threads_share_a_context(P):
    """Calls on one device's context from several Python threads are serialised by the
    library (one call at a time per context); every thread gets its own correct result."""
    import torch
    from paper_1903_03180_b200.synth import config_clip
    g = json.load(open(_golden("C1.json")[0]))
    clip, tw, th = config_clip("C1")
    dev = torch.from_numpy(clip).cuda()
    cfg = P.RetargetConfig(target_width=tw, mode="buffered")
    errors, outs = [], {}

    def work(k):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                o, m = P.retarget_video_tensor(dev, cfg)
                torch.cuda.current_stream().synchronize()
                outs[k] = (o.cpu().numpy(), m)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for o, m in outs.values():
        assert m.dp_passes == g["dp_passes"]
        assert [sha(o[t]) for t in range(o.shape[0])] == g["frames_sha"]


@pytest.mark.skipif("not __import__('torch').cuda.device_count() > 1")
def test_two_devices_one_process(P):
    """One process driving two GPUs: per-device kernel attributes and the clip's own stream."""
    import torch
    from paper_1903_03180_b200.synth import config_clip
    g = json.load(open(_golden("C1.json")[0]))
    clip, tw, th = config_clip("C1")
    cfg = P.RetargetConfig(target_width=tw, mode="buffered")
    for d in (1, 0):
        o, m = P.retarget_video_tensor(torch.from_numpy(clip).to(f"cuda:{d}"), cfg)
        assert o.device.index == d and m.dp_passes == g["dp_passes"]
        o = o.cpu().numpy()
        assert [sha(o[t]) for t in range(o.shape[0])] == g["frames_sha"]


@pytest.mark.parametrize("world", [1, 3])
def test_host_split_into_shared_buffer(P, world):
    """One HOST clip split by runs, outputs gathered on the host (sharding.py): each rank's
    host-buffer call carves its LPT share of the runs (scanned once) and its per-run D2H copies
    land in one shared, pinned /dev/shm buffer.  The ranks run one after another here (they never
    wait on each other); the merged buffer is the reference's clip."""
    import uuid
    import torch
    from paper_1903_03180_b200 import sharding
    from paper_1903_03180_b200.pipeline import _run_device
    from paper_1903_03180_b200.synth import config_clip
    g = json.load(open(_c4_goldens()[1]))
    clip, tw, th = config_clip("C4", clip=g["clip"])
    host = torch.from_numpy(clip).pin_memory()
    cfg = P.RetargetConfig(target_width=tw, mode="buffered")
    name = f"scpl_gpu_test_{uuid.uuid4().hex[:8]}"
    out = sharding.shared_host_buffer(name, (clip.shape[0],) + tuple(g["out_shape"]))
    try:
        if world == 1:
            res, m = sharding.retarget_clip_sharded_host(host, cfg, out)
            assert m.dp_passes == g["dp_passes"] and [list(r) for r in m.runs] == g["runs"]
        else:
            runs = P.scan_runs(host, cfg)
            owners = sharding.lpt_owners(runs, world)
            dp = 0
            for rank in range(world):
                mine = [r for r, o in zip(runs, owners) if o == rank]
                _, d, _, _ = _run_device(host, cfg, tw, clip.shape[1], out=out, runs_in=mine)
                dp += d
            assert dp == g["dp_passes"]
        o = out.numpy()
        bad = [t for t in range(o.shape[0]) if sha(o[t]) != g["frames_sha"][t]]
        assert not bad, f"{len(bad)} frames differ"
    finally:
        sharding.release_host_buffer(out, name)
