"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden vectors
and the CPU oracle. Bit-exact everywhere (integer/byte outputs and float64 maps alike).
"""
import glob
import json
import os

import numpy as np
import pytest

import cases
from cases import fhex, sha

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def small():
    with open(os.path.join(GOLD, "small.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def P():
    import paper_1903_03180_b200 as P
    return P


def _batch_rec(b):
    offs = np.stack([s.offsets for s in b.seams], axis=1).astype(np.int32) if len(b) else np.zeros((0, 0), np.int32)
    return {"b": len(b), "cols": [int(s.offsets[-1]) for s in b.seams], "costs": [fhex(s.cost) for s in b.seams],
            "offsets_sha": sha(offs), "source_width": b.source_width}


# ------------------------------------------------------------------ energy
def test_luma_all_2pow24_triples(P):
    lt = cases.luma_table_frame()
    want = open(os.path.join(GOLD, "luma_table.sha256")).read().strip()
    assert sha(P.to_luma(lt)) == want


def test_energy_golden(P, small):
    for s in cases.ENERGY_SEEDS:
        curr, prev = cases.energy_case(s)
        g = small["energy"][str(s)]
        assert sha(P.to_luma(curr)) == g["luma"], s
        assert sha(P.gradient_energy(P.to_luma(curr))) == g["grad"], s
        assert sha(P.motion_energy(curr, prev)) == g["motion"], s
        assert sha(P.motion_energy(curr, None)) == g["motion_first"], s
        assert sha(P.motion_energy(curr, prev, 0.3, 0.7)) == g["motion_w"], s


def test_energy_known_answers(P):
    assert (P.to_luma(np.full((4, 5, 3), 100, np.uint8)) == 100).all()
    red = np.zeros((3, 3, 3), np.uint8)
    red[..., 0] = 255
    assert P.to_luma(red)[0, 0] == 76
    assert (P.motion_energy(np.full((5, 5), 60, np.uint8), np.full((5, 5), 50, np.uint8)) == 6.0).all()
    f = np.zeros((6, 6), np.uint8)
    f[:, 3:] = 255
    assert sorted(set(np.nonzero(P.gradient_energy(f))[1].tolist())) == [2, 3]


def test_energy_codes_random_frames_vs_oracle(P):
    from oracle import scpl_oracle as O
    rng = np.random.default_rng(5)
    for h, w in [(3, 3), (7, 13), (64, 80), (241, 333), (1080, 1920)]:
        a = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        b = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        assert np.array_equal(P.motion_energy(a, b), O.motion_energy(a, b)), (h, w)
        assert np.array_equal(P.motion_energy(a, None), O.motion_energy(a, None)), (h, w)


def test_energy_codes_clip_tiles_vs_oracle(P):
    """RGB clips through the tiled codes kernel (TMA rows: W*3 % 16 == 0, and plain rows),
    frame 0 pure gradient, then motion against the previous frame; also a chunk whose
    previous frame comes from a separate pointer."""
    import torch
    from oracle import scpl_oracle as O
    from paper_1903_03180_b200 import _lib
    lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
    rng = np.random.default_rng(6)
    for T, h, w in [(7, 70, 272), (5, 33, 130), (3, 161, 400), (4, 32, 128)]:
        clip = rng.integers(0, 256, size=(T, h, w, 3), dtype=np.uint8)
        clip[2] = clip[1] // 2 + 7  # some structure between frames
        dev = torch.from_numpy(clip).cuda()
        codes = torch.empty((T, h, w), dtype=torch.int16, device="cuda")
        _lib.check(lib.scpl_energy_codes(cx, dev.data_ptr(), None, T, h, w, 3, codes.data_ptr(), st))
        out = torch.empty((T, h, w), dtype=torch.float64, device="cuda")
        _lib.check(lib.scpl_decode_energy(cx, codes.data_ptr(), T, h, w, 1, 0.6, 0.4, out.data_ptr(), st))
        got = out.cpu().numpy()
        for t in range(T):
            ref = O.motion_energy(clip[t], clip[t - 1] if t else None)
            assert np.array_equal(got[t], ref), (T, h, w, t)
        # frames 2.. with the previous frame given separately
        sub = dev[2:].contiguous()
        c2 = torch.empty((T - 2, h, w), dtype=torch.int16, device="cuda")
        _lib.check(lib.scpl_energy_codes(cx, sub.data_ptr(), dev[1].data_ptr(), T - 2, h, w, 3, c2.data_ptr(), st))
        assert torch.equal(c2, codes[2:]), (T, h, w)


# ------------------------------------------------------------------ DP / labels / batches
def test_dp_labels_batches_golden(P, small):
    for s in cases.MAP_SEEDS:
        m = cases.map_case(s)
        g = small["dp"][str(s)]
        t = P.cumulative_energy(m)
        assert sha(t.ce) == g["ce"] and sha(t.back) == g["back"], s
        lab = P.label_parents(t)
        assert lab.tolist() == g["labels"], s
        assert _batch_rec(P.select_batch(t, lab)) == g["batch"], s
        assert _batch_rec(P.select_batch(t, lab, k=g["k"])) == g["batch_k"], s


def test_known_answer_tables(P):
    t = P.cumulative_energy(np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]], dtype=np.float64))
    assert t.ce.tolist() == [[1, 2, 3], [5, 6, 8], [12, 13, 15]]
    assert P.min_seam(t).offsets.tolist() == [0, 0, 0]
    t2 = P.cumulative_energy(np.full((2, 3), 5.0))
    lab = P.label_parents(t2)
    assert lab.tolist() == [0, 0, 1]
    b = P.select_batch(t2, lab)
    assert [s.offsets.tolist() for s in b] == [[0, 0], [1, 2]]
    assert P.remove_batch(np.array([[1, 2, 3], [4, 5, 6]], np.uint8), b).tolist() == [[3], [5]]


def test_batch_carve_golden(P, small):
    for s in cases.CARVE_SEEDS:
        frame, target, energy = cases.carve_case(s)
        carved, batches = P.batch_carve(frame, target, energy=energy)
        g = small["carve"][str(s)]
        assert [_batch_rec(b) for b in batches] == g["batches"], s
        assert sha(carved) == g["carved"], s


def test_batch_carve_zero_band(P):
    energy = np.full((2, 12), 100.0)
    energy[:, 5:8] = 0.0
    out, batches = P.batch_carve(np.zeros((2, 12), np.uint8), 10, energy=energy)
    assert out.shape == (2, 10) and len(batches[0]) == 2
    for seam in batches[0]:
        assert seam.cost == 0.0 and all(5 <= int(c) <= 7 for c in seam.offsets)


def test_batch_carve_random_vs_oracle(P):
    from oracle import scpl_oracle as O
    rng = np.random.default_rng(9)
    for k in range(6):
        h, w = int(rng.integers(16, 200)), int(rng.integers(16, 300))
        frame = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        energy = rng.uniform(0, 255, size=(h, w)) / 3 if k % 2 else None
        tgt = int(rng.integers(max(1, w // 2), w))
        c1, b1 = P.batch_carve(frame, tgt, energy=energy)
        c2, b2 = O.batch_carve(frame, tgt, energy=energy)
        assert np.array_equal(c1, c2)
        assert [len(x) for x in b1] == [len(x) for x in b2]
        for x, y in zip(b1, b2):
            assert [int(s.offsets[-1]) for s in x] == [int(c) for c in y.cols]
            assert [s.cost for s in x] == [float(c) for c in y.costs]
            assert np.array_equal(np.stack([s.offsets for s in x], 1), y.offsets)


# ------------------------------------------------------------------ buffer
def test_buffer_stream_golden(P, small):
    for s in cases.STREAM_SEEDS:
        maps = cases.stream_case(s)
        g = small["stream"][str(s)]
        buf = P.SpatioTemporalBuffer(policy=P.BufferPolicy())
        runs = []
        for m in maps:
            r = buf.push(np.zeros(m.shape, np.uint8), m)
            if r is not None:
                runs.append(len(r))
        runs.append(len(buf.flush()))
        assert runs == g["runs"], s


def test_buffer_known_answers(P):
    assert P.threshold(2, P.BufferPolicy()) == pytest.approx(25.5, abs=1e-12)
    buf = P.SpatioTemporalBuffer(policy=P.BufferPolicy(alpha=1000.0))
    for m in [np.zeros((3, 3)), np.full((3, 3), 255.0)]:
        buf.push(np.zeros((3, 3), np.uint8), m)
    assert buf.asde() == pytest.approx(127.5, abs=1e-12)
    assert (buf.uniform_energy() == 127.5).all()
    pol = P.BufferPolicy(max_len=4)
    b2 = P.SpatioTemporalBuffer(policy=pol)
    runs = [len(r) for r in (b2.push(np.zeros((3, 3), np.uint8), np.full((3, 3), 50.0)) for _ in range(10)) if r]
    runs.append(len(b2.flush()))
    assert runs == [4, 4, 2]


# ------------------------------------------------------------------ pipeline
def _cfg(P, cfg):
    cfg = dict(cfg)
    pol = P.BufferPolicy(**{k: cfg.pop(k) for k in ("alpha", "max_len") if k in cfg})
    return P.RetargetConfig(policy=pol, **cfg)


def test_pipeline_small_clips_golden(P, small):
    for name, (ck, cfg) in cases.CLIP_CASES.items():
        frames = cases.small_clip(**ck)
        out, m = P.retarget_video(frames, _cfg(P, cfg))
        g = small["clips"][name]
        assert m.dp_passes == g["dp_passes"], name
        assert [list(f.shape) for f in out] == g["shapes"], name
        assert [sha(f) for f in out] == g["frames"], name


@pytest.mark.parametrize("i", range(len(cases.SIZE_CASES)))
def test_size_cases_vs_oracle(P, i):
    """Every carve cluster size and plane shape class against the oracle (host frames and a CUDA clip)."""
    import torch
    from oracle import scpl_oracle as O
    frames, cfg = cases.size_clip(i)
    ref = O.retarget_video(frames, **cfg)
    out, m = P.retarget_video(frames, P.RetargetConfig(**cfg))
    assert m.dp_passes == ref.dp_passes
    if cfg["mode"] == "buffered":
        assert [tuple(r) for r in m.runs] == [tuple(r) for r in ref.runs]
    assert len(out) == len(ref.frames)
    for a, b in zip(out, ref.frames):
        assert np.array_equal(a, b)
    clip = torch.from_numpy(np.stack(frames)).cuda()
    dev, m2 = P.retarget_video_tensor(clip, P.RetargetConfig(**cfg))
    assert m2.dp_passes == ref.dp_passes
    assert np.array_equal(dev.cpu().numpy(), np.stack(ref.frames))


@pytest.mark.parametrize("wm,wg", cases.WEIGHT_CASES)
def test_energy_weights_golden(P, wm, wg):
    """Motion / gradient weight pairs through the scan, the uniform map and the carve against the
    reference's own outputs (tests/golden/weights.json, make_weights_golden.py) and the oracle:
    (0.08, 0.92) and (0.46, 0.54) give fl(fl(255 wm) + fl(255 wg)) > 255, so those clips take the
    clamped kernel variants, the others the clamp-free ones (energy.py:86-87)."""
    import torch
    from oracle import scpl_oracle as O
    with open(os.path.join(os.path.dirname(__file__), "golden", "weights.json")) as fh:
        g = json.load(fh)[f"{wm}/{wg}"]
    assert ((np.float64(wm) * 255.0) + (np.float64(wg) * 255.0) > 255.0) == ((wm, wg) in [(0.08, 0.92), (0.46, 0.54)])
    frames, tw = cases.weights_clip(wm)
    cfg = dict(target_width=tw, mode="buffered", w_motion=wm, w_grad=wg)
    out, m = P.retarget_video(frames, P.RetargetConfig(**cfg))
    assert [list(r) for r in m.runs] == g["runs"]
    assert m.dp_passes == g["dp_passes"]
    assert [sha(f) for f in out] == g["frames"]
    ref = O.retarget_video(frames, **cfg)
    for a, b in zip(out, ref.frames):
        assert np.array_equal(a, b)
    dev, m2 = P.retarget_video_tensor(torch.from_numpy(np.stack(frames)).cuda(), P.RetargetConfig(**cfg))
    assert [sha(f) for f in dev.cpu().numpy()] == g["frames"]


def test_pipeline_errors(P):
    with pytest.raises(ValueError, match="exceeds"):
        P.retarget_image(np.zeros((8, 8), np.uint8), P.RetargetConfig(target_width=9))
    with pytest.raises(ValueError, match="too small"):
        P.retarget_image(np.zeros((2, 8), np.uint8), P.RetargetConfig(target_width=4))
    with pytest.raises(ValueError, match="frame 1"):
        P.retarget_video([np.zeros((8, 8), np.uint8), np.zeros((8, 9), np.uint8)], P.RetargetConfig(target_width=4))
    out, m = P.retarget_video([], P.RetargetConfig(target_width=4, mode="buffered"))
    assert out == [] and m.frames_out == 0 and m.dp_passes == 0


def test_image_raw_pass_counts(P):
    rng = np.random.default_rng(51)
    frame = rng.integers(0, 256, size=(10, 15, 3), dtype=np.uint8)
    out, m = P.retarget_image(frame, P.RetargetConfig(target_width=10, mode="raw"))
    assert out.shape == (10, 10, 3) and m.dp_passes == 5


def _config_golden(name):
    return sorted(glob.glob(os.path.join(GOLD, f"{name}*.json")))


@pytest.mark.parametrize("path", _config_golden("C1") + _config_golden("C2") + _config_golden("C3")
                         + _config_golden("C4") + _config_golden("C5"))
def test_config_clip_golden(P, path):
    """Full BASELINE config clips vs the reference's own run (runs, dp_passes, every frame)."""
    from paper_1903_03180_b200.synth import config_clip
    import torch
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    dev = torch.from_numpy(clip).cuda()
    out, m = P.retarget_video_tensor(dev, P.RetargetConfig(target_width=tw, target_height=th, mode="buffered",
                                                           reaverage_energy=g.get("reaverage", False)))
    assert [list(r) for r in m.runs] == g["runs"]
    assert m.dp_passes == g["dp_passes"]
    host = out.cpu().numpy()
    assert list(host.shape[1:]) == g["out_shape"]
    bad = [t for t in range(host.shape[0]) if sha(host[t]) != g["frames_sha"][t]]
    assert not bad, f"{len(bad)} frames differ, first {bad[:5]}"


@pytest.mark.parametrize("path", _config_golden("C2") + _config_golden("C4_clip0") + _config_golden("C5"))
def test_config_clip_golden_host_buffers(P, path):
    """scpl_retarget_video_host (chunked H2D overlapped with the scan, per-run D2H) vs the reference."""
    from paper_1903_03180_b200.synth import config_clip
    import torch
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    host_in = torch.from_numpy(clip).pin_memory()
    out = torch.full((clip.shape[0],) + tuple(g["out_shape"]), 7, dtype=torch.uint8).pin_memory()
    res, m = P.retarget_video(host_in, P.RetargetConfig(target_width=tw, target_height=th, mode="buffered",
                                                        reaverage_energy=g.get("reaverage", False)), out=out)
    assert res.data_ptr() == out.data_ptr() and not res.is_cuda
    assert [list(r) for r in m.runs] == g["runs"]
    assert m.dp_passes == g["dp_passes"]
    host = res.numpy()
    bad = [t for t in range(host.shape[0]) if sha(host[t]) != g["frames_sha"][t]]
    assert not bad, f"{len(bad)} frames differ, first {bad[:5]}"


def test_host_buffers_unpinned_and_odd_chunks(P):
    """Unpinned host clip whose length is not a multiple of the 16-frame H2D chunk."""
    import torch
    rng = np.random.default_rng(77)
    clip = rng.integers(0, 256, size=(37, 24, 40, 3), dtype=np.uint8)
    clip[10:20] = clip[10]
    cfg = P.RetargetConfig(target_width=29, target_height=21, mode="buffered")
    a, ma = P.retarget_video(torch.from_numpy(clip), cfg)
    b, mb = P.retarget_video_tensor(torch.from_numpy(clip).cuda(), cfg)
    assert ma.runs == mb.runs and ma.dp_passes == mb.dp_passes
    assert torch.equal(a, b.cpu())
    from oracle import scpl_oracle as O
    r = O.retarget_video(list(clip), target_width=29, target_height=21, mode="buffered")
    assert r.dp_passes == ma.dp_passes
    assert all(np.array_equal(a[t].numpy(), r.frames[t]) for t in range(len(clip)))


def test_host_driven_loops_match(P, monkeypatch):
    """SCPL_HOST_LOOPS (profiling mode: scan and carve loops driven from the host instead of
    conditional graphs) gives the same runs, passes and frames as the graph loops."""
    from paper_1903_03180_b200.synth import config_clip
    import torch
    path = _config_golden("C4_clip0")[0]
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    monkeypatch.setenv("SCPL_HOST_LOOPS", "1")
    out, m = P.retarget_video_tensor(torch.from_numpy(clip).cuda(),
                                     P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))
    assert [list(r) for r in m.runs] == g["runs"] and m.dp_passes == g["dp_passes"]
    host_out = out.cpu().numpy()
    assert all(sha(host_out[i]) == g["frames_sha"][i] for i in range(host_out.shape[0]))


@pytest.mark.parametrize("group_min", ["1", "3", "1000"])
@pytest.mark.parametrize("host", [False, True])
def test_run_grouping_does_not_change_results(P, group_min, host, monkeypatch):
    """Runs are carved in groups dispatched as the scan closes them; any grouping (one run per
    group, a few, or one group after the whole scan) must give the reference's frames."""
    from paper_1903_03180_b200.synth import config_clip
    import torch
    path = _config_golden("C4_clip0")[0]
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    monkeypatch.setenv("SCPL_GROUP_MIN", group_min)
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
    t = torch.from_numpy(clip)
    out, m = P.retarget_video(t.pin_memory() if host else t.cuda(), cfg)
    host_out = out.cpu().numpy()
    assert [list(r) for r in m.runs] == g["runs"] and m.dp_passes == g["dp_passes"]
    bad = [i for i in range(host_out.shape[0]) if sha(host_out[i]) != g["frames_sha"][i]]
    assert not bad, f"{len(bad)} frames differ"


def test_reaverage_small_clips_golden(P, small):
    """reaverage_energy (pipeline.py:269-270, 280-296): runs carved on the mean gradient of
    all their carved frames, vs the reference's outputs."""
    names = [n for n in cases.CLIP_CASES if n.startswith("rea")]
    assert names
    for name in names:
        ck, cfg = cases.CLIP_CASES[name]
        frames = cases.small_clip(**ck)
        out, m = P.retarget_video(frames, _cfg(P, cfg))
        g = small["clips"][name]
        assert m.dp_passes == g["dp_passes"], name
        assert [list(f.shape) for f in out] == g["shapes"], name
        assert [sha(f) for f in out] == g["frames"], name


def test_jitter_golden(P, small):
    """bench.jitter (bench.py:39-57) on the GPU: exact integer pair sums, the reference's float
    means -- bit-equal values."""
    for name, (ck, win) in cases.JITTER_CASES.items():
        rep = P.jitter(cases.small_clip(**ck), window=win)
        assert rep.window == win
        assert float(rep.value).hex() == small["jitter"][name], name
    with pytest.raises(ValueError, match="at least 2 frames"):
        P.jitter([np.zeros((4, 4, 3), np.uint8)])


def test_pnm_stream_retarget_roundtrip(P, small):
    """The `vidcarve video - -` pipe on the GPU: PNM bytes -> pinned clip -> retarget ->
    PNM bytes, frames equal to the reference's retarget_video outputs."""
    import io
    from paper_1903_03180_b200 import media
    for name in ("buf_w", "buf_wh", "rea_w"):
        ck, cfg = cases.CLIP_CASES[name]
        frames = cases.small_clip(**ck)
        src = io.BytesIO()
        media.write_frames(src, frames)
        src.seek(0)
        clip = media.read_clip_pinned(src)
        assert clip.is_pinned() and tuple(clip.shape) == (len(frames),) + frames[0].shape
        src.seek(0)
        dst = io.BytesIO()
        media.retarget_stream(src, dst, _cfg(P, cfg))
        dst.seek(0)
        out = list(media.read_frames(dst))
        assert [sha(f) for f in out] == small["clips"][name]["frames"], name


@pytest.mark.parametrize("mode", [None, "SCPL_SCAN_EXACT", "SCPL_SCAN_FORCE_FALLBACK"])
def test_scan_screening_modes_match(P, mode, monkeypatch):
    """The buffer scan screens each window with a cheap bounded ASDE (buffering.py:119 decided
    from |asde~ - asde| <= bound) and re-runs it exactly only when the bound cannot settle a
    threshold test.  Screened (default), all-exact and screened-then-always-re-run scans give
    the reference's run boundaries (and so its passes) on the config clips."""
    from paper_1903_03180_b200 import pipeline
    from paper_1903_03180_b200.synth import config_clip
    import torch
    if mode:
        monkeypatch.setenv(mode, "1")
    for path in _config_golden("C2") + _config_golden("C4_clip0") + _config_golden("C5"):
        g = json.load(open(path))
        if g.get("reaverage"):
            continue
        clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
        out, m = P.retarget_video_tensor(torch.from_numpy(clip).cuda(),
                                         P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))
        assert [list(r) for r in m.runs] == g["runs"], path
        assert m.dp_passes == g["dp_passes"], path
        ph = pipeline.last_phase_ms
        if mode == "SCPL_SCAN_FORCE_FALLBACK":
            assert ph["scan_fallbacks"] > 0
        elif mode is None:  # screening settles (almost) every window
            assert ph["scan_fallbacks"] * 10 <= ph["scan_windows"], ph
        else:
            assert ph["scan_fallbacks"] == 0


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_clip_matches_reference(P, world):
    """One clip split across `world` ranks (sharding.py): each rank scans the whole clip and
    carves only its runs; the union of the ranks' outputs is the reference's clip and their
    passes add up to its dp_passes.  (The ranks run one after another on one GPU here: they
    never wait on each other, so this is exactly what each GPU of a multi-GPU job computes.)"""
    from paper_1903_03180_b200 import sharding
    from paper_1903_03180_b200.synth import config_clip
    import torch
    for name in ("C4_clip0", "C5"):
        g = json.load(open(_config_golden(name)[0]))
        clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
        dev = torch.from_numpy(clip).cuda()
        cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
        merged = np.zeros((clip.shape[0],) + tuple(g["out_shape"]), dtype=np.uint8)
        dp = 0
        for rank in range(world):
            out, m = P.retarget_video_tensor(dev, cfg, shard=(rank, world))
            assert [list(r) for r in m.runs] == g["runs"]
            dp += m.dp_passes
            host = out.cpu().numpy()
            for s, n in sharding.owned_spans(m.runs, rank, world, "buffered", clip.shape[0]):
                merged[s:s + n] = host[s:s + n]
        assert dp == g["dp_passes"]
        bad = [t for t in range(merged.shape[0]) if sha(merged[t]) != g["frames_sha"][t]]
        assert not bad, f"{name}: {len(bad)} frames differ"
        # scan once, runs dealt longest-processing-time first, each rank carves exactly its runs
        runs = P.scan_runs(dev, cfg)
        owners = sharding.lpt_owners(runs, world)
        merged[:] = 0
        dp = 0
        for rank in range(world):
            mine = [r for r, o in zip(runs, owners) if o == rank]
            out, m = P.retarget_video_tensor(dev, cfg, runs=mine)
            dp += m.dp_passes
            host = out.cpu().numpy()
            for s, n in mine:
                merged[s:s + n] = host[s:s + n]
        assert dp == g["dp_passes"]
        bad = [t for t in range(merged.shape[0]) if sha(merged[t]) != g["frames_sha"][t]]
        assert not bad, f"{name} (scan once): {len(bad)} frames differ"


@pytest.mark.parametrize("host_loops", [False, True])
def test_fused_passes_match(P, host_loops, monkeypatch):
    """SCPL_FUSED=1 (experimental fused int passes: the pass kernel's producer warps remove the
    previous batch and compute the Sobel energy into the DP's ring) gives the reference's runs,
    passes and frames -- a C4 clip against its golden, random single frames against the oracle."""
    from oracle import scpl_oracle as O
    from paper_1903_03180_b200.synth import config_clip
    import torch
    monkeypatch.setenv("SCPL_FUSED", "1")
    if host_loops:
        monkeypatch.setenv("SCPL_HOST_LOOPS", "1")
    path = _config_golden("C4_clip0")[0]
    g = json.load(open(path))
    clip, tw, th = config_clip(g["config"], frames=g["frames"], clip=g["clip"])
    out, m = P.retarget_video_tensor(torch.from_numpy(clip).cuda(),
                                     P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))
    assert [list(r) for r in m.runs] == g["runs"] and m.dp_passes == g["dp_passes"]
    host_out = out.cpu().numpy()
    assert all(sha(host_out[i]) == g["frames_sha"][i] for i in range(host_out.shape[0]))
    rng = np.random.default_rng(21)
    for h, w, t in [(100, 300, 250), (34, 520, 400), (200, 100, 60), (65, 1100, 1000)]:
        frame = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        c1, b1 = P.batch_carve(frame, t)
        c2, b2 = O.batch_carve(frame, t)
        assert np.array_equal(c1, c2) and [len(x) for x in b1] == [len(x) for x in b2]
