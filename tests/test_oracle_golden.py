"""Pin the CPU oracle (oracle/) against golden vectors made by the reference itself.

CPU-only (no GPU marker). tests/golden/*.json come from tests/golden/make_golden.py,
which ran /root/reference's vidcarve in the build container.
"""
import json
import os

import numpy as np
import pytest

import cases
from cases import fhex, sha
from oracle import scpl_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def small():
    with open(os.path.join(GOLD, "small.json")) as f:
        return json.load(f)


def _batch_rec(b, labels=False):
    r = {"b": len(b), "cols": [int(c) for c in b.cols], "costs": [fhex(c) for c in b.costs],
         "offsets_sha": sha(b.offsets.astype(np.int32)) if len(b) else sha(np.zeros((0, 0), np.int32)),
         "source_width": b.source_width}
    if labels:
        r["labels_sha"] = sha(np.asarray(b.labels, dtype=np.int64))
    return r


def test_luma_table_pinned():
    lt = cases.luma_table_frame()
    want = open(os.path.join(GOLD, "luma_table.sha256")).read().strip()
    assert sha(O.to_luma_c(lt)) == want
    assert sha(O.to_luma(lt)) == want


def test_energy_golden(small):
    for s in cases.ENERGY_SEEDS:
        curr, prev = cases.energy_case(s)
        g = small["energy"][str(s)]
        assert sha(O.to_luma(curr)) == g["luma"]
        assert sha(O.gradient_energy(O.to_luma(curr))) == g["grad"]
        assert sha(O.motion_energy(curr, prev)) == g["motion"]
        assert sha(O.motion_energy(curr, None)) == g["motion_first"]
        assert sha(O.motion_energy(curr, prev, 0.3, 0.7)) == g["motion_w"]
        luma = O.to_luma(curr)
        out = np.empty_like(luma)
        O.clib().oracle_sobel(np.ascontiguousarray(luma).ctypes.data, luma.shape[0], luma.shape[1], out.ctypes.data)
        assert np.array_equal(out.astype(np.float64), O.gradient_energy(luma))


def test_dp_labels_batches_golden(small):
    for s in cases.MAP_SEEDS:
        m = cases.map_case(s)
        g = small["dp"][str(s)]
        ce, back = O.cumulative_energy(m)
        assert sha(ce) == g["ce"] and sha(back) == g["back"]
        lab = O.label_parents(back)
        assert lab.tolist() == g["labels"]
        assert _batch_rec(O.select_batch(ce, back, lab)) == g["batch"]
        assert _batch_rec(O.select_batch(ce, back, lab, k=g["k"])) == g["batch_k"]


def test_batch_carve_golden(small):
    for s in cases.CARVE_SEEDS:
        frame, target, energy = cases.carve_case(s)
        carved, batches = O.batch_carve(frame, target, energy=energy)
        g = small["carve"][str(s)]
        assert sha(carved) == g["carved"]
        assert [_batch_rec(b) for b in batches] == g["batches"]
        # the composed-index gather equals batch-by-batch removal (finding 7)
        idx = O.compose_index(frame.shape[0], frame.shape[1], batches)
        assert np.array_equal(O.replay_gather([frame], idx)[0], carved)


def test_buffer_scan_golden(small):
    for s in cases.STREAM_SEEDS:
        maps = cases.stream_case(s)
        tr = O.ScanTrace()
        runs = O.buffer_scan(maps, O.BufferPolicy(), tr)
        g = small["stream"][str(s)]
        assert [n for _, n in runs] == g["runs"]
        assert [fhex(a) for _, _, a, _ in tr.asde] == g["asde"]
        # the C restatement of numpy's pairwise mean gives the same ASDE, push by push
        S, Q, n_in = None, None, 0
        for (t, n, a, ok), e in zip(tr.asde, maps[1:]):
            if n_in == 0 or n == 2 and S is None:
                S, Q, n_in = maps[t - 1].copy(), maps[t - 1] * maps[t - 1], 1
            assert n == n_in + 1
            cS, cQ = S + e, Q + e * e
            assert fhex(O.asde_from_sums_c(cS, cQ, n)) == fhex(a)
            if ok:
                S, Q, n_in = cS, cQ, n
            else:
                S, Q, n_in = e.copy(), e * e, 1


def test_asde_c_matches_numpy():
    rng = np.random.default_rng(7)
    for shape in [(3, 3), (24, 32), (240, 320), (250, 333), (1080, 1920)]:
        S = rng.uniform(0, 255 * 4, size=shape)
        Q = S * S / 4 + rng.uniform(0, 500, size=shape)
        for n in (2, 5, 64):
            assert O.asde_from_sums(S, Q, n) == O.asde_from_sums_c(S, Q, n)


def test_threshold_known_answers():
    p = O.BufferPolicy()
    assert O.threshold(1, p) == 0.0
    assert O.threshold(2, p) == pytest.approx(25.5, abs=1e-12)
    vals = [O.threshold(n, p) for n in range(2, 200)]
    assert all(a > b for a, b in zip(vals, vals[1:]))


def _clip_cfg(cfg):
    cfg = dict(cfg)
    pol = O.BufferPolicy(**{k: cfg.pop(k) for k in ("alpha", "max_len") if k in cfg})
    return pol, cfg


def test_pipeline_small_clips_golden(small):
    for name, (ck, cfg) in cases.CLIP_CASES.items():
        frames = cases.small_clip(**ck)
        pol, cfg = _clip_cfg(cfg)
        res = O.retarget_video(frames, policy=pol, **cfg)
        g = small["clips"][name]
        assert res.dp_passes == g["dp_passes"], name
        assert [sha(f) for f in res.frames] == g["frames"], name


def test_pipeline_C1_golden():
    from paper_1903_03180_b200.synth import config_clip
    g = json.load(open(os.path.join(GOLD, "C1.json")))
    clip, tw, th = config_clip("C1")
    res = O.retarget_video(list(clip), target_width=tw, target_height=th, keep_batches=True)
    assert [list(r) for r in res.runs] == g["runs"]
    assert res.dp_passes == g["dp_passes"]
    assert [[[_batch_rec(b, labels=True) for b in ph] for ph in rb] for rb in res.batches] == g["batches"]
    assert [sha(f) for f in res.frames] == g["frames_sha"]


@pytest.mark.parametrize("wm,wg", cases.WEIGHT_CASES)
def test_pipeline_weights_golden(wm, wg):
    """Non-default motion / gradient weights (two pairs with a live 255 clamp): the oracle against
    the reference's outputs (tests/golden/make_weights_golden.py)."""
    with open(os.path.join(GOLD, "weights.json")) as fh:
        g = json.load(fh)[f"{wm}/{wg}"]
    frames, tw = cases.weights_clip(wm)
    ref = O.retarget_video(frames, target_width=tw, mode="buffered", w_motion=wm, w_grad=wg)
    assert [list(r) for r in ref.runs] == g["runs"]
    assert ref.dp_passes == g["dp_passes"]
    assert [sha(f) for f in ref.frames] == g["frames"]
