"""Seeded parity cases shared by tests/golden/make_golden.py and the tests.

Every input is regenerated from its seed here, so the committed golden files
only hold the reference's OUTPUTS (hashes, seam columns, run boundaries,
dp_passes). Case shapes follow the reference's own tests (pkg/tests/*.py):
tiny maps for the DP/label/batch invariants, small streams for the buffer,
small clips for every pipeline mode and axis combination.
"""

from __future__ import annotations

import hashlib

import numpy as np


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def fhex(x) -> str:
    return float(x).hex()


def luma_table_frame() -> np.ndarray:
    """All 2^24 RGB triples as one (4096, 4096, 3) frame (r major)."""
    v = np.arange(1 << 24, dtype=np.uint32)
    return np.stack([(v >> 16) & 255, (v >> 8) & 255, v & 255], -1).astype(np.uint8).reshape(4096, 4096, 3)


# ------------------------------------------------------------------ energy cases
def energy_case(seed: int):
    rng = np.random.default_rng(1000 + seed)
    h, w = int(rng.integers(3, 41)), int(rng.integers(3, 41))
    curr = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    prev = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    return curr, prev


ENERGY_SEEDS = list(range(12))


# ------------------------------------------------------------------ DP / batch cases
def map_case(seed: int, hmax=20, wmax=20):
    rng = np.random.default_rng(2000 + seed)
    h, w = int(rng.integers(1, hmax + 1)), int(rng.integers(1, wmax + 1))
    kind = seed % 3
    if kind == 0:
        m = rng.uniform(0, 255, size=(h, w))
    elif kind == 1:  # integer-valued (gradient-like) with many ties
        m = rng.integers(0, 4, size=(h, w)).astype(np.float64)
    else:            # uniform-like means of motion energies
        m = rng.uniform(0, 255, size=(h, w)) / 3.0
    return m


MAP_SEEDS = list(range(40))


def carve_case(seed: int):
    rng = np.random.default_rng(3000 + seed)
    h, w = int(rng.integers(3, 30)), int(rng.integers(4, 48))
    frame = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    target = int(rng.integers(1, w))
    energy = None
    if seed % 2 == 0:
        energy = rng.uniform(0, 255, size=(h, w)) / float(rng.integers(1, 7))
    return frame, target, energy


CARVE_SEEDS = list(range(16))


# ------------------------------------------------------------------ buffer streams
def stream_case(seed: int):
    """Energy-map streams in the style of test_buffering.py:158-179 (drift + upheavals)."""
    rng = np.random.default_rng(4000 + seed)
    h, w = int(rng.integers(3, 24)), int(rng.integers(3, 24))
    base = rng.uniform(20, 120, size=(h, w))
    maps = []
    for k in range(40):
        jump = 120.0 if rng.random() < 0.1 else 0.0
        maps.append(np.clip(base + rng.uniform(-6, 6, size=(h, w)) + jump, 0, 255))
    return maps


STREAM_SEEDS = list(range(8))


# ------------------------------------------------------------------ small clips
def small_clip(seed: int, t=10, h=24, w=32, gray=False, motion=2, rects=3):
    """Moving rectangles on a noisy gradient, small enough for the reference in seconds."""
    rng = np.random.default_rng(5000 + seed)
    x = np.round(255.0 * np.arange(w) / (w - 1))
    frames = []
    params = [(rng.integers(0, 256, 3), int(rng.integers(3, max(4, h // 2))), int(rng.integers(3, max(4, w // 2))),
               int(rng.integers(0, h)), int(rng.integers(0, w)),
               int(rng.integers(-motion, motion + 1)), int(rng.integers(-motion, motion + 1))) for _ in range(rects)]
    for k in range(t):
        img = np.empty((h, w, 3)); img[:] = x[None, :, None]
        for col, rh, rw, y0, x0, vy, vx in params:
            img[np.ix_((y0 + vy * k + np.arange(rh)) % h, (x0 + vx * k + np.arange(rw)) % w)] = col
        img += rng.normal(0, 4, size=img.shape)
        f = np.clip(np.rint(img), 0, 255).astype(np.uint8)
        frames.append(f[:, :, 0].copy() if gray else f)
    return frames


# name -> (clip kwargs, config kwargs)
CLIP_CASES = {
    "buf_w": (dict(seed=0), dict(target_width=24, mode="buffered")),
    "buf_h": (dict(seed=1), dict(target_height=17, mode="buffered")),
    "buf_wh": (dict(seed=2), dict(target_width=25, target_height=19, mode="buffered")),
    "buf_wh_hf": (dict(seed=3), dict(target_width=25, target_height=19, mode="buffered", height_first=True)),
    "buf_gray": (dict(seed=4, gray=True), dict(target_width=20, mode="buffered")),
    "buf_fast": (dict(seed=5, motion=6, t=14), dict(target_width=22, mode="buffered")),
    "buf_maxlen3": (dict(seed=6, t=11), dict(target_width=26, mode="buffered", max_len=3)),
    "buf_alpha": (dict(seed=7, t=12), dict(target_width=23, mode="buffered", alpha=0.05)),
    "buf_w1": (dict(seed=8, t=4, h=9, w=8), dict(target_width=1, mode="buffered")),
    "buf_tall": (dict(seed=9, t=6, h=70, w=20), dict(target_width=11, mode="buffered")),
    "buf_wide": (dict(seed=10, t=6, h=5, w=90), dict(target_width=40, mode="buffered")),
    "buf_weights": (dict(seed=11), dict(target_width=24, mode="buffered", w_motion=0.25, w_grad=0.75)),
    "scpl_w": (dict(seed=12, t=6), dict(target_width=24, mode="scpl")),
    "scpl_wh": (dict(seed=13, t=5), dict(target_width=27, target_height=20, mode="scpl")),
    "raw_w": (dict(seed=14, t=4), dict(target_width=26, mode="raw")),
    "raw_h": (dict(seed=15, t=3), dict(target_height=20, mode="raw")),
    "buf_single": (dict(seed=16, t=1), dict(target_width=20, mode="buffered")),
    # reaverage_energy (pipeline.py:269-270, 280-296): every pass after a run's first on the
    # mean gradient of all the run's carved frames
    "rea_w": (dict(seed=17), dict(target_width=24, mode="buffered", reaverage_energy=True)),
    "rea_wh": (dict(seed=18), dict(target_width=25, target_height=19, mode="buffered", reaverage_energy=True)),
    "rea_hf": (dict(seed=19), dict(target_width=26, target_height=18, mode="buffered", height_first=True,
                                   reaverage_energy=True)),
    "rea_scpl": (dict(seed=20, t=5), dict(target_width=24, mode="scpl", reaverage_energy=True)),
    "rea_gray": (dict(seed=21, gray=True), dict(target_width=21, mode="buffered", reaverage_energy=True)),
}


# Wider / taller clips than the reference finishes quickly, checked against the oracle: every
# carve cluster size (1..8 CTAs: widths up to the 4096-column limit), the staged and unstaged
# landing-delta table (tall planes), height carving of tall frames, raw / scpl / reaverage.
# (h, w, t, config)
SIZE_CASES = [
    (150, 600, 5, dict(target_width=430)),
    (120, 1100, 4, dict(target_width=800)),
    (100, 2100, 4, dict(target_width=1500)),
    (80, 3300, 3, dict(target_width=2700)),
    (64, 4096, 3, dict(target_width=3000)),
    (1500, 40, 3, dict(target_width=29)),
    (700, 24, 4, dict(target_height=520)),
    (90, 2600, 4, dict(target_width=2000, target_height=70)),
    (100, 1100, 4, dict(target_width=1000, mode="raw")),
    (100, 1100, 4, dict(target_width=900, mode="scpl")),
    (96, 1300, 6, dict(target_width=1000, reaverage_energy=True)),
]


def size_clip(i: int):
    h, w, t, cfg = SIZE_CASES[i]
    return small_clip(seed=100 + i, t=t, h=h, w=w, rects=6), dict(mode="buffered", **cfg) if "mode" not in cfg else cfg


# ------------------------------------------------------------------ media / jitter
def media_streams():
    """(name, bytes) PNM streams exercising the byte grammar and its errors (media.py:139-223)."""
    rng = np.random.default_rng(31)
    rgb = rng.integers(0, 256, (5, 7, 3), dtype=np.uint8)
    gray = rng.integers(0, 256, (4, 6), dtype=np.uint8)
    rgb2 = rng.integers(0, 256, (5, 7, 3), dtype=np.uint8)
    p6 = b"P6\n7 5\n255\n" + rgb.tobytes()
    return [
        ("p6_two", p6 + b"P6 7 5 255 " + rgb2.tobytes()),
        ("p5_comment", b"P5 # a comment\n6\t4\r\n# more\n255\n" + gray.tobytes()),
        ("empty", b""),
        ("whitespace_only", b" \n\t "),
        ("bad_magic", b"P3 7 5 255\n" + rgb.tobytes()),
        ("bad_maxval", b"P6 7 5 65535\n" + rgb.tobytes()),
        ("bad_dims", b"P6 0 5 255\n"),
        ("bad_width", b"P6 x 5 255\n"),
        ("truncated", p6[:-5]),
        ("header_eof", b"P6 7"),
        ("dim_change", p6 + b"P6 6 5 255\n" + rgb[:, :6].tobytes()),
        ("mixed_gray_rgb", p6 + b"P5 7 5 255\n" + gray.ravel()[:1].tobytes() * 35),
    ]


JITTER_CASES = {  # name -> (small_clip kwargs, window)
    "j_default": (dict(seed=40, t=9), 4),
    "j_short": (dict(seed=41, t=3), 4),
    "j_two": (dict(seed=42, t=2), 4),
    "j_w2": (dict(seed=43, t=12), 2),
    "j_gray": (dict(seed=44, t=7, gray=True), 3),
    "j_long": (dict(seed=45, t=40, h=30, w=50), 5),
}


# Motion / gradient weight pairs (w_motion, w_grad): (0.08, 0.92) and (0.46, 0.54) give
# fl(fl(255 wm) + fl(255 wg)) > 255, so the energy clamp min(e, 255) is live for them.
WEIGHT_CASES = [(0.6, 0.4), (0.08, 0.92), (0.46, 0.54), (1.0, 0.0), (0.0, 1.0), (0.25, 0.75)]


def weights_clip(wm):
    """14 frames 40x72: slow drift, one cut, saturated patches (energies at the 255 end), a noisy row."""
    rng = np.random.default_rng(int(wm * 1000) + 17)
    T, H, W = 14, 40, 72
    base = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    frames = []
    for t in range(T):
        f = np.roll(base, (t // 3, t // 2), axis=(0, 1)).copy()
        if t >= 9:
            f = 255 - f
        f[:6, :8] = 255 * (t & 1)
        f[(t * 2) % H, :, :] = rng.integers(0, 256, (W, 3), dtype=np.uint8)
        frames.append(f)
    return frames, W - 13
