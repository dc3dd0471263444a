"""Seeded synthetic clips for the five BASELINE configurations.

The reference measures on the paper's own videos ("Big Belly", "Lion", ...,
`PAPER.md:159-174`), which are not available; these generators stand in for
them with the shapes, sizes and content BASELINE.json names. One generator
feeds both the CPU oracle and the GPU path, so parity is checked on identical
bytes.

Recipe (fixed once, recorded here and in DESIGN.md):

* background: horizontal linear gradient ``round(255*x/(W-1))`` on all three
  channels; C2 frames 100-199 replace it with a full-frame sinusoid
  ``128 + 100*sin(2*pi*(x - 2*(t-100))/32)`` (panning 2 px/frame);
* rectangles: solid colour uniform in [0,255]^3, integer sides uniform in the
  stated range, integer velocity per axis uniform in the stated range with a
  random sign, wrap-around at the borders (drawn in order, later ones on top);
* C5 only: a per-frame global brightness offset in U{-10..10} on all channels;
* noise: per-pixel, per-channel N(0, sigma) in float32 (frame t draws from
  ``default_rng([seed, t])``), added in float, ``rint`` and clipped to
  [0, 255] -> uint8.

Frames are produced in parallel threads (numpy releases the GIL while
drawing normals), so the 1.9 GB C2 clip is generated in seconds.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
import os

import numpy as np


@dataclass(frozen=True)
class ClipSpec:
    frames: int
    height: int
    width: int
    n_rects: int
    rect_size: tuple[int, int]
    speed: tuple[int, int]
    sigma: float
    seed: int = 0
    pan: tuple[int, int] | None = None  # [start, stop) frames with the sinusoid background
    flicker: int = 0                    # max |global brightness offset| per frame


# name -> (spec, target_width, target_height)
CONFIGS: dict[str, tuple[ClipSpec, int | None, int | None]] = {
    "C1": (ClipSpec(30, 240, 320, 3, (20, 60), (1, 3), 4.0), 256, None),
    "C2": (ClipSpec(300, 1080, 1920, 8, (40, 300), (0, 6), 4.0, pan=(100, 200)), 1440, None),
    "C3": (ClipSpec(120, 2160, 3840, 8, (80, 600), (0, 1), 2.0), 2880, None),
    "C4": (ClipSpec(90, 720, 1280, 8, (40, 300), (0, 6), 4.0), 960, None),
    "C5": (ClipSpec(240, 1080, 1920, 12, (40, 300), (4, 10), 4.0, flicker=10), None, 810),
}
C4_CLIPS = 64


def _rects(spec: ClipSpec):
    rng = np.random.default_rng(spec.seed)
    rects = []
    for _ in range(spec.n_rects):
        colour = rng.integers(0, 256, size=3)
        rh = int(rng.integers(spec.rect_size[0], spec.rect_size[1] + 1))
        rw = int(rng.integers(spec.rect_size[0], spec.rect_size[1] + 1))
        y0 = int(rng.integers(0, spec.height))
        x0 = int(rng.integers(0, spec.width))
        vy = int(rng.integers(spec.speed[0], spec.speed[1] + 1)) * (1 if rng.random() < 0.5 else -1)
        vx = int(rng.integers(spec.speed[0], spec.speed[1] + 1)) * (1 if rng.random() < 0.5 else -1)
        rects.append((colour.astype(np.float32), min(rh, spec.height), min(rw, spec.width), y0, x0, vy, vx))
    flick = rng.integers(-spec.flicker, spec.flicker + 1, size=spec.frames) if spec.flicker else None
    return rects, flick


def _frame(spec: ClipSpec, t: int, rects, flick, out: np.ndarray) -> None:
    h, w = spec.height, spec.width
    x = np.arange(w, dtype=np.float64)
    if spec.pan is not None and spec.pan[0] <= t < spec.pan[1]:
        row = 128.0 + 100.0 * np.sin(2.0 * np.pi * (x - 2.0 * (t - spec.pan[0])) / 32.0)
    else:
        row = np.round(255.0 * x / (w - 1))
    img = np.empty((h, w, 3), dtype=np.float32)
    img[:] = row.astype(np.float32)[None, :, None]
    for colour, rh, rw, y0, x0, vy, vx in rects:
        ys = (y0 + vy * t + np.arange(rh)) % h
        xs = (x0 + vx * t + np.arange(rw)) % w
        img[np.ix_(ys, xs)] = colour
    if flick is not None:
        img += np.float32(flick[t])
    rng = np.random.default_rng([spec.seed, t])
    img += rng.standard_normal((h, w, 3), dtype=np.float32) * np.float32(spec.sigma)
    np.rint(img, out=img)
    np.clip(img, 0, 255, out=img)
    out[...] = img.astype(np.uint8)


def generate_clip(spec: ClipSpec, frames: int | None = None, out: np.ndarray | None = None,
                  threads: int | None = None, start: int = 0) -> np.ndarray:
    """(T, H, W, 3) uint8 clip; ``frames`` truncates to T frames, from frame ``start`` (every
    frame is a function of its index alone, so any window is generated directly)."""
    t_total = (spec.frames - start) if frames is None else min(frames, spec.frames - start)
    if out is None:
        out = np.empty((t_total, spec.height, spec.width, 3), dtype=np.uint8)
    rects, flick = _rects(spec)
    threads = threads or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda t: _frame(spec, start + t, rects, flick, out[t]), range(t_total)))
    return out


def config_clip(name: str, frames: int | None = None, clip: int = 0, **kw):
    """(clip array, target_width, target_height) for config C1..C5 (C4: clip index = seed)."""
    spec, tw, th = CONFIGS[name]
    if name == "C4":
        spec = ClipSpec(**{**spec.__dict__, "seed": clip})
    return generate_clip(spec, frames=frames, **kw), tw, th
