"""Temporal jitter (the reference's `vidcarve.bench.jitter`, bench.py:23-57) on the GPU.

Jitter = windowed mean absolute inter-frame luma difference. The per-pair pixel sums of
|luma(t+1) - luma(t)| are exact integers computed by libscpl (scpl_jitter_sums); the
reference's float64 means of those integers are exact up to one division, which is done
here with numpy exactly as the reference does, as are the window averages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class JitterReport:
    window: int
    value: float


def jitter(frames, window: int = 4) -> JitterReport:
    """Mean over sliding windows of the mean |dL| between consecutive frames; a stream shorter
    than the window is one window over all its frames (bench.py:39-57)."""
    torch = _lib.torch_cuda()
    if isinstance(frames, torch.Tensor):
        clip = frames if frames.is_cuda else frames.cuda()
        n = clip.shape[0]
    else:
        frames = [np.asarray(f) for f in frames]
        n = len(frames)
        if n < 2:
            raise ValueError(f"need at least 2 frames, got {n}")
        for i, f in enumerate(frames[1:], start=1):
            if f.shape[:2] != frames[0].shape[:2]:
                raise ValueError(f"frame {i}: dimensions differ from frame 0")
        clip = torch.from_numpy(np.stack(frames)).cuda()
    if n < 2:
        raise ValueError(f"need at least 2 frames, got {n}")
    h, w = clip.shape[1:3]
    c = clip.shape[3] if clip.dim() == 4 else 1
    sums = torch.empty(n - 1, dtype=torch.int64, device=clip.device)
    _lib.check(_lib.load().scpl_jitter_sums(_lib.ctx(clip.device.index), clip.contiguous().data_ptr(), n, h, w, c,
                                            sums.data_ptr(), _lib.stream()))
    diffs = sums.cpu().numpy().astype(np.float64) / np.float64(h * w)
    win = min(window, n)
    pairs = win - 1
    values = [diffs[t:t + pairs].mean() for t in range(n - win + 1)]
    return JitterReport(window=window, value=float(np.mean(values)))


# ------------------------------------------------------------------ corpora and comparison
SYNTHETIC_KINDS = ("static", "moving-box", "brightness-ramp")


@dataclass(frozen=True)
class SyntheticSpec:
    """Deterministic corpus recipe (bench.py:29-36)."""

    kind: str
    width: int = 320
    height: int = 240
    frames: int = 32
    seed: int = 0


def generate(spec: SyntheticSpec) -> list:
    """The reference's three synthetic corpora, byte for byte (bench.py:60-97): a static noise
    frame, a bright box sliding over a noise background, a wrapping brightness ramp."""
    if spec.kind not in SYNTHETIC_KINDS:
        raise ValueError(f"unknown corpus kind {spec.kind!r}, expected one of {SYNTHETIC_KINDS}")
    if spec.width < 3 or spec.height < 3:
        raise ValueError(f"corpus frames must be at least 3x3, got {spec.width}x{spec.height}")
    if spec.frames < 1:
        raise ValueError(f"frame count must be >= 1, got {spec.frames}")
    rng = np.random.default_rng(spec.seed)
    h, w, n = spec.height, spec.width, spec.frames
    if spec.kind == "static":
        still = rng.integers(112, 144, size=(h, w, 3), dtype=np.uint8)
        return [still.copy() for _ in range(n)]
    if spec.kind == "moving-box":
        bg = rng.integers(0, 128, size=(h, w, 3), dtype=np.uint8)
        bw, bh, top = max(4, w // 8), max(4, h // 8), h // 4
        out = []
        for t in range(n):
            f = bg.copy()
            left = t % (w - bw + 1)
            f[top:top + bh, left:left + bw] = 250
            out.append(f)
        return out
    ramp = rng.integers(0, 64, size=(h, w, 3), dtype=np.int64)
    return [np.clip(ramp + (16 * t) % 192, 0, 255).astype(np.uint8) for t in range(n)]


def compare(frames, variants: dict) -> dict:
    """Every config variant over the corpus, metrics with jitter (bench.py:100-112)."""
    from .pipeline import retarget_video
    if not variants:
        raise ValueError("need at least one config variant")
    results = {}
    for name, config in variants.items():
        out, metrics = retarget_video(frames, config)
        if len(out) >= 2:
            metrics.jitter = jitter(out).value
        results[name] = metrics
    return results


def format_metrics(results) -> str:
    """Flat key=value report, variant-prefixed keys when comparing (bench.py:115-131)."""
    lines = []

    def emit(prefix, m):
        lines.extend([f"{prefix}dp_passes={m.dp_passes}", f"{prefix}wall_time_s={m.wall_time:.6f}",
                      f"{prefix}frames_out={m.frames_out}"])
        if m.jitter is not None:
            lines.append(f"{prefix}jitter={m.jitter:.6f}")

    if isinstance(results, dict):
        for name, m in results.items():
            emit(f"{name}.", m)
    else:
        emit("", results)
    return "\n".join(lines) + "\n"


__all__ = ["JitterReport", "SYNTHETIC_KINDS", "SyntheticSpec", "compare", "format_metrics", "generate", "jitter"]
