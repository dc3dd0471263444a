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


__all__ = ["JitterReport", "jitter"]
