"""Temporal buffer -- drop-in for vidcarve.buffering (pkg/src/vidcarve/buffering.py).

BufferPolicy and threshold are host arithmetic, computed exactly as the reference does
(the C-ABI receives the phi table from here). SpatioTemporalBuffer keeps its per-pixel
sums S, Q on the GPU and evaluates ASDE with libscpl's bit-exact pairwise kernels.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .energy import MAXVAL


@dataclass(frozen=True)
class BufferPolicy:
    """buffering.py:26-43."""

    alpha: float = 0.2
    maxval: float = MAXVAL
    max_len: int = 64

    def __post_init__(self) -> None:
        if self.alpha <= 0:
            raise ValueError(f"alpha must be positive, got {self.alpha}")
        if self.max_len < 1:
            raise ValueError(f"max_len must be >= 1, got {self.max_len}")


def threshold(n: int, policy: BufferPolicy) -> float:
    """buffering.py:46-56: alpha*sqrt(((m - m/n)^2 + (n-1)(m/n)^2)/n)."""
    if n < 1:
        raise ValueError(f"buffer size must be >= 1, got {n}")
    m = policy.maxval
    step = m / n
    return policy.alpha * math.sqrt(((m - step) ** 2 + (n - 1) * step**2) / n)


@dataclass(eq=False)
class FixedRun:
    """buffering.py:59-71: a flushed buffer."""

    frames: list
    energy_maps: list

    def __len__(self) -> int:
        return len(self.frames)

    def uniform_energy(self) -> np.ndarray:
        """Per-pixel mean of the run's maps (sequential sum / T, on the GPU)."""
        return _stats_map(self.energy_maps, "mean")


def _stats_map(maps, what: str, sums=None):
    torch = _lib.torch_cuda()
    lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
    if sums is None:
        first = _lib.to_device(np.ascontiguousarray(maps[0], dtype=np.float64))
        S = first.clone()
        Q = torch.empty_like(S)
        _lib.check(lib.scpl_sums_start(cx, first.data_ptr(), S.numel(), S.data_ptr(), Q.data_ptr(), st))
        for m in maps[1:]:
            e = _lib.to_device(np.ascontiguousarray(m, dtype=np.float64))
            _lib.check(lib.scpl_sums_push(cx, e.data_ptr(), S.numel(), S.data_ptr(), Q.data_ptr(),
                                          S.data_ptr(), Q.data_ptr(), st))
        n = len(maps)
    else:
        S, Q, n = sums
    out = torch.empty_like(S)
    _lib.check(lib.scpl_sums_map(cx, S.data_ptr(), Q.data_ptr(), S.numel(), n, 0 if what == "mean" else 1,
                                 out.data_ptr(), st))
    return _lib.to_host(out)


@dataclass(eq=False)
class SpatioTemporalBuffer:
    """buffering.py:74-171: single-owner buffer of frames and energy maps with running stats."""

    policy: BufferPolicy = field(default_factory=BufferPolicy)
    frames: list = field(default_factory=list)
    energy_maps: list = field(default_factory=list)
    _sum: object = None
    _sum_sq: object = None
    last_candidate_asde: float | None = None

    def __len__(self) -> int:
        return len(self.frames)

    def push(self, frame: np.ndarray, energy: np.ndarray) -> FixedRun | None:
        arr = np.asarray(frame)
        emap = np.asarray(energy, dtype=np.float64)
        if emap.shape != arr.shape[:2]:
            raise ValueError(f"energy map shape {emap.shape} does not match frame {arr.shape[:2]}")
        if self.frames and arr.shape[:2] != self.frames[0].shape[:2]:
            raise ValueError(
                f"dimension mismatch: buffer holds {self.frames[0].shape[:2]}, got {arr.shape[:2]}")
        if not self.frames:
            self._start(arr, emap)
            return None
        torch = _lib.torch_cuda()
        lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
        n = len(self.frames) + 1
        e = _lib.to_device(np.ascontiguousarray(emap))
        cS = torch.empty_like(self._sum)
        cQ = torch.empty_like(self._sum)
        _lib.check(lib.scpl_sums_push(cx, e.data_ptr(), e.numel(), self._sum.data_ptr(), self._sum_sq.data_ptr(),
                                      cS.data_ptr(), cQ.data_ptr(), st))
        asde = ctypes.c_double()
        _lib.check(lib.scpl_asde_from_sums(cx, cS.data_ptr(), cQ.data_ptr(), e.numel(), n, ctypes.byref(asde), st))
        self.last_candidate_asde = float(asde.value)  # the value tested (buffering.py:118), for parity checks
        if asde.value <= threshold(n, self.policy) and n <= self.policy.max_len:
            self.frames.append(arr)
            self.energy_maps.append(emap)
            self._sum, self._sum_sq = cS, cQ
            return None
        run = FixedRun(frames=self.frames, energy_maps=self.energy_maps)
        self._start(arr, emap)
        return run

    def flush(self) -> FixedRun | None:
        if not self.frames:
            return None
        run = FixedRun(frames=self.frames, energy_maps=self.energy_maps)
        self.frames, self.energy_maps, self._sum, self._sum_sq = [], [], None, None
        return run

    def std_map(self) -> np.ndarray:
        self._require_nonempty()
        return _stats_map(None, "std", (self._sum, self._sum_sq, len(self.energy_maps))).reshape(
            self.energy_maps[0].shape)

    def pixel_std(self, i: int, j: int) -> float:
        return float(self.std_map()[i, j])

    def asde(self) -> float:
        self._require_nonempty()
        asde = ctypes.c_double()
        _lib.check(_lib.load().scpl_asde_from_sums(_lib.ctx(), self._sum.data_ptr(), self._sum_sq.data_ptr(),
                                                   self._sum.numel(), len(self.energy_maps), ctypes.byref(asde),
                                                   _lib.stream()))
        return float(asde.value)

    def uniform_energy(self) -> np.ndarray:
        self._require_nonempty()
        return _stats_map(None, "mean", (self._sum, self._sum_sq, len(self.energy_maps))).reshape(
            self.energy_maps[0].shape)

    def _start(self, frame, emap) -> None:
        torch = _lib.torch_cuda()
        self.frames = [frame]
        self.energy_maps = [emap]
        e = _lib.to_device(np.ascontiguousarray(emap))
        self._sum = torch.empty_like(e)
        self._sum_sq = torch.empty_like(e)
        _lib.check(_lib.load().scpl_sums_start(_lib.ctx(), e.data_ptr(), e.numel(), self._sum.data_ptr(),
                                               self._sum_sq.data_ptr(), _lib.stream()))

    def _require_nonempty(self) -> None:
        if not self.frames:
            raise ValueError("empty buffer")


__all__ = ["BufferPolicy", "threshold", "FixedRun", "SpatioTemporalBuffer"]
