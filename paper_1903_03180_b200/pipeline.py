"""Retargeting orchestration -- drop-in for vidcarve.pipeline (pkg/src/vidcarve/pipeline.py).

retarget_video / retarget_image keep the reference signatures, validation order and
messages; the work (energy codes, buffer scan, carve, replay) runs inside
libscpl.so's scpl_retarget_video (one call per clip).

Besides numpy frame lists, retarget_video accepts a CUDA uint8 tensor (T, H, W[, C]);
the result is then a CUDA tensor (T, H', W'[, C]) and nothing touches the host.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Iterable

import numpy as np

from . import _lib
from .buffering import BufferPolicy, threshold
from .energy import DEFAULT_GRADIENT_WEIGHT, DEFAULT_MOTION_WEIGHT
from .seams import transpose

MODES = ("raw", "scpl", "buffered")     # pipeline.py:39
_MODE_ID = {"raw": 0, "scpl": 1, "buffered": 2}


@dataclass
class RetargetConfig:
    """pipeline.py:42-67."""

    target_width: int | None = None
    target_height: int | None = None
    mode: str = "scpl"
    policy: BufferPolicy = field(default_factory=BufferPolicy)
    w_motion: float = DEFAULT_MOTION_WEIGHT
    w_grad: float = DEFAULT_GRADIENT_WEIGHT
    reaverage_energy: bool = False
    height_first: bool = False

    def __post_init__(self) -> None:
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}, expected one of {MODES}")
        if self.w_motion < 0 or self.w_grad < 0 or abs(self.w_motion + self.w_grad - 1.0) > 1e-9:
            raise ValueError(
                f"weights must be non-negative and sum to 1, got {self.w_motion} + {self.w_grad}")


@dataclass
class RunMetrics:
    """pipeline.py:70-77 (+ the run boundaries the buffer chose, for inspection)."""

    dp_passes: int = 0
    wall_time: float = 0.0
    frames_out: int = 0
    jitter: float | None = None
    runs: list = field(default_factory=list)


def _check_carvable(arr) -> None:
    """pipeline.py:174-179."""
    if arr.ndim not in (2, 3):
        raise ValueError(f"expected a 2-d or 3-d frame array, got shape {arr.shape}")
    h, w = arr.shape[:2]
    if h < 3 or w < 3:
        raise ValueError(f"frame too small to carve: {w}x{h}, need at least 3x3")


def _resolve_target(size: int, target: int | None, axis: str) -> int:
    """pipeline.py:182-189."""
    if target is None:
        return size
    if target < 1:
        raise ValueError(f"target {axis} must be >= 1, got {target}")
    if target > size:
        raise ValueError(f"target {axis} {target} exceeds source {size} (reduction only)")
    return target


def _channels(shape) -> int:
    if len(shape) == 2:
        return 1
    if shape[2] in (1, 3):
        return shape[2]
    raise ValueError(f"unsupported channel count: expected 1 or 3, got shape {tuple(shape)}")


def _phi_table(policy: BufferPolicy):
    """threshold(n) for n = 0..max_len, exactly as buffering.py:46-56 computes it."""
    vals = [0.0] + [threshold(n, policy) for n in range(1, policy.max_len + 1)]
    return (ctypes.c_double * len(vals))(*vals)


def _run_device(clip, config: RetargetConfig, tw: int, th: int, out=None, shard=(0, 1)):
    """Call libscpl on a uint8 clip (T, H, W, C); returns (out, dp, runs).

    shard = (rank, count): carve only this rank's runs (sharding.py); dp counts those runs.

    A CUDA clip goes through scpl_retarget_video (device in, device out).  A host clip goes
    through scpl_retarget_video_host, which streams it in chunks, overlaps the copies with the
    energy/scan kernels and ships every run's output frames back as soon as they are carved;
    clip and out should be pinned for the copies to run asynchronously.
    """
    torch = _lib.torch_cuda()
    T, H, W = clip.shape[:3]
    C = clip.shape[3] if clip.dim() == 4 else 1
    host = not clip.is_cuda
    if out is None:
        out = (torch.empty((T, th, tw, C), dtype=torch.uint8, pin_memory=True) if host
               else torch.empty((T, th, tw, C), dtype=torch.uint8, device=clip.device))
    elif (tuple(out.shape) not in ((T, th, tw, C), (T, th, tw) if C == 1 else ()) or out.dtype != torch.uint8
          or out.is_cuda == host or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous uint8 {'host' if host else 'CUDA'} tensor of shape "
                         f"{(T, th, tw, C)}")
    phi = _phi_table(config.policy)
    params = _lib.VideoParams(tw, th, _MODE_ID[config.mode], int(config.height_first), config.policy.max_len,
                              float(config.w_motion), float(config.w_grad),
                              ctypes.cast(phi, ctypes.POINTER(ctypes.c_double)), 0, int(config.reaverage_energy),
                              int(shard[0]), int(shard[1]))
    starts = (ctypes.c_int * max(T, 1))()
    lens = (ctypes.c_int * max(T, 1))()
    res = _lib.VideoResult(0, 0, ctypes.cast(starts, ctypes.POINTER(ctypes.c_int)),
                           ctypes.cast(lens, ctypes.POINTER(ctypes.c_int)))
    fn = _lib.load().scpl_retarget_video_host if host else _lib.load().scpl_retarget_video
    dev = torch.cuda.current_device() if host else clip.device.index
    _lib.check(fn(_lib.ctx(dev), clip.data_ptr(), T, H, W, C, ctypes.byref(params), out.data_ptr(),
                  ctypes.byref(res), _lib.stream()))
    runs = [(starts[i], lens[i]) for i in range(res.n_runs)]
    global last_phase_ms
    # device time from the call's start: codes done, scan done, every group carved + replayed
    # (the groups overlap the scan; the last one finishes carve_after_scan ms after it)
    last_phase_ms = dict(zip(("codes", "scan", "carve_after_scan"), (float(x) for x in res.phase_ms[:3])))
    # device clock cycles of the slowest run's pass kernels (dp rows / select+trace), summed
    last_phase_ms.update({f"carve_{k}_Mcyc": c / 1e6 for k, c in zip(("dp", "select"), res.carve_cycles[:2])})
    last_phase_ms["slowest_run_iters"] = int(res.carve_cycles[2])
    last_phase_ms["carve_cluster"] = res.carve_cluster
    last_phase_ms["pass_launches"] = int(res.carve_cycles[3])
    last_phase_ms["pass_launch_ms"] = float(res.phase_ms[3])
    last_phase_ms["scan_windows"] = int(res.scan_windows)
    last_phase_ms["scan_fallbacks"] = int(res.scan_fallbacks)
    return out, int(res.dp_passes), runs


last_phase_ms: dict = {}   # device time per phase of the last clip (bench instrumentation)


def retarget_video_tensor(clip, config: RetargetConfig, out=None, shard=None):
    """Device-resident variant: clip is a CUDA uint8 tensor (T,H,W[,C]); returns (tensor, RunMetrics).

    shard = (rank, count) (extension, sharding.py): the whole scan runs, but only this rank's runs
    are carved and written; RunMetrics.dp_passes then counts those runs only."""
    start = time.perf_counter()
    if clip.dim() not in (3, 4):
        raise ValueError(f"expected a (T, H, W[, C]) clip, got shape {tuple(clip.shape)}")
    T = clip.shape[0]
    if T == 0:
        return clip[:0], RunMetrics(0, time.perf_counter() - start, 0)
    _check_carvable(clip[0])
    _channels(tuple(clip.shape[1:]))
    H, W = clip.shape[1:3]
    tw = _resolve_target(W, config.target_width, "width")
    th = _resolve_target(H, config.target_height, "height")
    out, dp, runs = _run_device(clip.contiguous(), config, tw, th, out=out, shard=shard or (0, 1))
    if clip.dim() == 3 and out.dim() == 4:
        out = out[..., 0]
    return out, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=T, runs=runs)


def _retarget_host_tensor(clip, config: RetargetConfig, out=None):
    """Host (ideally pinned) uint8 tensor (T,H,W[,C]) in, host tensor out (pinned, or `out`).

    The host<->device copies overlap the kernels inside libscpl (scpl_retarget_video_host)."""
    start = time.perf_counter()
    if clip.dim() not in (3, 4):
        raise ValueError(f"expected a (T, H, W[, C]) clip, got shape {tuple(clip.shape)}")
    T = clip.shape[0]
    if T == 0:
        return clip[:0], RunMetrics(0, time.perf_counter() - start, 0)
    _check_carvable(clip[0])
    _channels(tuple(clip.shape[1:]))
    H, W = clip.shape[1:3]
    tw = _resolve_target(W, config.target_width, "width")
    th = _resolve_target(H, config.target_height, "height")
    res, dp, runs = _run_device(clip.contiguous(), config, tw, th, out=out)
    if clip.dim() == 3 and res.dim() == 4:
        res = res[..., 0]
    return res, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=T, runs=runs)


def retarget_video(frames: Iterable[np.ndarray], config: RetargetConfig, out=None):
    """pipeline.py:92-137: carve a stream of frames; output count always equals input count.

    `out` (extension): a preallocated output tensor for tensor inputs (pinned host tensor for a
    host clip, CUDA tensor for a CUDA clip)."""
    torch = None
    try:
        import torch  # noqa: F401
    except ImportError:  # pragma: no cover
        pass
    if torch is not None and isinstance(frames, torch.Tensor):
        if frames.is_cuda:
            return retarget_video_tensor(frames, config, out=out)
        return _retarget_host_tensor(frames, config, out=out)
    start = time.perf_counter()
    arrs = []
    shape = None
    targets = None
    for idx, frame in enumerate(frames):   # _admit, pipeline.py:157-171
        arr = np.asarray(frame)
        if shape is None:
            _check_carvable(arr)
            shape = arr.shape[:2]
            targets = (_resolve_target(shape[1], config.target_width, "width"),
                       _resolve_target(shape[0], config.target_height, "height"))
        elif arr.shape[:2] != shape:
            raise ValueError(
                f"frame {idx}: dimension change mid-stream, expected {shape}, got {arr.shape[:2]}")
        arrs.append(arr)
    if not arrs:
        return [], RunMetrics(dp_passes=0, wall_time=time.perf_counter() - start, frames_out=0)
    c0 = _channels(arrs[0].shape)
    for a in arrs[1:]:
        if _channels(a.shape) != c0 or a.ndim != arrs[0].ndim:
            raise ValueError("all frames of a clip must have the same channel layout")
    tw, th = targets
    T = len(arrs)
    torch = _lib.torch_cuda()
    host = torch.empty((T,) + tuple(arrs[0].shape), dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    for t, a in enumerate(arrs):
        hv[t] = a
    if host.dim() == 3:
        host = host.unsqueeze(-1)
    res, dp, runs = _run_device(host, config, tw, th)
    rv = res.numpy()
    if arrs[0].ndim == 2:
        rv = rv[..., 0]
    frames_out = [rv[t] for t in range(T)]
    return frames_out, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=T, runs=runs)


def retarget_image(frame: np.ndarray, config: RetargetConfig):
    """pipeline.py:80-89: carve a single frame to the configured targets.

    _retarget_single with initial_energy=None (pipeline.py:196-226) equals a one-frame
    scpl (or raw) video: the first frame's motion energy is its pure gradient, which is
    default_energy for any carvable (>= 3x3) frame.
    """
    start = time.perf_counter()
    arr = np.asarray(frame)
    _check_carvable(arr)
    tw = _resolve_target(arr.shape[1], config.target_width, "width")
    th = _resolve_target(arr.shape[0], config.target_height, "height")
    _channels(arr.shape)
    cfg = RetargetConfig(target_width=tw, target_height=th, mode="raw" if config.mode == "raw" else "scpl",
                         policy=config.policy, w_motion=config.w_motion, w_grad=config.w_grad,
                         height_first=config.height_first)
    clip = _lib.to_device(np.ascontiguousarray(arr, dtype=np.uint8)[None])
    if clip.dim() == 3:
        clip = clip.unsqueeze(-1)
    out, dp, _ = _run_device(clip, cfg, tw, th)
    res = _lib.to_host(out[0])
    if arr.ndim == 2:
        res = res[..., 0]
    return res, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=1)


def replay_batches(run_frames, batches):
    """pipeline.py:140-154: apply recorded batches, in order, to every frame of a run."""
    from .batching import remove_batch
    out = []
    for frame in run_frames:
        cur = np.asarray(frame)
        for batch in batches:
            cur = remove_batch(cur, batch)
        out.append(cur)
    return out


__all__ = ["MODES", "RetargetConfig", "RunMetrics", "retarget_image", "retarget_video", "retarget_video_tensor",
           "replay_batches"]
