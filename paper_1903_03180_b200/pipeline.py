"""Retargeting orchestration -- drop-in for vidcarve.pipeline (pkg/src/vidcarve/pipeline.py).

retarget_video / retarget_image keep the reference signatures, validation order and
messages; the work (energy codes, buffer scan, carve, replay) runs inside
libscpl.so's scpl_retarget_video (one call per clip).

Besides numpy frame lists, retarget_video accepts a CUDA uint8 tensor (T, H, W[, C]);
the result is then a CUDA tensor (T, H', W'[, C]) and nothing touches the host.
"""

from __future__ import annotations

import ctypes
import os
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
    seams: dict | None = None  # seam-dump parity mode only (parse_seam_dump)


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


def _params(config: RetargetConfig, tw: int, th: int, shard=(0, 1), runs_in=None, scan_only=False):
    """scpl_video_params for a call (plus the ctypes buffers it points at, to keep alive)."""
    phi = _phi_table(config.policy)
    flat = [int(x) for r in (runs_in or ()) for x in r]
    runs_arr = (ctypes.c_int * max(1, len(flat)))(*flat) if runs_in is not None else None
    params = _lib.VideoParams(tw, th, _MODE_ID[config.mode], int(config.height_first), config.policy.max_len,
                              float(config.w_motion), float(config.w_grad),
                              ctypes.cast(phi, ctypes.POINTER(ctypes.c_double)), 0, int(config.reaverage_energy),
                              int(shard[0]), int(shard[1]),
                              ctypes.cast(runs_arr, ctypes.POINTER(ctypes.c_int)) if runs_arr is not None else None,
                              len(flat) // 2, int(scan_only))
    return params, (phi, runs_arr)


def _new_result(T: int, dump_cap: int = 0):
    starts = (ctypes.c_int * max(T, 1))()
    lens = (ctypes.c_int * max(T, 1))()
    res = _lib.VideoResult(0, 0, ctypes.cast(starts, ctypes.POINTER(ctypes.c_int)),
                           ctypes.cast(lens, ctypes.POINTER(ctypes.c_int)))
    dump = None
    if dump_cap:
        dump = np.empty(dump_cap, np.uint8)  # (pages are touched only where records land)
        res.seam_dump = dump.ctypes.data
        res.seam_dump_cap = dump_cap
    return res, (starts, lens, dump)


def _runs_of(res, keep) -> list:
    starts, lens = keep[0], keep[1]
    return [(starts[i], lens[i]) for i in range(res.n_runs)]


def _record_phases(res) -> None:
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


def _pad8(x: int) -> int:
    return (x + 7) & ~7


def parse_seam_dump(buf: np.ndarray, used: int) -> dict:
    """Records of the seam-dump parity mode (include/scpl.h, scpl_video_result) ->
    {(run, axis): [batch, ...]}, axis 0 = width, 1 = height, batches in carve order; each batch
    is a dict with what batch_carve decided (batching.py:118-153): "source_width", "cols"
    (last-row columns), "costs" (Seam.cost), "offsets" (rows x b, Seam.offsets as columns) and
    "labels" (label_parents of the pass, source_width entries)."""
    out = {}
    off = 0
    while off < used:
        run, axis, rows, cols, passes, removed = (int(x) for x in np.frombuffer(buf, np.int32, 6, off))
        off += 32
        sizes = np.frombuffer(buf, np.int32, passes, off)
        off += _pad8(4 * passes)
        last = np.frombuffer(buf, np.int16, removed, off)
        off += _pad8(2 * removed)
        costs = np.frombuffer(buf, np.float64, removed, off)
        off += 8 * removed
        offs = np.frombuffer(buf, np.int16, rows * removed, off).reshape(rows, removed)
        off += _pad8(2 * rows * removed)
        labs = np.frombuffer(buf, np.int16, passes * cols, off).reshape(passes, cols)
        off += _pad8(2 * passes * cols)
        batches, o, width = [], 0, cols
        for k, b in enumerate(sizes.tolist()):
            batches.append({"source_width": width, "cols": last[o:o + b].astype(np.int64),
                            "costs": costs[o:o + b].copy(), "offsets": offs[:, o:o + b].astype(np.int64),
                            "labels": labs[k, :width].astype(np.int64)})
            o += b
            width -= b
        out[(run, axis)] = batches
    return out


def _dump_cap(T: int, H: int, W: int, tw: int, th: int, nruns: int) -> int:
    cap = 0
    for rows, cols, tgt in ((H, W, tw), (W, H, th), (th, W, tw), (tw, H, th)):
        rem = cols - tgt
        if rem > 0:
            cap = max(cap, 32 + _pad8(4 * rem) + _pad8(2 * rem) + 8 * rem + _pad8(2 * rows * rem)
                      + _pad8(2 * rem * cols))
    return 2 * cap * max(nruns, 1) + 64


def _check_clip_tensor(clip, torch) -> None:
    if clip.dtype != torch.uint8:
        raise TypeError(f"expected a uint8 clip, got {clip.dtype}")
    if clip.dim() not in (3, 4):
        raise ValueError(f"expected a (T, H, W[, C]) clip, got shape {tuple(clip.shape)}")


def _run_device(clip, config: RetargetConfig, tw: int, th: int, out=None, shard=(0, 1), runs_in=None,
                scan_only=False, seam_dump=False):
    """Call libscpl on a uint8 clip (T, H, W, C); returns (out, dp, runs, seams).

    shard = (rank, count): carve only this rank's runs (sharding.py); dp counts those runs.
    runs_in: carve exactly these (start, len) runs (a previous scan's); scan_only: run boundaries
    only (out is None).  seam_dump: also return every batch of every run (parse_seam_dump).

    A CUDA clip goes through scpl_retarget_video (device in, device out).  A host clip goes
    through scpl_retarget_video_host, which streams it in chunks, overlaps the copies with the
    energy/scan kernels and ships every run's output frames back as soon as they are carved;
    clip and out should be pinned for the copies to run asynchronously.
    """
    torch = _lib.torch_cuda()
    _check_clip_tensor(clip, torch)
    T, H, W = clip.shape[:3]
    C = clip.shape[3] if clip.dim() == 4 else 1
    host = not clip.is_cuda
    dev = torch.cuda.current_device() if host else clip.device.index
    if seam_dump and config.mode == "buffered" and runs_in is None:
        runs_in = _run_device(clip, config, tw, th, scan_only=True)[2]  # sizes the dump exactly
    if scan_only:
        out = None
    elif out is None:
        out = (torch.empty((T, th, tw, C), dtype=torch.uint8, pin_memory=True) if host
               else torch.empty((T, th, tw, C), dtype=torch.uint8, device=clip.device))
    elif (tuple(out.shape) not in ((T, th, tw, C), (T, th, tw) if C == 1 else ()) or out.dtype != torch.uint8
          or out.is_cuda == host or not out.is_contiguous() or (not host and out.device != clip.device)):
        raise ValueError(f"out must be a contiguous uint8 {'host' if host else 'CUDA'} tensor of shape "
                         f"{(T, th, tw, C)}")
    params, keep_p = _params(config, tw, th, shard, runs_in, scan_only)
    res, keep_r = _new_result(T, _dump_cap(T, H, W, tw, th, len(runs_in) if runs_in is not None else T)
                              if seam_dump else 0)
    fn = _lib.load().scpl_retarget_video_host if host else _lib.load().scpl_retarget_video
    with torch.cuda.device(dev):
        _lib.check(fn(_lib.ctx(dev), clip.data_ptr(), T, H, W, C, ctypes.byref(params),
                      out.data_ptr() if out is not None else None, ctypes.byref(res), _lib.stream(dev)))
    runs = _runs_of(res, keep_r)
    _record_phases(res)
    seams = parse_seam_dump(keep_r[2], res.seam_dump_used) if seam_dump else None
    return out, int(res.dp_passes), runs, seams


last_phase_ms: dict = {}   # device time per phase of the last clip (bench instrumentation)


def _targets(clip, config):
    if clip.dim() not in (3, 4):
        raise ValueError(f"expected a (T, H, W[, C]) clip, got shape {tuple(clip.shape)}")
    _check_carvable(clip[0])
    _channels(tuple(clip.shape[1:]))
    H, W = clip.shape[1:3]
    return _resolve_target(W, config.target_width, "width"), _resolve_target(H, config.target_height, "height")


def retarget_video_tensor(clip, config: RetargetConfig, out=None, shard=None, runs=None, seam_dump=False):
    """Device-resident variant: clip is a CUDA uint8 tensor (T,H,W[,C]); returns (tensor, RunMetrics).

    Extensions: shard = (rank, count) (sharding.py): the whole scan runs, but only this rank's
    runs are carved and written; runs = [(start, len), ...] from an earlier scan_runs() of the same
    clip: exactly those runs are carved and written.  RunMetrics.dp_passes then counts those runs
    only.  seam_dump=True (parity mode): RunMetrics.seams = parse_seam_dump's record of every
    batch of every run."""
    start = time.perf_counter()
    if clip.dim() not in (3, 4):
        raise ValueError(f"expected a (T, H, W[, C]) clip, got shape {tuple(clip.shape)}")
    T = clip.shape[0]
    if T == 0:
        return clip[:0], RunMetrics(0, time.perf_counter() - start, 0)
    tw, th = _targets(clip, config)
    out, dp, runs_out, seams = _run_device(clip.contiguous(), config, tw, th, out=out, shard=shard or (0, 1),
                                           runs_in=runs, seam_dump=seam_dump)
    if clip.dim() == 3 and out.dim() == 4:
        out = out[..., 0]
    return out, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=T, runs=runs_out,
                           seams=seams)


def scan_runs(clip, config: RetargetConfig) -> list:
    """The buffer scan alone (buffering.py:93-138 over the clip): the (start, len) runs that
    retarget_video would carve, for a uint8 clip tensor (CUDA or host)."""
    if config.mode != "buffered":
        return [(t, 1) for t in range(clip.shape[0])]
    if clip.shape[0] == 0:
        return []
    tw, th = _targets(clip, config)
    return _run_device(clip.contiguous(), config, tw, th, scan_only=True)[2]


def _retarget_host_tensor(clip, config: RetargetConfig, out=None, seam_dump=False):
    """Host (ideally pinned) uint8 tensor (T,H,W[,C]) in, host tensor out (pinned, or `out`).

    The host<->device copies overlap the kernels inside libscpl (scpl_retarget_video_host)."""
    start = time.perf_counter()
    if clip.dim() not in (3, 4):
        raise ValueError(f"expected a (T, H, W[, C]) clip, got shape {tuple(clip.shape)}")
    T = clip.shape[0]
    if T == 0:
        return clip[:0], RunMetrics(0, time.perf_counter() - start, 0)
    tw, th = _targets(clip, config)
    res, dp, runs, seams = _run_device(clip.contiguous(), config, tw, th, out=out, seam_dump=seam_dump)
    if clip.dim() == 3 and res.dim() == 4:
        res = res[..., 0]
    return res, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=T, runs=runs,
                           seams=seams)


def _as_u8_frame(arr: np.ndarray, idx: int) -> np.ndarray:
    """uint8 view of a frame; integer frames with values in 0..255 are converted exactly (the
    reference computes on their values, energy.py:34-35, and keeps the dtype, batching.py:100)."""
    if arr.dtype == np.uint8:
        return arr
    if arr.dtype.kind in "iub" and (arr.size == 0 or (arr.min() >= 0 and arr.max() <= 255)):
        return arr.astype(np.uint8)
    raise ValueError(f"frame {idx}: expected uint8 pixels (or integers in 0..255), got {arr.dtype}")


def _admit_frames(frames, config):
    """_admit (pipeline.py:157-171) over a frame list: (arrays, targets)."""
    arrs = []
    shape = None
    targets = None
    for idx, frame in enumerate(frames):
        arr = np.asarray(frame)
        if shape is None:
            _check_carvable(arr)
            shape = arr.shape[:2]
            targets = (_resolve_target(shape[1], config.target_width, "width"),
                       _resolve_target(shape[0], config.target_height, "height"))
        elif arr.shape[:2] != shape:
            raise ValueError(
                f"frame {idx}: dimension change mid-stream, expected {shape}, got {arr.shape[:2]}")
        _channels(arr.shape)
        arrs.append(arr)
    return arrs, targets


def _stack_pinned(arrs):
    """Pinned (T, H, W, C) uint8 host tensor of the frames, plus how to give each output frame back
    its own layout.  A clip that mixes gray and RGB frames is carved as RGB with the gray frames
    replicated to three channels: luma(v, v, v) == v exactly, so every energy, seam and output
    pixel is the reference's (which handles each frame's layout on its own, energy.py:30-37,
    batching.py:100-101); the gray frames' outputs are channel 0 of theirs."""
    torch = _lib.torch_cuda()
    chans = {(a.ndim, a.shape[2] if a.ndim == 3 else 1) for a in arrs}
    mixed = len(chans) > 1
    C = 3 if mixed else (arrs[0].shape[2] if arrs[0].ndim == 3 else 1)
    T = len(arrs)
    h, w = arrs[0].shape[:2]
    host = torch.empty((T, h, w, C), dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()

    def put(t):
        a8 = _as_u8_frame(arrs[t], t)
        if a8.ndim == 2:
            a8 = a8[:, :, None]
        hv[t] = a8  # (broadcasts a gray frame over three channels when mixed)

    if T * h * w * C >= (64 << 20):  # large clips: the host copy in parallel (numpy releases the GIL)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(put, range(T)))
    else:
        for t in range(T):
            put(t)
    return host


def _unstack(rv, arrs):
    out = []
    for t, a in enumerate(arrs):
        f = rv[t]
        if a.ndim == 2:
            f = f[..., 0]
        elif a.shape[2] == 1 and f.shape[2] != 1:
            f = f[..., :1]
        if a.dtype != np.uint8:
            f = f.astype(a.dtype)
        out.append(f)
    return out


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
    arrs, targets = _admit_frames(frames, config)
    if not arrs:
        return [], RunMetrics(dp_passes=0, wall_time=time.perf_counter() - start, frames_out=0)
    tw, th = targets
    T = len(arrs)
    host = _stack_pinned(arrs)
    res, dp, runs, _ = _run_device(host, config, tw, th)
    frames_out = _unstack(res.numpy(), arrs)
    return frames_out, RunMetrics(dp_passes=dp, wall_time=time.perf_counter() - start, frames_out=T, runs=runs)


def retarget_videos(clips, config: RetargetConfig, outs=None, seam_dump=False):
    """Many independent clips of one shape in one call (BASELINE config C4; libscpl
    scpl_retarget_batch): identical results to one retarget_video per clip, but every clip's
    codes and buffer scan run at once and closed runs of all clips share carve groups.

    clips: CUDA uint8 tensors (T, H, W[, C]) -> CUDA outputs; host uint8 tensors (ideally
    pinned) -> pinned host outputs; or frame lists (numpy) -> frame lists.  Returns a list of
    (output, RunMetrics), one per clip."""
    torch = _lib.torch_cuda()
    clips = list(clips)
    if not clips:
        return []
    start = time.perf_counter()
    lists = not isinstance(clips[0], torch.Tensor)
    arrs_per = None
    if lists:
        arrs_per = [_admit_frames(c, config)[0] for c in clips]
        if any(len(a) == 0 for a in arrs_per):
            raise ValueError("every clip needs at least one frame")
        tens = [_stack_pinned(a) for a in arrs_per]
    else:
        tens = [c if c.dim() == 4 else c.unsqueeze(-1) for c in clips]
    for c in tens:
        _check_clip_tensor(c, torch)
    shape, host = tuple(tens[0].shape), not tens[0].is_cuda
    if any(tuple(c.shape) != shape or (not c.is_cuda) != host for c in tens):
        raise ValueError("retarget_videos needs clips of one shape, all on the device or all on the host")
    if not host and any(c.device != tens[0].device for c in tens):
        raise ValueError("retarget_videos needs every CUDA clip on one device")
    tens = [c.contiguous() for c in tens]
    T, H, W, C = shape
    tw, th = _targets(tens[0], config)
    dev = torch.cuda.current_device() if host else tens[0].device.index
    n = len(tens)
    if outs is None:
        outs = [torch.empty((T, th, tw, C), dtype=torch.uint8, pin_memory=True) if host
                else torch.empty((T, th, tw, C), dtype=torch.uint8, device=tens[0].device) for _ in range(n)]
    else:
        outs = [o if o.dim() == 4 else o.unsqueeze(-1) for o in outs]
        if len(outs) != n or any(tuple(o.shape) != (T, th, tw, C) or o.dtype != torch.uint8 or o.is_cuda == host
                                 or not o.is_contiguous() for o in outs):
            raise ValueError(f"outs must be {n} contiguous uint8 {'host' if host else 'CUDA'} tensors of shape "
                             f"{(T, th, tw, C)}")
    params, keep_p = _params(config, tw, th)
    results = (_lib.VideoResult * n)()
    keeps = []
    for i in range(n):
        nr = (len(scan_runs(tens[i], config)) if config.mode == "buffered" else T) if seam_dump else 0
        r, k = _new_result(T, _dump_cap(T, H, W, tw, th, nr) if seam_dump else 0)
        results[i] = r
        keeps.append(k)
    cp = (ctypes.c_void_p * n)(*[c.data_ptr() for c in tens])
    op = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
    with torch.cuda.device(dev):
        _lib.check(_lib.load().scpl_retarget_batch(_lib.ctx(dev), n, cp, T, H, W, C, ctypes.byref(params), op,
                                                   results, int(host), _lib.stream(dev)))
    _record_phases(results[0])
    wall = time.perf_counter() - start
    ret = []
    for i in range(n):
        res = results[i]
        seams = parse_seam_dump(keeps[i][2], res.seam_dump_used) if seam_dump else None
        m = RunMetrics(dp_passes=int(res.dp_passes), wall_time=wall, frames_out=T, runs=_runs_of(res, keeps[i]),
                       seams=seams)
        o = outs[i]
        if lists:
            o = _unstack(o.numpy(), arrs_per[i])
        elif clips[i].dim() == 3:
            o = o[..., 0]
        ret.append((o, m))
    return ret


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
    out, dp, _, _ = _run_device(clip, cfg, tw, th)
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
           "retarget_videos", "scan_runs", "parse_seam_dump", "replay_batches"]
