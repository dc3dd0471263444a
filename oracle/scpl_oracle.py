"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the buffered SCPL retargeting path.

This module restates, with numpy, the reference algorithm of `vidcarve` 0.1.0
(`/root/reference/pkg/src/vidcarve`), function by function, each citing the
reference file:line it follows. It exists to CHECK the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package (``paper_1903_03180_b200``) never imports it and has no
  CPU fallback.

Pinning: tests/test_oracle_golden.py checks this module against golden
vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py``), plus the known-answer tests of the
reference's own suite (``pkg/tests/test_*.py``). Arithmetic that lives in
numpy/OpenBLAS (the luma matmul, the pairwise ``mean``) is restated in
``scpl_oracle.c`` and pinned the same way.

Replay is restated as one gather through the composed per-row index map; the
reference applies ``remove_batch`` batch by batch (pipeline.py:140-154). The
two are byte-identical because removed columns address the frame the batch
was selected on (batching.py:76-107); tests/test_oracle_golden.py checks it.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

MAXVAL = 255.0                              # energy.py:14
LUMA_WEIGHTS = np.array([0.299, 0.587, 0.114])  # energy.py:17

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def clib():
    """ctypes handle on oracle/_build/liboracle.so (built by oracle/Makefile)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        lib.oracle_luma.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        lib.oracle_pairwise_sum.argtypes = [ctypes.c_void_p, ctypes.c_long]
        lib.oracle_pairwise_sum.restype = ctypes.c_double
        lib.oracle_asde.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_int,
                                    ctypes.c_void_p]
        lib.oracle_asde.restype = ctypes.c_double
        lib.oracle_sobel.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        _LIB = lib
    return _LIB


# --------------------------------------------------------------------------- energy

def to_luma(frame: np.ndarray) -> np.ndarray:
    """energy.py:23-37: gray passes through; RGB -> rint(f64 dot BT.601) as uint8."""
    a = np.asarray(frame)
    if a.ndim == 2:
        return a
    if a.ndim == 3 and a.shape[2] == 1:
        return a[:, :, 0]
    if a.ndim == 3 and a.shape[2] == 3:
        return np.rint(a.astype(np.float64) @ LUMA_WEIGHTS).astype(np.uint8)
    raise ValueError(f"unsupported channel count: expected 1 or 3, got shape {a.shape}")


def to_luma_c(frame: np.ndarray) -> np.ndarray:
    """Same as to_luma via the C restatement of OpenBLAS's evaluation order."""
    a = np.ascontiguousarray(frame, dtype=np.uint8)
    out = np.empty(a.shape[:-1], dtype=np.uint8)
    clib().oracle_luma(a.ctypes.data, out.size, out.ctypes.data)
    return out


def gradient_energy(luma: np.ndarray) -> np.ndarray:
    """energy.py:40-59: edge-replicated Sobel |Gx|+|Gy| clamped to 255 (float64)."""
    y = np.asarray(luma)
    if y.ndim != 2:
        raise ValueError(f"expected a single-channel frame, got shape {y.shape}")
    h, w = y.shape
    if h < 3 or w < 3:
        raise ValueError(f"frame too small for 3x3 Sobel: {w}x{h}, need at least 3x3")
    pad = np.pad(y.astype(np.int32), 1, mode="edge")
    col = pad[:-2] + 2 * pad[1:-1] + pad[2:]          # vertical [1,2,1] smoothing
    row = pad[:, :-2] + 2 * pad[:, 1:-1] + pad[:, 2:]  # horizontal [1,2,1] smoothing
    gx = col[:, 2:] - col[:, :-2]
    gy = row[2:] - row[:-2]
    return np.minimum(np.abs(gx) + np.abs(gy), 255).astype(np.float64)


def motion_energy(curr, prev, w_motion=0.6, w_grad=0.4) -> np.ndarray:
    """energy.py:62-87: min(fl(fl(wm*|dL|) + fl(wg*grad)), 255); pure gradient if prev is None."""
    if w_motion < 0 or w_grad < 0 or abs(w_motion + w_grad - 1.0) > 1e-9:
        raise ValueError(f"weights must be non-negative and sum to 1, got {w_motion} + {w_grad}")
    lc = to_luma(curr)
    g = gradient_energy(lc)
    if prev is None:
        return g
    lp = to_luma(prev)
    if lp.shape != lc.shape:
        raise ValueError(f"dimension mismatch: current frame {lc.shape}, previous {lp.shape}")
    d = np.abs(lc.astype(np.float64) - lp.astype(np.float64))
    return np.minimum(w_motion * d + w_grad * g, MAXVAL)


def default_energy(frame) -> np.ndarray:
    """batching.py:110-115: gradient of the frame's luma; zero map below 3x3."""
    y = to_luma(frame)
    if min(y.shape) < 3:
        return np.zeros(y.shape, dtype=np.float64)
    return gradient_energy(y)


# --------------------------------------------------------------------------- DP / SCPL

def cumulative_energy(energy: np.ndarray):
    """seams.py:39-65: ce[i] = e[i] + min(ce[i-1][j-1..j+1]); first-minimum (leftmost delta) wins.

    Returns (ce float64 (h,w), back int8 (h,w)).
    """
    e = np.asarray(energy, dtype=np.float64)
    if e.ndim != 2 or e.size == 0:
        raise ValueError(f"expected a non-empty 2-d energy map, got shape {e.shape}")
    h, w = e.shape
    ce = np.empty((h, w))
    back = np.zeros((h, w), dtype=np.int8)
    ce[0] = e[0]
    inf = np.array([np.inf])
    for i in range(1, h):
        up = ce[i - 1]
        left = np.concatenate([inf, up[:-1]])
        right = np.concatenate([up[1:], inf])
        best = left.copy()
        delta = np.full(w, -1, dtype=np.int8)
        take = up < best                   # strict: ties keep the smaller delta
        best[take] = up[take]
        delta[take] = 0
        take = right < best
        best[take] = right[take]
        delta[take] = 1
        ce[i] = e[i] + best
        back[i] = delta
    return ce, back


def trace_columns(back: np.ndarray, last_cols) -> np.ndarray:
    """seams.py:68-81: (h, b) column offsets walked bottom-up."""
    h = back.shape[0]
    cols = np.asarray(last_cols, dtype=np.intp)
    out = np.empty((h, cols.size), dtype=np.intp)
    out[h - 1] = cols
    for i in range(h - 1, 0, -1):
        cols = cols + back[i, cols]
        out[i - 1] = cols
    return out


def label_parents(back: np.ndarray) -> np.ndarray:
    """batching.py:39-46: first-row landing column of every last-row column."""
    return trace_columns(back, np.arange(back.shape[1]))[0].copy()


def min_seam(ce, back):
    """seams.py:84-89: (offsets, cost) of the leftmost cheapest last-row pixel."""
    c = int(np.argmin(ce[-1]))
    return trace_columns(back, [c])[:, 0], float(ce[-1][c])


@dataclass
class Batch:
    """SeamBatch (batching.py:20-36) as arrays: cols (b,) last-row columns, costs (b,), offsets (h, b)."""
    cols: np.ndarray
    costs: np.ndarray
    offsets: np.ndarray
    source_width: int
    labels: np.ndarray | None = None  # label_parents of the pass (batch_carve keeps it for parity)

    def __len__(self):
        return int(self.cols.size)


def select_batch(ce, back, labels, k=None) -> Batch:
    """batching.py:49-73: per parent the leftmost strict-min child; keep the k cheapest by (cost, col)."""
    if k is not None and k < 1:
        raise ValueError(f"k must be >= 1 or None, got {k}")
    last = ce[-1]
    w = last.size
    labels = np.asarray(labels)
    starts = np.flatnonzero(np.r_[True, labels[1:] != labels[:-1]])  # labels are non-decreasing
    cols = []
    for a, b in zip(starts, np.r_[starts[1:], w]):
        cols.append(a + int(np.argmin(last[a:b])))  # argmin = first minimum = leftmost strict min
    cols = np.array(cols, dtype=np.intp)
    if k is not None and k < cols.size:
        order = np.lexsort((cols, last[cols]))[:k]
        cols = np.sort(cols[order])
    offsets = trace_columns(back, cols)
    return Batch(cols=cols, costs=last[cols].astype(np.float64), offsets=offsets, source_width=w)


def remove_batch(frame: np.ndarray, batch: Batch) -> np.ndarray:
    """batching.py:76-107: drop each row's batch columns, keep order."""
    a = np.asarray(frame)
    h, w = a.shape[:2]
    if w != batch.source_width:
        raise ValueError(f"batch was selected on width {batch.source_width}, frame has width {w}")
    if len(batch) == 0:
        return a.copy()
    keep = np.ones((h, w), dtype=bool)
    keep[np.arange(h)[:, None], batch.offsets] = False
    assert (~keep).sum(axis=1).max() == len(batch), "non-disjoint seam batch"
    rest = a[keep]
    return rest.reshape((h, w - len(batch)) + a.shape[2:])


def batch_carve(frame, target_width: int, energy=None, kmax: int | None = None):
    """batching.py:118-153 (kmax=1 gives the raw mode's one-seam-per-pass loop, pipeline.py:229-243).

    Returns (carved frame, [Batch...]).
    """
    a = np.asarray(frame)
    width = a.shape[1]
    if target_width < 1:
        raise ValueError(f"target width must be >= 1, got {target_width}")
    if target_width > width:
        raise ValueError(f"target width {target_width} exceeds frame width {width}")
    emap = energy
    batches = []
    cur = a
    while cur.shape[1] > target_width:
        if emap is None:
            emap = default_energy(cur)
        ce, back = cumulative_energy(emap)
        if kmax == 1:
            cols, cost = min_seam(ce, back)
            b = Batch(cols=np.array([cols[-1]]), costs=np.array([cost]), offsets=cols[:, None],
                      source_width=cur.shape[1])
        else:
            labels = label_parents(back)
            b = select_batch(ce, back, labels, k=cur.shape[1] - target_width)
            b.labels = labels
        cur = remove_batch(cur, b)
        batches.append(b)
        emap = None
    return cur, batches


def compose_index(h: int, w: int, batches) -> np.ndarray:
    """Per-row original-column index of every surviving column after all batches (int32 (h, w'))."""
    idx = np.broadcast_to(np.arange(w, dtype=np.int32), (h, w)).copy()
    for b in batches:
        keep = np.ones(idx.shape, dtype=bool)
        keep[np.arange(h)[:, None], b.offsets] = False
        idx = idx[keep].reshape(h, -1)
    return idx


def replay_gather(frames, idx: np.ndarray):
    """pipeline.py:140-154 restated as one gather per frame through the composed index map."""
    rows = np.arange(idx.shape[0])[:, None]
    return [np.ascontiguousarray(np.asarray(f)[rows, idx]) for f in frames]


def replay_batches(frames, batches):
    """pipeline.py:140-154 literally: remove every batch in order from every frame."""
    out = []
    for f in frames:
        cur = np.asarray(f)
        for b in batches:
            cur = remove_batch(cur, b)
        out.append(cur)
    return out


# --------------------------------------------------------------------------- temporal buffer

@dataclass(frozen=True)
class BufferPolicy:
    """buffering.py:26-43."""
    alpha: float = 0.2
    maxval: float = MAXVAL
    max_len: int = 64


def threshold(n: int, policy: BufferPolicy) -> float:
    """buffering.py:46-56: phi(n) = alpha*sqrt(((m - m/n)^2 + (n-1)(m/n)^2)/n)."""
    if n < 1:
        raise ValueError(f"buffer size must be >= 1, got {n}")
    m = policy.maxval
    step = m / n
    return policy.alpha * math.sqrt(((m - step) ** 2 + (n - 1) * step ** 2) / n)


def asde_from_sums(total, total_sq, n) -> float:
    """buffering.py:174-176: numpy pairwise mean of the per-pixel population std."""
    var = total_sq / n - (total / n) ** 2
    return float(np.sqrt(np.maximum(var, 0.0)).mean())


def asde_from_sums_c(total, total_sq, n) -> float:
    """asde_from_sums through the C restatement of numpy's pairwise sum."""
    S = np.ascontiguousarray(total, dtype=np.float64)
    Q = np.ascontiguousarray(total_sq, dtype=np.float64)
    work = np.empty(S.size)
    return clib().oracle_asde(S.ctypes.data, Q.ctypes.data, S.size, int(n), work.ctypes.data)


def pairwise_sum_c(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    return clib().oracle_pairwise_sum(a.ctypes.data, a.size)


@dataclass
class ScanTrace:
    """What the buffer scan decided: runs as (start, length) and each push's ASDE."""
    runs: list = field(default_factory=list)
    asde: list = field(default_factory=list)   # (frame index, n, asde, accepted)


def buffer_scan(emaps, policy: BufferPolicy, trace: ScanTrace | None = None):
    """SpatioTemporalBuffer.push/flush (buffering.py:93-138) over a stream of energy maps.

    Yields nothing; returns [(start, length), ...]. S and Q accumulate in stream
    order (buffering.py:116-117); a breach restarts with the breaching frame.
    """
    runs = []
    start, n_in, S, Q = 0, 0, None, None
    for t, e in enumerate(emaps):
        e = np.asarray(e, dtype=np.float64)
        if n_in == 0:
            start, n_in, S, Q = t, 1, e.copy(), e * e
            continue
        n = n_in + 1
        cS = S + e
        cQ = Q + e * e
        a = asde_from_sums(cS, cQ, n)
        ok = a <= threshold(n, policy) and n <= policy.max_len
        if trace is not None:
            trace.asde.append((t, n, a, ok))
        if ok:
            n_in, S, Q = n, cS, cQ
        else:
            runs.append((start, n_in))
            start, n_in, S, Q = t, 1, e.copy(), e * e
    if n_in:
        runs.append((start, n_in))
    if trace is not None:
        trace.runs = runs
    return runs


def uniform_energy(emaps) -> np.ndarray:
    """FixedRun.uniform_energy (buffering.py:69-71): stack-mean == sequential sum / T."""
    return np.stack([np.asarray(m, dtype=np.float64) for m in emaps]).mean(axis=0)


# --------------------------------------------------------------------------- pipeline

MODES = ("raw", "scpl", "buffered")


@dataclass
class Result:
    frames: list
    dp_passes: int
    runs: list
    wall_time: float
    batches: list   # per run: list over phases of [Batch, ...]


def _transpose(a):
    """seams.py:108-111."""
    return np.ascontiguousarray(np.swapaxes(np.asarray(a), 0, 1))


def _carve_run_reaverage(frames, target_width, energy):
    """pipeline.py:280-296: batch carve a whole run, re-averaging the gradient energy over
    every carved frame (np.stack(...).mean(0)) before each pass after the first."""
    cur = [np.asarray(f) for f in frames]
    batches = []
    emap = energy
    while cur[0].shape[1] > target_width:
        if emap is None:
            emap = np.stack([default_energy(f) for f in cur]).mean(axis=0)
        ce, back = cumulative_energy(emap)
        labels = label_parents(back)
        b = select_batch(ce, back, labels, k=cur[0].shape[1] - target_width)
        cur = [remove_batch(f, b) for f in cur]
        batches.append(b)
        emap = None
    return cur, batches


def _carve_frames(frames, tw, th, first_energy, height_first, kmax, literal_replay=False, reaverage=False):
    """_process_run / _retarget_single (pipeline.py:196-226, 246-277): width then height,
    the first carved phase on `first_energy`, later phases on gradient energy; the carve
    runs on frames[0] and is replayed on every frame of the group (reaverage: on the mean
    gradient of all the group's carved frames, pipeline.py:269-270)."""
    cur = list(frames)
    passes = 0
    emap = first_energy
    per_phase = []
    for axis in (("height", "width") if height_first else ("width", "height")):
        target = th if axis == "height" else tw
        size = cur[0].shape[0] if axis == "height" else cur[0].shape[1]
        if target >= size:
            continue
        work = [_transpose(f) for f in cur] if axis == "height" else cur
        pe = (_transpose(emap) if emap is not None else None) if axis == "height" else emap
        if reaverage:
            work, batches = _carve_run_reaverage(work, target, pe)
            passes += len(batches)
            per_phase.append(batches)
            cur = [_transpose(f) for f in work] if axis == "height" else work
            emap = None
            continue
        _, batches = batch_carve(work[0], target, energy=pe, kmax=kmax)
        if literal_replay:   # the reference's batch-by-batch remove_batch loop (timing fidelity)
            work = replay_batches(work, batches)
        else:
            idx = compose_index(work[0].shape[0], work[0].shape[1], batches)
            work = replay_gather(work, idx)
        passes += len(batches)
        per_phase.append(batches)
        cur = [_transpose(f) for f in work] if axis == "height" else work
        emap = None
    return cur, passes, per_phase


def _resolve(size, target, axis):
    if target is None:
        return size
    if target < 1:
        raise ValueError(f"target {axis} must be >= 1, got {target}")
    if target > size:
        raise ValueError(f"target {axis} {target} exceeds source {size} (reduction only)")
    return target


def retarget_video(frames, target_width=None, target_height=None, mode="buffered",
                   policy: BufferPolicy = BufferPolicy(), w_motion=0.6, w_grad=0.4,
                   height_first=False, keep_batches=False, literal_replay=False,
                   reaverage_energy=False) -> Result:
    """pipeline.py:92-137 (buffered, scpl, raw branches; reaverage_energy for buffered/scpl)."""
    t0 = time.perf_counter()
    frames = [np.asarray(f) for f in frames]
    if not frames:
        return Result([], 0, [], time.perf_counter() - t0, [])
    h, w = frames[0].shape[:2]
    if h < 3 or w < 3:
        raise ValueError(f"frame too small to carve: {w}x{h}, need at least 3x3")
    tw = _resolve(w, target_width, "width")
    th = _resolve(h, target_height, "height")
    for i, f in enumerate(frames):
        if f.shape[:2] != (h, w):
            raise ValueError(f"frame {i}: dimension change mid-stream, expected {(h, w)}, got {f.shape[:2]}")
    out, passes, all_batches = [], 0, []
    if mode == "raw":
        for f in frames:
            c, n, b = _carve_frames([f], tw, th, None, height_first, kmax=1, literal_replay=literal_replay)
            out += c
            passes += n
            all_batches.append(b if keep_batches else None)
        runs = [(t, 1) for t in range(len(frames))]
    else:
        emaps = [motion_energy(frames[0], None, w_motion, w_grad)]
        emaps += [motion_energy(f, p, w_motion, w_grad) for p, f in zip(frames, frames[1:])]
        if mode == "scpl":
            runs = [(t, 1) for t in range(len(frames))]
        else:
            runs = buffer_scan(emaps, policy)
        for s, n in runs:
            u = emaps[s] if n == 1 else uniform_energy(emaps[s:s + n])
            if mode == "scpl":
                u = emaps[s]
            c, p, b = _carve_frames(frames[s:s + n], tw, th, u, height_first, kmax=None,
                                    literal_replay=literal_replay, reaverage=reaverage_energy)
            out += c
            passes += p
            all_batches.append(b if keep_batches else None)
    return Result(out, passes, runs, time.perf_counter() - t0, all_batches)
