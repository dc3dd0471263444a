"""Batched seam removal via parental labeling -- drop-in for vidcarve.batching
(pkg/src/vidcarve/batching.py).

batch_carve runs its whole DP -> label -> select -> remove loop inside libscpl.so
(scpl_batch_carve, the same kernels as the video path); the table-level functions
(label_parents, select_batch, remove_batch) have their own kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .energy import gradient_energy, to_luma
from .seams import DpTables, Seam, trace_columns


@dataclass(frozen=True, eq=False)
class SeamBatch:
    """batching.py:20-36: pairwise-disjoint vertical seams, sorted by last-row column."""

    seams: tuple
    source_width: int | None = None

    def __len__(self) -> int:
        return len(self.seams)

    def __iter__(self):
        return iter(self.seams)


def label_parents(tables: DpTables) -> np.ndarray:
    """batching.py:39-46: first-row landing column for every last-row column."""
    torch = _lib.torch_cuda()
    back = np.ascontiguousarray(tables.back, dtype=np.int8)
    h, w = back.shape
    bd = _lib.to_device(back)
    lab = torch.empty(w, dtype=torch.int64, device=bd.device)
    _lib.check(_lib.load().scpl_label_parents(_lib.ctx(), bd.data_ptr(), h, w, lab.data_ptr(), _lib.stream()))
    return _lib.to_host(lab).astype(np.intp, copy=False)


def _select_cols(last: np.ndarray, labels: np.ndarray, k: int | None):
    torch = _lib.torch_cuda()
    last = np.ascontiguousarray(last, dtype=np.float64)
    w = last.size
    ld = _lib.to_device(last)
    lab = _lib.to_device(np.ascontiguousarray(labels, dtype=np.int64))
    cols = torch.empty(w, dtype=torch.int64, device=ld.device)
    costs = torch.empty(w, dtype=torch.float64, device=ld.device)
    nb = ctypes.c_int()
    _lib.check(_lib.load().scpl_select_batch(_lib.ctx(), ld.data_ptr(), lab.data_ptr(), w, 0 if k is None else k,
                                             cols.data_ptr(), costs.data_ptr(), ctypes.byref(nb), _lib.stream()))
    n = nb.value
    return _lib.to_host(cols[:n]).astype(np.intp), _lib.to_host(costs[:n])


def select_batch(tables: DpTables, labels: np.ndarray, k: int | None = None) -> SeamBatch:
    """batching.py:49-73: one cheapest child per parent, optionally the k cheapest by (cost, col)."""
    if k is not None and k < 1:
        raise ValueError(f"k must be >= 1 or None, got {k}")
    last = np.asarray(tables.ce)[-1]
    cols, costs = _select_cols(last, labels, k)
    offsets = trace_columns(tables.back, cols)
    seams = tuple(Seam(offsets=offsets[:, i].copy(), cost=float(costs[i])) for i in range(cols.size))
    return SeamBatch(seams=seams, source_width=int(last.size))


def _remove_offsets(arr: np.ndarray, offs: np.ndarray):
    """Remove per-row columns offs (b, h) on the GPU; returns (out, max removed per row).

    Any dtype and channel count (the reference's removal is dtype-generic, batching.py:100-107):
    a pixel is moved as its raw bytes, so the output keeps the input's dtype and values."""
    torch = _lib.torch_cuda()
    arr = np.ascontiguousarray(arr)
    h, w = arr.shape[:2]
    bpp = arr.dtype.itemsize * int(np.prod(arr.shape[2:], dtype=np.int64))  # bytes per pixel
    b = offs.shape[0]
    src = _lib.to_device(arr.view(np.uint8).reshape(h, w, bpp))
    od = _lib.to_device(np.ascontiguousarray(offs, dtype=np.int64))
    out = torch.empty((h, w - b, bpp), dtype=torch.uint8, device=src.device)
    cnt = torch.empty(h, dtype=torch.int32, device=src.device)
    _lib.check(_lib.load().scpl_remove_columns(_lib.ctx(), src.data_ptr(), h, w, bpp, od.data_ptr(), b,
                                               out.data_ptr(), cnt.data_ptr(), _lib.stream()))
    res = _lib.to_host(out).view(arr.dtype).reshape((h, w - b) + arr.shape[2:])
    return res, int(cnt.max().item()) if h else 0


def remove_batch(frame: np.ndarray, batch: SeamBatch) -> np.ndarray:
    """batching.py:76-107: remove every seam of the batch in one pass."""
    arr = np.asarray(frame)
    h, w = arr.shape[:2]
    if batch.source_width is not None and w != batch.source_width:
        raise ValueError(f"batch was selected on width {batch.source_width}, frame has width {w}")
    if len(batch) == 0:
        return arr.copy()
    offs = []
    for seam in batch:
        o = np.asarray(seam.offsets)
        if o.shape != (h,):
            raise ValueError(f"seam length {o.shape} does not match frame height {h}")
        if (o < 0).any() or (o >= w).any():
            raise ValueError(f"seam offset out of range for width {w}")
        offs.append(o)
    out, most = _remove_offsets(arr, np.stack(offs))
    assert most == len(batch), "non-disjoint seam batch"
    return out


def default_energy(frame: np.ndarray) -> np.ndarray:
    """batching.py:110-115."""
    luma = to_luma(frame)
    if min(luma.shape) < 3:
        return np.zeros(luma.shape, dtype=np.float64)
    return gradient_energy(luma)


def batch_carve(frame: np.ndarray, target_width: int, energy: np.ndarray | None = None,
                energy_fn=default_energy, kmax: int | None = None):
    """batching.py:118-153: carve to target_width in batches; returns (carved, [SeamBatch]).

    The loop runs on the GPU with the reference's default energy (gradient of the carved
    frame); ``kmax=1`` is raw mode's one-seam-per-pass loop (pipeline.py:229-243).
    """
    arr = np.asarray(frame)
    width = arr.shape[1]
    if target_width < 1:
        raise ValueError(f"target width must be >= 1, got {target_width}")
    if target_width > width:
        raise ValueError(f"target width {target_width} exceeds frame width {width}")
    if energy is not None and np.asarray(energy).shape != arr.shape[:2]:
        raise ValueError(f"energy map shape {np.asarray(energy).shape} does not match frame {arr.shape[:2]}")
    c = 1 if arr.ndim == 2 else arr.shape[2]
    integral = arr.dtype == np.uint8 or (arr.dtype.kind in "iub" and (arr.size == 0 or (
        int(arr.min()) >= 0 and int(arr.max()) <= 255)))
    if energy_fn is not default_energy or c not in (1, 3) or arr.ndim > 3 or not integral:
        # the reference loop (batching.py:144-152) over the GPU primitives, with the caller's
        # energy function evaluated on the host each pass and its map uploaded
        return _batch_carve_loop(arr, target_width, energy, energy_fn, kmax)
    if arr.dtype != np.uint8:  # exact: the values are bytes; the output keeps the input's dtype
        carved, batches = batch_carve(arr.astype(np.uint8), target_width, energy=energy, kmax=kmax)
        return carved.astype(arr.dtype), batches
    torch = _lib.torch_cuda()
    h, w = arr.shape[:2]
    src = _lib.to_device(np.ascontiguousarray(arr, dtype=np.uint8))
    ed = _lib.to_device(np.ascontiguousarray(energy, dtype=np.float64)) if energy is not None else None
    index = torch.empty((h, target_width), dtype=torch.int16, device=src.device)
    nb = ctypes.c_int()
    sizes = np.zeros(max(w, 1), dtype=np.int32)
    cols = np.zeros(max(w, 1), dtype=np.int16)
    costs = np.zeros(max(w, 1), dtype=np.float64)
    offsets = np.zeros((max(w, 1), h), dtype=np.int16)
    _lib.check(_lib.load().scpl_batch_carve(
        _lib.ctx(), src.data_ptr(), h, w, c, target_width, _lib.ptr(ed), 1 if kmax == 1 else 0, index.data_ptr(),
        ctypes.byref(nb), sizes.ctypes.data, cols.ctypes.data, costs.ctypes.data, offsets.ctypes.data,
        _lib.stream()))
    batches = []
    pos, cur_w = 0, w
    for k in range(nb.value):
        b = int(sizes[k])
        seams = tuple(Seam(offsets=offsets[pos + s].astype(np.intp), cost=float(costs[pos + s])) for s in range(b))
        batches.append(SeamBatch(seams=seams, source_width=cur_w))
        pos += b
        cur_w -= b
    carved = torch.empty((h, target_width) + arr.shape[2:], dtype=torch.uint8, device=src.device)
    _lib.check(_lib.load().scpl_replay(_lib.ctx(), src.data_ptr(), 1, h, w, c, index.data_ptr(), target_width,
                                       target_width, 0, carved.data_ptr(), _lib.stream()))
    return _lib.to_host(carved), batches


def _batch_carve_loop(arr, target_width, energy, energy_fn, kmax):
    """batching.py:144-152 step by step: energy (the given map, then energy_fn of the carved
    frame) -> cumulative_energy -> label_parents -> select_batch -> remove_batch, each on the GPU."""
    from .seams import cumulative_energy, min_seam
    cur = arr
    emap = energy
    batches = []
    while cur.shape[1] > target_width:
        if emap is None:
            emap = energy_fn(cur)
        tables = cumulative_energy(np.asarray(emap, dtype=np.float64))
        if kmax == 1:  # raw mode (pipeline.py:236-242)
            batch = SeamBatch(seams=(min_seam(tables),), source_width=int(cur.shape[1]))
        else:
            labels = label_parents(tables)
            batch = select_batch(tables, labels, k=cur.shape[1] - target_width)
        cur = remove_batch(cur, batch)
        batches.append(batch)
        emap = None
    return cur, batches


__all__ = ["SeamBatch", "label_parents", "select_batch", "remove_batch", "batch_carve", "default_energy"]
