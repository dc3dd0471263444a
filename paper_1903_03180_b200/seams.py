"""Seam DP and single-seam operations -- drop-in for vidcarve.seams (pkg/src/vidcarve/seams.py)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True, eq=False)
class Seam:
    """seams.py:18-24."""

    offsets: np.ndarray
    cost: float
    orientation: str = "vertical"


@dataclass(eq=False)
class DpTables:
    """seams.py:27-36: cumulative energy (float64) and predecessor deltas (int8)."""

    ce: np.ndarray
    back: np.ndarray


def cumulative_energy(energy: np.ndarray) -> DpTables:
    """seams.py:39-65 on the GPU: leftmost (-1 < 0 < +1) tie-break, +inf borders."""
    e = np.asarray(energy, dtype=np.float64)
    if e.ndim != 2 or e.size == 0:
        raise ValueError(f"expected a non-empty 2-d energy map, got shape {e.shape}")
    torch = _lib.torch_cuda()
    h, w = e.shape
    ed = _lib.to_device(np.ascontiguousarray(e))
    ce = torch.empty((h, w), dtype=torch.float64, device=ed.device)
    back = torch.empty((h, w), dtype=torch.int8, device=ed.device)
    _lib.check(_lib.load().scpl_cumulative_energy(_lib.ctx(), ed.data_ptr(), h, w, ce.data_ptr(), back.data_ptr(),
                                                  _lib.stream()))
    return DpTables(ce=_lib.to_host(ce), back=_lib.to_host(back))


def trace_columns(back: np.ndarray, last_cols: np.ndarray) -> np.ndarray:
    """seams.py:68-81: (h, len(last_cols)) column offsets, top row first."""
    torch = _lib.torch_cuda()
    b = np.ascontiguousarray(back, dtype=np.int8)
    h, w = b.shape
    cols = np.ascontiguousarray(np.asarray(last_cols, dtype=np.int64).ravel())
    if cols.size == 0:
        return np.empty((h, 0), dtype=np.intp)
    bd = _lib.to_device(b)
    cd = _lib.to_device(cols)
    off = torch.empty((cols.size, h), dtype=torch.int64, device=bd.device)
    _lib.check(_lib.load().scpl_trace_columns(_lib.ctx(), bd.data_ptr(), h, w, cd.data_ptr(), cols.size,
                                              off.data_ptr(), _lib.stream()))
    return np.ascontiguousarray(_lib.to_host(off).T).astype(np.intp, copy=False)


def min_seam(tables: DpTables) -> Seam:
    """seams.py:84-89: the leftmost cheapest last-row pixel, traced."""
    from .batching import _select_cols
    last = np.asarray(tables.ce)[-1]
    cols, costs = _select_cols(last, np.zeros(last.size, dtype=np.int64), 1)
    offsets = trace_columns(tables.back, cols)[:, 0]
    return Seam(offsets=offsets, cost=float(costs[0]))


def remove_seam(frame: np.ndarray, seam: Seam) -> np.ndarray:
    """seams.py:92-105: drop one pixel per row."""
    from .batching import _remove_offsets
    arr = np.asarray(frame)
    h, w = arr.shape[:2]
    offs = np.asarray(seam.offsets)
    if offs.shape != (h,):
        raise ValueError(f"seam length {offs.shape} does not match frame height {h}")
    if (offs < 0).any() or (offs >= w).any():
        raise ValueError(f"seam offset out of range for width {w}")
    out, _ = _remove_offsets(arr, offs[None, :])
    return out


def transpose(frame: np.ndarray) -> np.ndarray:
    """seams.py:108-111: swap rows and columns (channels untouched); its own inverse."""
    arr = np.asarray(frame)
    return np.ascontiguousarray(np.swapaxes(arr, 0, 1))


__all__ = ["Seam", "DpTables", "cumulative_energy", "trace_columns", "min_seam", "remove_seam", "transpose"]
