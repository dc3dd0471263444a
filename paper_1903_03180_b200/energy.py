"""Energy maps on the GPU -- drop-in for vidcarve.energy (pkg/src/vidcarve/energy.py).

Same names, signatures, return types and error messages as the reference; the
arithmetic runs in libscpl.so (scpl_to_luma / scpl_energy_codes /
scpl_decode_energy / scpl_gradient_energy) and is bit-exact with it.
"""

from __future__ import annotations

import numpy as np

from . import _lib

MAXVAL = 255.0                    # energy.py:14
DEFAULT_MOTION_WEIGHT = 0.6       # energy.py:19
DEFAULT_GRADIENT_WEIGHT = 0.4     # energy.py:20


def _channels(arr: np.ndarray) -> int:
    if arr.ndim == 2:
        return 1
    if arr.ndim == 3 and arr.shape[2] in (1, 3):
        return arr.shape[2]
    raise ValueError(f"unsupported channel count: expected 1 or 3, got shape {arr.shape}")


def as_u8(arr: np.ndarray) -> np.ndarray:
    """Pixels as uint8: integer arrays with values in 0..255 convert exactly (the reference
    computes on the values, energy.py:34-35); anything else is rejected, never wrapped."""
    arr = np.asarray(arr)
    if arr.dtype == np.uint8:
        return arr
    if arr.dtype.kind in "iub" and (arr.size == 0 or (int(arr.min()) >= 0 and int(arr.max()) <= 255)):
        return arr.astype(np.uint8)
    raise ValueError(f"expected uint8 pixels (or integers in 0..255), got {arr.dtype}")


def _luma_dev(arr: np.ndarray):
    """(h, w) uint8 luma on the device (energy.py:23-37)."""
    torch = _lib.torch_cuda()
    c = _channels(arr)
    src = _lib.to_device(np.ascontiguousarray(as_u8(arr)))
    h, w = arr.shape[:2]
    out = torch.empty((h, w), dtype=torch.uint8, device=src.device)
    _lib.check(_lib.load().scpl_to_luma(_lib.ctx(), src.data_ptr(), h * w, c, out.data_ptr(), _lib.stream()))
    return out


def to_luma(frame: np.ndarray) -> np.ndarray:
    """energy.py:23-37: luma input is returned unchanged; RGB -> BT.601 rint on the GPU."""
    arr = np.asarray(frame)
    if arr.ndim == 2:
        return arr
    if arr.ndim == 3 and arr.shape[2] == 1:
        return arr[:, :, 0]
    if arr.ndim == 3 and arr.shape[2] == 3:
        return _lib.to_host(_luma_dev(arr))
    raise ValueError(f"unsupported channel count: expected 1 or 3, got shape {arr.shape}")


def gradient_energy(luma: np.ndarray) -> np.ndarray:
    """energy.py:40-59: edge-replicated Sobel |Gx|+|Gy| clamped to 255, float64."""
    img = np.asarray(luma)
    if img.ndim != 2:
        raise ValueError(f"expected a single-channel frame, got shape {img.shape}")
    h, w = img.shape
    if h < 3 or w < 3:
        raise ValueError(f"frame too small for 3x3 Sobel: {w}x{h}, need at least 3x3")
    torch = _lib.torch_cuda()
    src = _lib.to_device(np.ascontiguousarray(as_u8(img)))
    out = torch.empty((h, w), dtype=torch.float64, device=src.device)
    _lib.check(_lib.load().scpl_gradient_energy(_lib.ctx(), src.data_ptr(), h, w, out.data_ptr(), _lib.stream()))
    return _lib.to_host(out)


def motion_energy(curr: np.ndarray, prev: np.ndarray | None, w_motion: float = DEFAULT_MOTION_WEIGHT,
                  w_grad: float = DEFAULT_GRADIENT_WEIGHT) -> np.ndarray:
    """energy.py:62-87: min(wm*|dL| + wg*grad, 255); pure gradient when prev is None."""
    if w_motion < 0 or w_grad < 0 or abs(w_motion + w_grad - 1.0) > 1e-9:
        raise ValueError(f"weights must be non-negative and sum to 1, got {w_motion} + {w_grad}")
    torch = _lib.torch_cuda()
    c_arr = np.asarray(curr)
    lc = _luma_dev(c_arr) if c_arr.ndim == 3 and c_arr.shape[2] == 3 else _lib.to_device(
        np.ascontiguousarray(as_u8(to_luma(c_arr))))
    h, w = lc.shape
    if h < 3 or w < 3:
        raise ValueError(f"frame too small for 3x3 Sobel: {w}x{h}, need at least 3x3")
    lp = None
    if prev is not None:
        p_arr = np.asarray(prev)
        lp = _luma_dev(p_arr) if p_arr.ndim == 3 and p_arr.shape[2] == 3 else _lib.to_device(
            np.ascontiguousarray(as_u8(to_luma(p_arr))))
        if tuple(lp.shape) != (h, w):
            raise ValueError(f"dimension mismatch: current frame {(h, w)}, previous {tuple(lp.shape)}")
    codes = torch.empty((h, w), dtype=torch.int16, device=lc.device)
    lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
    _lib.check(lib.scpl_energy_codes(cx, lc.data_ptr(), _lib.ptr(lp), 1, h, w, 1, codes.data_ptr(), st))
    out = torch.empty((h, w), dtype=torch.float64, device=lc.device)
    _lib.check(lib.scpl_decode_energy(cx, codes.data_ptr(), 1, h, w, 1 if prev is None else 0,
                                      float(w_motion), float(w_grad), out.data_ptr(), st))
    return _lib.to_host(out)


__all__ = ["MAXVAL", "DEFAULT_MOTION_WEIGHT", "DEFAULT_GRADIENT_WEIGHT", "to_luma", "gradient_energy",
           "motion_energy"]
