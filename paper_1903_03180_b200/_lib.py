"""ctypes binding of libscpl.so (include/scpl.h) plus the device plumbing around it.

There is no CPU fallback: if the library or a CUDA device is missing, every compute
entry point raises. Device memory is torch-owned (torch is plumbing here); the .so
only sees raw pointers and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCPL_CHECKED=1 loads the checked build (device-side invariant checks, build_ext.py)
LIB_PATH = os.path.join(_HERE, "libscpl_checked.so" if os.environ.get("SCPL_CHECKED") else "libscpl.so")

_c_int_p = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p


class VideoParams(ctypes.Structure):
    _fields_ = [
        ("target_width", ctypes.c_int), ("target_height", ctypes.c_int), ("mode", ctypes.c_int),
        ("height_first", ctypes.c_int), ("max_len", ctypes.c_int),
        ("w_motion", ctypes.c_double), ("w_grad", ctypes.c_double),
        ("phi", ctypes.POINTER(ctypes.c_double)), ("spec_len", ctypes.c_int), ("reaverage", ctypes.c_int),
        ("shard_rank", ctypes.c_int), ("shard_count", ctypes.c_int),
        ("runs_in", ctypes.POINTER(ctypes.c_int)), ("n_runs_in", ctypes.c_int), ("scan_only", ctypes.c_int),
    ]


class VideoResult(ctypes.Structure):
    _fields_ = [
        ("dp_passes", ctypes.c_long), ("n_runs", ctypes.c_int),
        ("run_start", _c_int_p), ("run_len", _c_int_p), ("phase_ms", ctypes.c_float * 4),
        ("carve_cycles", ctypes.c_longlong * 4), ("carve_cluster", ctypes.c_int),
        ("scan_windows", ctypes.c_int), ("scan_fallbacks", ctypes.c_int),
        ("seam_dump", ctypes.c_void_p), ("seam_dump_cap", ctypes.c_size_t), ("seam_dump_used", ctypes.c_size_t),
    ]


# name -> argtypes (all return int unless listed in _RESTYPE)
_SIGS = {
    "scpl_version": [],
    "scpl_kernel_launches": [],
    "scpl_last_error": [],
    "scpl_create": [ctypes.c_int, ctypes.POINTER(_vp)],
    "scpl_destroy": [_vp],
    "scpl_to_luma": [_vp, _vp, ctypes.c_long, ctypes.c_int, _vp, _vp],
    "scpl_gradient_energy": [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp],
    "scpl_energy_codes": [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp],
    "scpl_decode_energy": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                           ctypes.c_double, _vp, _vp],
    "scpl_window_asde": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                         ctypes.c_int, ctypes.c_double, ctypes.c_double, _vp, ctypes.c_int, _vp, _vp],
    "scpl_uniform_energy": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                            ctypes.c_double, ctypes.c_int, _vp, _vp],
    "scpl_batch_carve": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                         _vp, _c_int_p, _vp, _vp, _vp, _vp, _vp],
    "scpl_replay": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                    ctypes.c_int, ctypes.c_int, _vp, _vp],
    "scpl_jitter_sums": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp],
    "scpl_retarget_video": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.POINTER(VideoParams), _vp, ctypes.POINTER(VideoResult), _vp],
    "scpl_retarget_video_host": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.POINTER(VideoParams), _vp, ctypes.POINTER(VideoResult), _vp],
    "scpl_retarget_batch": [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, ctypes.POINTER(VideoParams), ctypes.POINTER(_vp),
                            ctypes.POINTER(VideoResult), ctypes.c_int, _vp],
    "scpl_cumulative_energy": [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp],
    "scpl_label_parents": [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp],
    "scpl_trace_columns": [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp, _vp],
    "scpl_select_batch": [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _c_int_p, _vp],
    "scpl_remove_columns": [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp, _vp, _vp],
    "scpl_sums_start": [_vp, _vp, ctypes.c_long, _vp, _vp, _vp],
    "scpl_sums_push": [_vp, _vp, ctypes.c_long, _vp, _vp, _vp, _vp, _vp],
    "scpl_sums_map": [_vp, _vp, _vp, ctypes.c_long, ctypes.c_int, ctypes.c_int, _vp, _vp],
    "scpl_asde_from_sums": [_vp, _vp, _vp, ctypes.c_long, ctypes.c_int, ctypes.POINTER(ctypes.c_double), _vp],
}
_RESTYPE = {"scpl_last_error": ctypes.c_char_p, "scpl_destroy": None, "scpl_kernel_launches": ctypes.c_long}

_lib = None
_lock = threading.Lock()
_ctx: dict[int, int] = {}


def load() -> ctypes.CDLL:
    """Load libscpl.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1903_03180_b200.build_ext` "
                "(the SCPL path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load().scpl_last_error() or b"").decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(f"libscpl: {msg}")


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the SCPL path needs a CUDA device (B200); no CPU fallback exists")
    return torch


def ctx(device: int | None = None) -> int:
    torch = torch_cuda()
    dev = torch.cuda.current_device() if device is None else device
    with _lock:
        if dev not in _ctx:
            out = _vp()
            check(load().scpl_create(dev, ctypes.byref(out)))
            _ctx[dev] = out.value
        return _ctx[dev]


def stream(device=None) -> int:
    """The current torch stream of `device` (default: the current device)."""
    torch = torch_cuda()
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    return t.data_ptr() if t is not None else None


def to_device(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (pinned staging for host arrays)."""
    torch = torch_cuda()
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.pin_memory().cuda(non_blocking=True)
    else:
        arr = np.ascontiguousarray(a)
        t = torch.from_numpy(arr)
        t = t.pin_memory().cuda(non_blocking=True) if arr.nbytes >= (1 << 16) else t.cuda()
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    return t.contiguous()


def to_host(t) -> np.ndarray:
    return t.cpu().numpy()
