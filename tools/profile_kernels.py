"""Drive the scan/energy kernels outside graphs at the C2 shape, for ncu captures.

    ncu --set full -k regex:'codes_kernel|window_stats|fold_partial' python tools/profile_kernels.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1903_03180_b200 import _lib  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402


def main():
    frames = int(os.environ.get("FRAMES", "64"))
    clip, _, _ = config_clip("C2", frames=frames)
    T, H, W, C = clip.shape
    dev = torch.from_numpy(clip).cuda()
    lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
    codes = torch.empty((T, H, W), dtype=torch.int16, device="cuda")
    for _ in range(2):
        _lib.check(lib.scpl_energy_codes(cx, dev.data_ptr(), None, T, H, W, C, codes.data_ptr(), st))
    state = torch.empty((2, H * W), dtype=torch.float64, device="cuda")
    asde = (ctypes.c_double * 8)()
    _lib.check(lib.scpl_window_asde(cx, codes.data_ptr(), T, H, W, 0, 1, 8, 0.6, 0.4, state.data_ptr(), 1,
                                    asde, st))
    _lib.check(lib.scpl_window_asde(cx, codes.data_ptr(), T, H, W, 0, 9, 8, 0.6, 0.4, state.data_ptr(), 0,
                                    asde, st))
    torch.cuda.synchronize()
    print("asde", list(asde))


if __name__ == "__main__":
    main()
