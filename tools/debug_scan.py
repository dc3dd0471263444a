"""Debug: compare the GPU buffer scan with the oracle on a config clip."""
import sys, os, json, math
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import paper_1903_03180_b200 as P
from paper_1903_03180_b200 import _lib
from paper_1903_03180_b200.synth import config_clip
from oracle import scpl_oracle as O

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
ref_runs = json.loads(sys.argv[2]) if len(sys.argv) > 2 else None
clip, tw, th = config_clip(name)
dev = torch.from_numpy(clip).cuda()
out, m = P.retarget_video_tensor(dev, P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))
print("gpu runs", [n for _, n in m.runs], "dp", m.dp_passes)
T, H, W, C = clip.shape
codes = torch.empty((T, H, W), dtype=torch.int16, device="cuda")
lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
_lib.check(lib.scpl_energy_codes(cx, dev.data_ptr(), None, T, H, W, C, codes.data_ptr(), st))
gr = [tuple(r) for r in m.runs]
if ref_runs:
    starts = np.concatenate([[0], np.cumsum(ref_runs)[:-1]])
    rr = list(zip(starts.tolist(), ref_runs))
    for a, b in zip(gr, rr):
        if a != b:
            print("first diff gpu", a, "ref", b)
            s = b[0]; n = min(max(a[1], b[1]) + 1, T - s)
            break
    else:
        s = None
    if s is not None:
        frames = list(clip[max(0, s - 1): s + n])
        em = [O.motion_energy(frames[k], frames[k - 1] if k > 0 else None) for k in range(len(frames))]
        if s > 0: em = em[1:]
        S, Q = em[0].copy(), em[0] * em[0]
        state = torch.empty(2 * H * W, dtype=torch.float64, device="cuda")
        g = (ctypes.c_double * (n - 1))()
        _lib.check(lib.scpl_window_asde(cx, codes.data_ptr(), T, H, W, s, 1, n - 1, 0.6, 0.4, state.data_ptr(), 1, g, st))
        pol = O.BufferPolicy()
        for k in range(1, n):
            S = S + em[k]; Q = Q + em[k] * em[k]
            a = O.asde_from_sums(S, Q, k + 1)
            print(f"n={k+1} oracle {a!r} gpu {g[k-1]!r} phi {O.threshold(k+1, pol)!r} {'SAME' if a == g[k-1] else 'DIFF'}")
