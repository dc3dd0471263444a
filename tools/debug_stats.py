import sys, os, numpy as np, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03180_b200 import _lib
from paper_1903_03180_b200.synth import config_clip
from oracle import scpl_oracle as O
clip, tw, th = config_clip("C2", frames=40)
T, H, W, C = clip.shape
dev = torch.from_numpy(clip).cuda()
lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
codes = torch.empty((T, H, W), dtype=torch.int16, device="cuda")
_lib.check(lib.scpl_energy_codes(cx, dev.data_ptr(), None, T, H, W, C, codes.data_ptr(), st))
state = torch.empty(2 * H * W, dtype=torch.float64, device="cuda")
res = []
for rep in range(6):
    g = (ctypes.c_double * 8)()
    _lib.check(lib.scpl_window_asde(cx, codes.data_ptr(), T, H, W, 0, 1, 8, 0.6, 0.4, state.data_ptr(), 1, g, st))
    g2 = (ctypes.c_double * 8)()
    _lib.check(lib.scpl_window_asde(cx, codes.data_ptr(), T, H, W, 0, 9, 8, 0.6, 0.4, state.data_ptr(), 0, g2, st))
    res.append(list(g) + list(g2))
for r in res: print([x.hex()[-6:] for x in r])
# oracle
em = [O.motion_energy(clip[0], None)] + [O.motion_energy(clip[k], clip[k-1]) for k in range(1, 17)]
S, Q = em[0].copy(), em[0]*em[0]
ora = []
for k in range(1, 17):
    S = S + em[k]; Q = Q + em[k]*em[k]; ora.append(O.asde_from_sums(S, Q, k+1))
print("oracle", [x.hex()[-6:] for x in ora])
print("match rep0:", [a == b for a, b in zip(res[0], ora)])
