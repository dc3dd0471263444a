import sys, os, numpy as np, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_03180_b200 as P
from paper_1903_03180_b200 import _lib
from paper_1903_03180_b200.synth import config_clip
from oracle import scpl_oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
clip, tw, th = config_clip(name)
T, H, W, C = clip.shape
dev = torch.from_numpy(clip).cuda()
lib, cx, st = _lib.load(), _lib.ctx(), _lib.stream()
outs = []
for rep in range(3):
    codes = torch.empty((T, H, W), dtype=torch.int16, device="cuda")
    _lib.check(lib.scpl_energy_codes(cx, dev.data_ptr(), None, T, H, W, C, codes.data_ptr(), st))
    outs.append(codes.cpu().numpy().view(np.uint16))
print("codes deterministic:", all(np.array_equal(outs[0], o) for o in outs[1:]))
# CPU codes
lib_o = O.clib()
bad = 0
prev = None
for t in range(T):
    l = O.to_luma_c(clip[t]); g = np.empty_like(l)
    lib_o.oracle_sobel(l.ctypes.data, H, W, g.ctypes.data)
    d = np.zeros_like(l) if prev is None else np.abs(l.astype(np.int16) - prev.astype(np.int16)).astype(np.uint8)
    ref = (d.astype(np.uint16) << 8) | g
    nb = int((ref != outs[0][t]).sum())
    if nb:
        bad += 1
        if bad < 5:
            ii = np.argwhere(ref != outs[0][t])[:5]
            print("frame", t, "mismatches", nb, "at", ii.tolist(), "gpu", outs[0][t][tuple(ii.T)].tolist(), "cpu", ref[tuple(ii.T)].tolist())
    prev = l
print("frames with code mismatches:", bad)
for rep in range(4):
    out, m = P.retarget_video_tensor(dev, P.RetargetConfig(target_width=tw, target_height=th, mode="buffered"))
    print("rep", rep, "runs", len(m.runs), [n for _, n in m.runs][-4:], "dp", m.dp_passes, flush=True)
