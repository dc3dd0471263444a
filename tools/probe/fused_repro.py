"""Fused-pass bring-up: batch_carve on single frames of several shapes, each in its own process
with a timeout, fused vs SCPL_NO_FUSED=1 vs the oracle.

    python tools/probe/fused_repro.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(h, w, tgt, seed, hl):
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_1903_03180_b200 as P
    from oracle import scpl_oracle as O
    rng = np.random.default_rng(seed)
    frame = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    c1, b1 = P.batch_carve(frame, tgt)
    c2, b2 = O.batch_carve(frame, tgt)
    ok = np.array_equal(c1, c2) and [len(x) for x in b1] == [len(x) for x in b2]
    print("RESULT", "OK" if ok else "MISMATCH", [len(x) for x in b1][:8], [len(x) for x in b2][:8], flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child(*map(int, sys.argv[2:7]))
        sys.exit(0)
    cases = [(48, 64, 40), (40, 200, 150), (40, 300, 200), (100, 300, 250), (200, 100, 60), (64, 700, 600),
             (33, 520, 400), (34, 520, 400), (65, 1100, 1000)]
    for env in ({}, {"SCPL_FUSED": "1"}, {"SCPL_FUSED": "1", "SCPL_HOST_LOOPS": "1"}):
        for (h, w, t) in cases:
            e = dict(os.environ, **env)
            try:
                r = subprocess.run([sys.executable, __file__, "--child", str(h), str(w), str(t), "1", "0"], env=e,
                                   capture_output=True, text=True, timeout=60)
                out = [ln for ln in (r.stdout + r.stderr).splitlines() if "RESULT" in ln or "rror" in ln or "DCHECK" in ln]
                print(env, (h, w, t), out[-3:], flush=True)
            except subprocess.TimeoutExpired:
                print(env, (h, w, t), "HANG", flush=True)
