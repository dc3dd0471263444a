"""C4 batch timing probe: device-resident 64-clip batch under env variants (one process each).

    python tools/probe/c4_batch.py [--clips 64] [--steps 3] VAR=VAL,VAR=VAL ...
"""
import argparse
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(clips, steps, warmup=2):
    sys.path.insert(0, ROOT)
    import torch
    import paper_1903_03180_b200 as P
    from paper_1903_03180_b200 import pipeline
    from paper_1903_03180_b200.synth import config_clip
    devs = []
    for i in range(clips):
        c, tw, th = config_clip("C4", clip=i)
        devs.append(torch.from_numpy(c).cuda())
    cfg = P.RetargetConfig(target_width=tw, mode="buffered")
    for _ in range(warmup):
        P.retarget_videos(devs, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        res = P.retarget_videos(devs, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ph = pipeline.last_phase_ms
    print(f"RESULT ms={ms:.2f} fps={clips * 90 / ms * 1e3:.0f} dp={sum(m.dp_passes for _, m in res)} "
          f"cl={ph['carve_cluster']} launches={ph['pass_launches']} launch_us={ph['pass_launch_ms'] * 1e3:.1f} "
          f"codes={ph['codes']:.2f} scan={ph['scan']:.2f} after={ph['carve_after_scan']:.2f}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--clips", type=int, default=64)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.clips, a.steps, a.warmup)
        sys.exit(0)
    for v in a.variants or [""]:
        env = dict(os.environ)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            env[k] = val
        t0 = time.time()
        r = subprocess.run([sys.executable, __file__, "--child", "--clips", str(a.clips), "--steps", str(a.steps)],
                           env=env, capture_output=True, text=True)
        lines = [ln for ln in (r.stdout + r.stderr).splitlines() if ln.startswith("RESULT") or "rror" in ln]
        print(f"[{v or 'default'}] {' | '.join(lines[-3:])} ({time.time() - t0:.0f}s)", flush=True)
