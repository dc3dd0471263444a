"""Back-to-back device-path calls on C2: Python wall time per call vs the device span of the call
(SCPL_TIMELINE host/device marks go to stderr).  Shows the host overhead between steps."""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    clip, tw, th = config_clip(name)
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
    dev = torch.from_numpy(clip).cuda()
    for _ in range(3):
        P.retarget_video_tensor(dev, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    walls = []
    for _ in range(n):
        t = time.perf_counter()
        P.retarget_video_tensor(dev, cfg)
        walls.append((time.perf_counter() - t) * 1e3)
    e1.record()
    torch.cuda.synchronize()
    print("per call wall ms:", " ".join(f"{x:.2f}" for x in walls))
    print(f"events over {n} calls: {e0.elapsed_time(e1) / n:.2f} ms/call; last phases {P.pipeline.last_phase_ms}")
    os.environ["SCPL_TIMELINE"] = "1"
    t = time.perf_counter()
    P.retarget_video_tensor(dev, cfg)
    print(f"timeline call wall {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)




def wrapper_costs():
    import timeit
    cfg = P.RetargetConfig(target_width=1440, mode="buffered")
    print("phi table us:", timeit.timeit(lambda: P.pipeline._phi_table(cfg.policy), number=100) * 1e4)


if __name__ == "__main__":
    main()
    wrapper_costs()
