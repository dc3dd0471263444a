"""Print the device timeline (SCPL_TIMELINE) of one clip through both public paths (C2 by default)."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1903_03180_b200 as P  # noqa: E402
from paper_1903_03180_b200.synth import config_clip  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    clip, tw, th = config_clip(name)
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
    host = torch.from_numpy(clip).pin_memory()
    dev = host.cuda()
    out = torch.empty((clip.shape[0], th or clip.shape[1], tw, clip.shape[3]), dtype=torch.uint8, pin_memory=True)
    for _ in range(2):
        P.retarget_video_tensor(dev, cfg)
        P.retarget_video(host, cfg, out=out)
    torch.cuda.synchronize()
    os.environ["SCPL_TIMELINE"] = "1"
    print("---- device path", flush=True)
    P.retarget_video_tensor(dev, cfg)
    torch.cuda.synchronize()
    print("---- host path", flush=True)
    P.retarget_video(host, cfg, out=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
