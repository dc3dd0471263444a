"""Summarise tools/probe/stream_kernels.sh: per streaming-kernel launch, the algorithmic bytes
(from the launch's own DRAM read volume: frames in, codes, ...) and GB/s = bytes / duration.

    python tools/stream_summary.py gpurun_out/sk_C2.csv H W TW
"""
import collections
import csv
import sys

path, H, W, TW = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
L = collections.defaultdict(dict)
for r in rows[1:]:
    L[(r[idi], r[ki])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for (i, k), m in sorted(L.items(), key=lambda x: int(x[0][0])):
    name = k.split("(")[0].split("<")[0].split("::")[-1]
    t = m["gpu__time_duration.sum"]
    rd = m["dram__bytes_read.sum"]
    if name == "replay_rows_vec_kernel":  # (its DRAM reads also hold the index map)
        T = max(1, int(rd / (H * W * 3)))
        alg = T * (H * W * 3 + H * TW * 3)
    elif name == "uniform_vec_kernel":
        T = max(1, round(rd / (H * W * 2)))
        alg = T * H * W * 2 + H * W * 8
    else:  # codes: frames in (3 B/px) + codes out (2 B/px)
        T = max(1, round(rd / (H * W * 3)))
        alg = T * H * W * 5
    agg[name][0] += alg
    agg[name][1] += t
    agg[name][2] += 1
    print(f"{name:24s} frames {T:3d}  {t * 1e6:8.1f} us  alg {alg / 1e6:8.1f} MB  {alg / t / 1e9:7.0f} GB/s")
for name, (a, t, n) in agg.items():
    print(f"TOTAL {name:24s} {n:3d} launches  {a / 1e6:9.1f} MB in {t * 1e6:9.1f} us = {a / t / 1e9:6.0f} GB/s")
