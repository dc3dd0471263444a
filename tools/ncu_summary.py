"""Summarise an ncu report: per kernel launch, the headline metrics and top stall reasons.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    launches = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = (d["ID"], d["Kernel Name"])
        if d["Metric Name"] in WANT:
            launches.setdefault(k, {})[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    dram = {}
    for r in rr[2:]:
        d = dict(zip(rh, r))
        try:
            rd = float(d.get("dram__bytes_read.sum", "nan").replace(",", ""))
            wr = float(d.get("dram__bytes_write.sum", "nan").replace(",", ""))
        except ValueError:
            continue
        dram[d["ID"]] = (rd, wr, rh)
    for (i, name), m in sorted(launches.items(), key=lambda kv: int(kv[0][0])):
        print(f"[{i}] {name[:100]}")
        for k in WANT:
            if k in m:
                print(f"    {k:34s} {m[k]}")
        if i in dram:
            print(f"    {'dram bytes read / write':34s} {dram[i][0]:.4g} / {dram[i][1]:.4g}")


if __name__ == "__main__":
    main(sys.argv[1])
