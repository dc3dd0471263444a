"""Summarise an ncu report: per kernel launch, the headline metrics (with ncu's units) and the
DRAM traffic converted to bytes, next to the launch's duration (achieved DRAM GB/s).

    python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes_per_launch]
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0}


def _num(v):
    return float(str(v).replace(",", ""))


def main(path, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    id_col = "ID" if "ID" in h else h[0]
    launches = {}
    dur = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = (d[id_col], d.get("Kernel Name", ""))
        if d["Metric Name"] in WANT:
            launches.setdefault(k, {})[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
        if d["Metric Name"] == "Duration":
            try:
                dur[d[id_col]] = _num(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1.0)
            except ValueError:
                pass
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh, ru = rr[0], rr[1]  # names, units
    rid = "ID" if "ID" in rh else rh[0]
    units = dict(zip(rh, ru))
    dram = {}
    for r in rr[2:]:
        d = dict(zip(rh, r))
        try:
            rd = _num(d["dram__bytes_read.sum"]) * SCALE.get(units.get("dram__bytes_read.sum", "byte"), 1.0)
            wr = _num(d["dram__bytes_write.sum"]) * SCALE.get(units.get("dram__bytes_write.sum", "byte"), 1.0)
        except (KeyError, ValueError):
            continue
        dram[d[rid]] = (rd, wr)
    for (i, name), m in sorted(launches.items(), key=lambda kv: int(kv[0][0])):
        print(f"[{i}] {name[:100]}")
        for k in WANT:
            if k in m:
                print(f"    {k:34s} {m[k]}")
        if i in dram:
            rd, wr = dram[i]
            line = f"    {'DRAM bytes read / write':34s} {rd / 1e6:.3f} MB / {wr / 1e6:.3f} MB"
            if i in dur and dur[i] > 0:
                line += f"  ({(rd + wr) / dur[i] / 1e9:.0f} GB/s)"
            print(line)
        if alg_bytes and i in dur and dur[i] > 0:
            print(f"    {'algorithmic bytes / duration':34s} {alg_bytes / 1e6:.3f} MB -> "
                  f"{alg_bytes / dur[i] / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
