"""Attribute ncu per-instruction stall samples to CUDA source lines.

    python tools/ncu_lines.py report.ncu-rep kernel_regex object.o [top]

Joins the SASS page of the report (per-address samples) with nvdisasm's line table of the
same build's cubin (extracted from the object file).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, func_regex):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True, check=True)
    cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cubin)], capture_output=True,
                         text=True).stdout
    table, cur, in_fn = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith("//--------------------- .text."):
            in_fn = re.search(func_regex, ln) is not None
            continue
        if not in_fn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def main(rep, kregex, obj, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                          f"regex:{kregex}", "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    data = [r for r in rows[2:] if len(r) > iE and r[iE].isdigit()]
    base = int(data[0][0], 16)
    table = line_table(obj, kregex)
    agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    for r in data:
        off = int(r[0], 16) - base
        key = table.get(off, ("?", 0))
        a = agg[key]
        a[0] += int(r[iS] or 0)
        a[1] += int(r[iE] or 0)
        for c in stall_cols:
            a[2][c] += int(r[h.index(c)] or 0)
    total = sum(a[0] for a in agg.values())
    print(f"total samples {total}")
    src = {}
    for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        if f not in src:
            p = os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "csrc", f)
            src[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = src[f][ln - 1].strip()[:70] if 0 < ln <= len(src[f]) else ""
        st = ", ".join(f"{k[6:]} {v}" for k, v in a[2].most_common(3) if v)
        print(f"{a[0]:6d} {100 * a[0] / max(total, 1):5.1f}%  {f}:{ln:<5d} inst {a[1]:>10d}  [{st}]  {text}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
