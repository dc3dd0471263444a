"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import collections
import csv
import sys


def main(path, first_kernel=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot/1e3:.2f} ms total (serialised, cold-cache: compare shares)")
    print(f"{'kernel':44s} {'n':>5s} {'total us':>10s} {'share':>6s} {'avg us':>9s}")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {n:5d} {us:10.1f} {100*us/tot:5.1f}% {us/n:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
