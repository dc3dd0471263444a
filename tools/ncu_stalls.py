"""Warp-stall summary of an ncu source-page export (SASS view).

  ncu -i REP --page source --csv --print-source sass > src.csv
  python tools/ncu_stalls.py src.csv [EXEC_COUNT]

Prints the stall mix over the whole kernel, the hottest instruction windows, and -- given the
execution count of a loop body's instructions -- the stall mix and opcode mix of that body."""
import csv
import sys
from collections import Counter, defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    recs = []
    for k, r in enumerate(data):
        if len(r) < len(hdr):
            continue
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        recs.append((k, n, r))
    total = Counter()
    for _, _, r in recs:
        for h in stall_cols:
            total[h] += int(r[ix[h]] or 0)
    S = sum(total.values())
    print(f"kernel: {rows[0][1]}\ntotal warp samples {S}")
    for h, v in total.most_common(8):
        print(f"  {h[6:]:22s} {v:7d} {v / S:6.1%}")
    win = defaultdict(int)
    for k, n, _ in recs:
        win[k // 50] += n
    print("hottest 50-instruction windows (index range, samples, top instruction, executions):")
    for b, v in sorted(win.items(), key=lambda x: -x[1])[:12]:
        top = max((x for x in recs if x[0] // 50 == b), key=lambda x: x[1])
        print(f"  {b * 50:6d}-{b * 50 + 49:<6d} {v:6d} {v / S:6.1%}  {top[2][ix['Source']].strip()[:48]:48s}"
              f" x{top[2][ix['Instructions Executed']]}")
    if len(sys.argv) > 2:
        body = [r for _, _, r in recs if r[ix["Instructions Executed"]] == sys.argv[2]]
        bt = Counter()
        ops, opn = Counter(), Counter()
        for r in body:
            for h in stall_cols:
                bt[h] += int(r[ix[h]] or 0)
            src = r[ix["Source"]].split()
            op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
            ops[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            opn[op] += 1
        B = sum(bt.values())
        print(f"loop body (instructions executed {sys.argv[2]} times): {len(body)} instructions, {B} samples "
              f"({B / S:.1%} of all warps' samples)")
        for h, v in bt.most_common(6):
            print(f"  {h[6:]:22s} {v:7d} {v / max(B, 1):6.1%}")
        print("  opcode mix (count, samples):", ", ".join(f"{o} {opn[o]}/{v}" for o, v in ops.most_common(10)))


if __name__ == "__main__":
    main()
