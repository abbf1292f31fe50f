"""Summarise an `ncu --page source --csv` dump: top SASS instructions by
warp-stall samples, plus totals by opcode."""
import csv
import sys
from collections import Counter


def main(path, top=40):
    top = int(top)
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[key] or 0) for d in data)
    by_op = Counter()
    for d in data:
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        by_op[op.split(".")[0]] += float(d[key] or 0)
    print(f"total samples {tot:.0f}")
    for op, v in by_op.most_common(20):
        print(f"  {op:14s} {100 * v / tot:5.1f}%")
    print("top instructions:")
    for d in sorted(data, key=lambda d: -float(d[key] or 0))[:top]:
        print(f"  {100 * float(d[key] or 0) / tot:5.1f}%  {d['Address']:>6s}  {d['Source'][:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
