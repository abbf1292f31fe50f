"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`):
per-kernel launch count, total device time and share.

    python tools/launch_summary.py gpurun_out/launches.csv [out.txt]

ncu serialises launches and runs them cold-cache, so absolute times are
pessimistic; the SHARES are what a bench-time roofline has to agree with.
"""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
         "second": 1.0, "s": 1.0}


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        rows.append((r["Kernel Name"], v * SCALE.get(r.get("Metric Unit", "ns"), 1e-9)))
    return rows


def short(name):
    name = name.split("(")[0] if not name.startswith("void ") else name[5:].split("(")[0]
    return name[:90]


def main(path, out=None):
    rows = load(path)
    agg = defaultdict(lambda: [0, 0.0])
    for n, t in rows:
        a = agg[short(n)]
        a[0] += 1
        a[1] += t
    total = sum(a[1] for a in agg.values())
    lines = [f"{len(rows)} launches, total {total * 1e3:.3f} ms device time (ncu, serialised, cold cache)"]
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"  {t * 1e3:9.3f} ms  {100 * t / total:6.2f}%  x{c:5d}  {t / c * 1e6:9.1f} us/launch  {n}")
    text = "\n".join(lines)
    if out:
        with open(out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
