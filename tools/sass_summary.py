"""Per-kernel SASS evidence from the built objects: counts of the Blackwell
mnemonics (tcgen05 MMA = UTC*MMA, TMEM ld/st = LDTM/STTM, TMA = UTMALDG /
UTMASTG / UBLKCP, legacy HMMA) for every kernel of libevoformer_sm100.

    python tools/sass_summary.py [out.txt]
"""
import glob
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "HMMA", "MUFU.EX2", "FFMA2"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def main(out=None):
    rows = []
    for obj in sorted(glob.glob(os.path.join(ROOT, "build", "csrc", "*.o"))):
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        fn, counts = None, defaultdict(Counter)
        for line in sass.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                fn = m.group(1)
                continue
            if fn is None:
                continue
            for k in KEYS:
                if re.search(r"\b" + re.escape(k) + r"\b", line):
                    counts[fn][k] += 1
        for fn, c in counts.items():
            if any(c[k] for k in KEYS[:8]):
                short = demangle(fn).replace("(anonymous namespace)::", "").replace("void ", "")
                short = short.split("(")[0].replace("evo::", "").replace("__nv_bfloat16", "bf16")
                rows.append((os.path.basename(obj), short, c))
    lines = [f"{'object':26s} {'kernel':60s} " + " ".join(f"{k:>8s}" for k in KEYS)]
    for o, k, c in rows:
        lines.append(f"{o:26s} {k[:60]:60s} " + " ".join(f"{c[x]:8d}" for x in KEYS))
    text = "\n".join(lines)
    print(text)
    if out:
        with open(out, "w") as f:
            f.write("# static SASS instruction counts per kernel (cuobjdump -sass build/csrc/*.o)\n" + text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
