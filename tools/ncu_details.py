"""Print selected rows of `ncu -i X --page details --csv` per kernel.

    python tools/ncu_details.py report.ncu-rep [regex]
"""
import csv
import io
import re
import subprocess
import sys


def main(path, pat="Stall|Occupancy|Block Limit|Registers|Shared Memory|Achieved|Theoretical|Issue|Eligible|Warp Cycles|Duration|DRAM|Memory Throughput|Compute"):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rx = re.compile(pat)
    last = None
    for r in csv.DictReader(io.StringIO(out)):
        k = r.get("Kernel Name", "")[:60] + " #" + r.get("ID", "")
        if k != last:
            print("==", k)
            last = k
        if rx.search(r.get("Metric Name", "")):
            print(f"   {r.get('Section Name','')[:24]:24s} {r['Metric Name'][:48]:48s} {r['Metric Value']:>14s} {r.get('Metric Unit','')}")


if __name__ == "__main__":
    main(*sys.argv[1:])
