"""One line of roofline evidence per kernel launch of an ncu --set full report:
duration, DRAM bytes (read + write), DRAM throughput, tensor-pipe and MUFU (xu)
activity, issue-slot use, achieved occupancy.

    python tools/ncu_summary.py report.ncu-rep [out.txt] [traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

M = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
    "issue_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, row, units)}


def main(path, out=None, traffic=None):
    lines, tr = [], {}
    lines.append(f"{'kernel':58s} {'us':>8s} {'DRAM MB':>9s} {'DRAM%':>6s} {'tensor%':>8s} {'xu%':>6s} "
                 f"{'issue%':>7s} {'occ%':>6s}")
    for d in rows(path):
        name = d["Kernel Name"][0].replace("(anonymous namespace)::", "").replace("evo::", "")
        name = name.split("(")[0].replace("void ", "")[:58]

        def val(k):
            v, u = d.get(M[k], ("nan", ""))
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                return float("nan")
            return x * UNIT.get(u, 1.0)
        dur = val("dur_us")
        mb = (val("dram_rd") + val("dram_wr")) / 1e6
        lines.append(f"{name:58s} {dur:8.1f} {mb:9.1f} {val('dram_pct'):6.1f} {val('tensor_pct'):8.1f} "
                     f"{val('xu_pct'):6.1f} {val('issue_pct'):7.1f} {val('occ_pct'):6.1f}")
        tr.setdefault(name, {"kernel": name, "traffic_bytes": mb * 1e6, "duration_us": dur})
    text = "\n".join(lines)
    print(text)
    if out:
        with open(out, "w") as f:
            f.write(f"# ncu --set full --clock-control none (cold, serialised replays): {path}\n" + text + "\n")
    if traffic:
        with open(traffic, "w") as f:
            json.dump(tr, f, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
