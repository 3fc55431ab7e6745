#!/usr/bin/env python
"""One row per profiled launch of an `ncu --set full` report: time, issue
slots, pipe utilisation, DRAM bytes and bandwidth against the measured HBM
peak.  python tools/ncu_table.py <report.ncu-rep> <out.md> [title]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = {"gpu__time_duration.sum": "us",
        "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue %",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "FMA %",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "XU %",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "ALU %",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "LSU %",
        "dram__bytes_read.sum": "DRAM rd",
        "dram__bytes_write.sum": "DRAM wr",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy %",
        "launch__registers_per_thread": "regs"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, u = rr[0], rr[1]
    lines = [f"# {title}\n", f"HBM peak for the bandwidth fraction: {peak} GB/s "
             "(MEASURED_PEAKS.json); ncu replays each launch with cold caches.\n",
             "| kernel | " + " | ".join(COLS.values()) + " | DRAM GB/s | of HBM peak |",
             "|---" * (len(COLS) + 3) + "|"]
    for v in rr[2:]:
        d = dict(zip(h, v))
        un = dict(zip(h, u))
        name = d.get("Kernel Name", "?").split("(")[0].replace("gi::<unnamed>::", "")
        name = name.replace("(anonymous namespace)::", "").replace("gi::", "").replace("unnamed>::", "")
        vals, num = [], {}
        for k in COLS:
            x = d.get(k, "")
            try:
                f = float(x.replace(",", "")) * SCALE.get(un.get(k, ""), 1)
            except ValueError:
                f = None
            num[k] = f
            vals.append("" if f is None else (f"{f:.2f}" if f < 1e4 else f"{f / 1e6:.2f}M"))
        t_us = num["gpu__time_duration.sum"]
        by = (num["dram__bytes_read.sum"] or 0) + (num["dram__bytes_write.sum"] or 0)
        gbs = by / (t_us * 1e-6) / 1e9 if t_us else 0.0
        frac = f"{100 * gbs / peak:.1f} %" if peak else ""
        lines.append(f"| `{name}` | " + " | ".join(vals) + f" | {gbs:.0f} | {frac} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
