#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and
optionally an `ncu --set full` report into profiles/<tag>_*.md / .json.

  python tools/ncu_summary.py <tag> [--launches gpurun_out/<tag>_launches.csv]
                                    [--report gpurun_out/<tag>_prof.ncu-rep]
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L2 Hit Rate", "Block Size", "Grid Size", "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("gi::<unnamed>::", "gi::")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(
            d["Metric Unit"], 1e-3)
        agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) * scale)
    return agg


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kernels = collections.OrderedDict()
    if rows:
        h = rows[0]
        for r in rows[1:]:
            d = dict(zip(h, r))
            k = d.get("Kernel Name", "?").split("(")[0].replace("gi::<unnamed>::", "gi::")
            if d.get("Metric Name") in KEEP:
                kernels.setdefault(k, {})[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        h, u = rr[0], rr[1]
        for v in rr[2:]:
            d = dict(zip(h, v))
            k = d.get("Kernel Name", "?").split("(")[0].replace("gi::<unnamed>::", "gi::")
            ent = kernels.setdefault(k, {})
            for name, unit in zip(h, u):
                if name in RAW or (name.startswith(STALLS) and not name.endswith("not_issued")):
                    val = d.get(name, "")
                    try:
                        if float(val.replace(",", "")) == 0:
                            continue
                    except ValueError:
                        continue
                    ent[name] = f"{val} {unit}"
    return kernels


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summary `{a.tag}`\n"]
    js = {"tag": a.tag}
    if a.launches:
        agg = launches(a.launches)
        tot = sum(sum(v) for v in agg.values())
        md.append("## Launch list (gpu__time_duration.sum, cold-cache, serialised; compare shares)\n")
        md.append("| kernel | launches | avg us | total us | share |\n|---|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | "
                      f"{100*sum(v)/tot:.1f}% |")
        js["launches"] = {k: {"n": len(v), "avg_us": sum(v) / len(v)} for k, v in agg.items()}
        md.append("")
    if a.report:
        ks = report(a.report)
        js["full"] = ks
        for k, ent in ks.items():
            md.append(f"## `ncu --set full`: `{k}`\n")
            md.append("| metric | value |\n|---|---|")
            for m, v in ent.items():
                md.append(f"| {m} | {v} |")
            md.append("")
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu.json"), "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(md[:40]))


if __name__ == "__main__":
    main()
