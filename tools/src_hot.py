#!/usr/bin/env python
"""Per CUDA source line instruction counts of an ncu report (needs -lineinfo):
  python tools/src_hot.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, out, tot = "", [], 0
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        ex = int(r[7])
    except (ValueError, IndexError):
        continue
    tot += ex
    out.append((ex, int(r[4]) if r[4].isdigit() else 0, f"{fname}:{r[0]}", r[1].strip()[:70]))
out.sort(reverse=True)
print(f"total {tot / 1e6:.2f}M")
for ex, sm, loc, src in out[:top]:
    print(f"{ex / 1e6:6.2f}M {100 * ex / tot:4.1f}% samp {sm:5d} {loc:28s} {src}")
