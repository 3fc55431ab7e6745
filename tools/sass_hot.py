#!/usr/bin/env python
"""Group an ncu report's SASS (source page) into runs of equal execution
count and print the heavy ones: where a kernel's instructions go.
  python tools/sass_hot.py <report.ncu-rep> [min_total_M]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, data = rows[1], rows[2:]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i_ex]) for r in data)
print(f"total {tot / 1e6:.2f}M warp instructions")
runs, prev, start, samp = [], None, 0, 0
for k, r in enumerate(data + [["", "-1"] + [""] * len(hdr)]):
    e = int(r[i_ex]) if k < len(data) else -1
    if e != prev:
        if prev is not None:
            runs.append((start, k - 1, prev, samp))
        prev, start, samp = e, k, 0
    if k < len(data):
        samp += int(r[i_s])
for s, e, c, sp in runs:
    n = e - s + 1
    if c * n >= thr * 1e6:
        print(f"{s:5d}-{e:5d} x{c:8d} {n:4d} inst = {c * n / 1e6:6.2f}M ({100 * c * n / tot:4.1f}%) "
              f"samples {sp:5d}  {data[s][i_src].strip()[:50]}")
