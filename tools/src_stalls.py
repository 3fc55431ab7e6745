#!/usr/bin/env python
"""Per source line (CUDA) instructions and warp-stall samples of an ncu report
(needs -lineinfo and --import-source), optionally grouped by line ranges:
  python tools/src_stalls.py <report.ncu-rep> [top] [--groups file:lo-hi=name,...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
groups = []
for a in sys.argv[2:]:
    if a.startswith("--groups="):
        for g in a.split("=", 1)[1].split(","):
            loc, name = g.split("=")
            f, rng = loc.split(":")
            lo, hi = rng.split("-")
            groups.append((f, int(lo), int(hi), name))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "", None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        ex = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("# Samples", "0") or 0)
    except ValueError:
        continue
    if ex == 0 and smp == 0:
        continue
    st = {k[6:]: int(v) for k, v in d.items()
          if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    rows.append((fname, int(r[0]), d.get("Source", "")[:60], ex, smp, st))
tot_ex = sum(x[3] for x in rows)
tot_s = sum(x[4] for x in rows)
print(f"instructions {tot_ex / 1e6:.2f}M, samples {tot_s}")


def fmt_st(st, n=4):
    return " ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:n])


if groups:
    agg = {}
    for f, ln, src, ex, smp, st in rows:
        name = next((g[3] for g in groups if g[0] == f and g[1] <= ln <= g[2]), f"{f}:other")
        a = agg.setdefault(name, [0, 0, {}])
        a[0] += ex
        a[1] += smp
        for k, v in st.items():
            a[2][k] = a[2].get(k, 0) + v
    for name, (ex, smp, st) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:24s} {ex / 1e6:6.2f}M {100 * ex / tot_ex:5.1f}%  samples {smp:5d} "
              f"{100 * smp / max(tot_s, 1):5.1f}%  {fmt_st(st)}")
else:
    for f, ln, src, ex, smp, st in sorted(rows, key=lambda x: -x[4])[:top]:
        print(f"{smp:5d} {ex / 1e6:6.2f}M {f}:{ln:<5d} {src:60s} {fmt_st(st)}")
