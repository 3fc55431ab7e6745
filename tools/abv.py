#!/usr/bin/env python
"""A/B of libgi variants on the box: for each variant (a lib built with
`python paper_2403_08551_b200/build.py <out.so>` and GI_NVCC_EXTRA flags, plus
env settings), run `bench.py --quick` `reps` times, interleaved, and print
the key numbers.
  python tools/abv.py name=lib[,ENV=V...] [name=lib,...] [--reps 2] [--steps 200]
`lib` may be "-" for the in-tree libgi.so."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 2
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 200
extra = sys.argv[sys.argv.index("--bench") + 1].split() if "--bench" in sys.argv else []
variants = []
for a in args:
    if a.isdigit():
        continue
    name, spec = a.split("=", 1)
    parts = spec.split(",")
    env = dict(os.environ)
    if parts[0] != "-":
        env["GI_LIB"] = os.path.join(ROOT, parts[0])
    for kv in parts[1:]:
        k, v = kv.split("=", 1)
        env[k] = v
    variants.append((name, env))
res = {n: [] for n, _ in variants}
for r in range(reps):
    for name, env in variants:
        cmd = [sys.executable, "bench.py", "--quick", "--batch-images", "0", "--no-cpu-baseline",
               "--steps", str(steps), "--warmup", "20"] + extra
        out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        if out.returncode != 0 or not line:
            print(name, "FAILED", out.stderr[-1500:], flush=True)
            continue
        d = json.loads(line[-1])
        sm = d["stage_ms"]
        row = dict(fit=d["value"], render=d["render_fps"], decode=d["decode_fps"],
                   adan=d["fit_its_adan"], tile=1e3 * sm["tile_kernel_fwd_l2_bwd"],
                   fin=1e3 * sm["finalize_adam_next_projection_binning"],
                   rk=1e3 * d["render_kernel_ms"], rep=(d.get("flush_per_replay") or {}).get("fit_its") or 0.0)
        res[name].append(row)
        print(f"{name:14s} rep {r}: fit {row['fit']:7.0f}  render {row['render']:7.0f}  "
              f"decode {row['decode']:7.0f}  adan {row['adan']:7.0f}  tile {row['tile']:5.1f} us  "
              f"fin {row['fin']:5.1f} us  rkern {row['rk']:5.1f} us  fit(flush) {row['rep']:7.0f}", flush=True)
print("median:")
for name, rows in res.items():
    if not rows:
        continue
    med = {k: sorted(r[k] for r in rows)[len(rows) // 2] for k in rows[0]}
    print(f"{name:14s} fit {med['fit']:7.0f}  render {med['render']:7.0f}  decode {med['decode']:7.0f}"
          f"  adan {med['adan']:7.0f}  tile {med['tile']:5.1f}  fin {med['fin']:5.1f}  rk {med['rk']:5.1f}"
          f"  fit(flush) {med['rep']:7.0f}")
