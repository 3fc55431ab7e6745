#!/usr/bin/env python
"""the oracle (oracle/gio.cpp, fp64, -O2 -fopenmp) timed on
the host cores beside the GPU numbers -- with 1 thread and with all of them
(nproc), C1 forward / backward / fit step in all-pairs mode, C2 and C3
forward and fit iteration in tiled mode.  Writes one JSON object (stdout)
with the CPU model and core counts.  Test infrastructure: it only runs the
oracle."""
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import gio  # noqa: E402

CFGS = {"C1": (64, 64, 256, 0, gio.ALL_PAIRS), "C2": (768, 512, 70000, 1, gio.TILED),
        "C3": (2040, 1356, 100000, 2, gio.TILED)}


def best_of(fn, reps, budget_s):
    ts = []
    t_end = time.perf_counter() + budget_s
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    return min(ts)


def main():
    gio.build()
    nproc = os.cpu_count() or 1
    try:
        lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in lscpu.splitlines()
                      if ln.startswith("Model name")), platform.processor())
        tpc = next((ln.split(":", 1)[1].strip() for ln in lscpu.splitlines()
                    if ln.startswith("Thread(s) per core")), "?")
    except Exception:
        model, tpc = platform.processor(), "?"
    out = {"nproc": nproc, "cpu": model, "threads_per_core": tpc, "build": "g++ -O2 -fopenmp",
           "runs": {}}
    for threads in sorted({1, nproc}):
        gio.set_threads(threads)
        res = {}
        for name, (W, H, n, seed, mode) in CFGS.items():
            p = synth.init_params(seed, n)
            t = synth.image(seed, W, H)
            m = np.zeros_like(p)
            v = np.zeros_like(p)
            big = n > 1000
            reps, budget = (2, 30.0) if big else (20, 5.0)
            r = {"mode": "tiled" if mode == gio.TILED else "all-pairs"}
            r["forward_s"] = best_of(lambda: gio.render(p, W, H, mode=mode), reps, budget)
            if not big:
                img = gio.render(p, W, H, mode=mode)
                _, g = gio.mse(img, t)
                r["backward_s"] = best_of(lambda: gio.backward(p, g, W, H, mode=mode), reps, budget)

            def step():
                _, _, gr = gio.loss_and_grads(p, t, mode=mode)
                gio.adam(p, gr.astype(np.float32), m, v, 1, 1e-3)
            r["fit_step_s"] = best_of(step, reps, budget)
            r["fit_its"] = 1.0 / r["fit_step_s"]
            r["render_fps"] = 1.0 / r["forward_s"]
            res[name] = r
        out["runs"][f"threads_{threads}"] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
