#!/usr/bin/env python
"""Per-stage timing of the libgi hot path on one GPU (CUDA events, graphs).

For each N: times gi_project, gi_bin (ABI: clear+count+scan+scatter+segsort),
gi_render (on gi_bin output), gi_render_backward, gi_render_frame (fused) and
gi_fit_step, each captured alone in a CUDA graph and replayed R times, with
warm L2 (no flush) and cold L2 (256 MB flush before each replay).  Prints a
JSON line per (N, stage).  Diagnostic tool; not part of the product.
"""
from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2403_08551_b200 import gi  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter, Pipeline  # noqa: E402


def timed(fn, reps, flush=None):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    st = torch.cuda.current_stream()
    for a, b in ev:
        if flush is not None:
            flush.zero_()
        a.record(st)
        g.replay()
        b.record(st)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1000.0 for a, b in ev)
    return ts[len(ts) // 2]


def main():
    reps = int(os.environ.get("REPS", "100"))
    W, H = 768, 512
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    for n in [int(x) for x in os.environ.get("NS", "70000,700000").split(",")]:
        p = torch.from_numpy(synth.init_params(1, n)).cuda().view(1, n, 8).contiguous()
        t = torch.from_numpy(synth.image(1, W, H)).cuda().view(1, 3, H, W).contiguous()
        pipe = Pipeline(n, W, H, 1, key_capacity=16 * n + 65536)
        pipe.render(p)
        torch.cuda.synchronize()
        fit = Fitter(p.clone(), t)
        stages = {
            "project": lambda: pipe.project(p),
            "bin(abi)": lambda: pipe.bin(),
            "render(abi)": lambda: pipe.raster(),
            "backward(abi)": lambda: pipe.backward(p, target=t),
            "render_frame": lambda: pipe.render_frame(p),
            "fit_step": lambda: fit.step(),
        }
        for name, fn in stages.items():
            for mode, fl in (("warm", None), ("cold", flush)):
                us = timed(fn, reps, fl)
                print(json.dumps({"n": n, "stage": name, "l2": mode, "us": round(us, 2)}), flush=True)


if __name__ == "__main__":
    main()
