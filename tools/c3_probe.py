#!/usr/bin/env python
"""Diagnostic: fit it/s and render FPS of the init and fitted-proxy clouds,
cold L2 (CUDA graphs, events).  Default C3 (2040x1356, 100k Gaussians);
CFG=C2 for 768x512, 70k."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter, Pipeline  # noqa: E402

CFG = os.environ.get("CFG", "C3")
W, H, N, SEED = (2040, 1356, 100000, 2) if CFG == "C3" else (768, 512, 70000, 1)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(g, reps=50):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]


t = torch.from_numpy(synth.image(SEED, W, H)).cuda()[None].contiguous()
for name, p in (("init", synth.init_params(SEED, N)), ("fitted", synth.fitted_params(SEED, N))):
    pd = torch.from_numpy(p).cuda()[None].contiguous()
    fit = Fitter(pd.clone(), t)
    fit.step()
    g = fit.capture(1)
    for _ in range(5):
        g.replay()
    ms_fit = timed(g)
    pipe = Pipeline(N, W, H, 1)
    pipe.render_frame(pd)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    rg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(rg, stream=s):
        pipe.render_frame(pd)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(5):
        rg.replay()
    ms_r = timed(rg)
    print(json.dumps({"config": CFG, "cloud": name, "fit_its": round(1000 / ms_fit),
                      "render_fps": round(1000 / ms_r), "keys": fit.n_keys()}), flush=True)
    del fit, g, pipe, rg
