#!/usr/bin/env python
"""Diagnostic: batched fused fit (B images per launch, C2 size) image-it/s vs B."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter  # noqa: E402

W, H, N = 768, 512, 70000
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for B in [int(x) for x in os.environ.get("BS", "1,8,16,32,64").split(",")]:
    p = torch.from_numpy(np.stack([synth.init_params(100 + b, N) for b in range(B)])).cuda()
    t = torch.from_numpy(np.stack([synth.image(100 + b, W, H) for b in range(B)])).cuda()
    fit = Fitter(p.contiguous(), t.contiguous())
    fit.step()
    g = fit.capture(1)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    reps = 20
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]
    print(json.dumps({"B": B, "ms_per_step": round(ms, 4), "image_its": round(B / ms * 1000)}), flush=True)
    del fit, g, p, t
    torch.cuda.empty_cache()
