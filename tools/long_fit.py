#!/usr/bin/env python
"""Diagnostic: a long C2 fit (the paper trains 50k steps) through the
chained fused step in CUDA graphs of 100 steps; prints PSNR along the
way for Adam (north_star) and Adan (the paper's optimiser)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter, Pipeline  # noqa: E402

W, H, N = 768, 512, 70000
STEPS = int(os.environ.get("STEPS", "50000"))
t = torch.from_numpy(synth.image(1, W, H)).cuda()[None].contiguous()
p0 = torch.from_numpy(synth.init_params(1, N)).cuda()[None].contiguous()
pipe = Pipeline(N, W, H, 1)
for opt in ("adam", "adan"):
    fit = Fitter(p0.clone(), t, optimizer=opt)
    fit.step()
    g = fit.capture(100)
    traj = []
    torch.cuda.synchronize()
    t0 = time.time()
    done = 1
    while done < STEPS:
        g.replay()
        done += 100
        if done % 5000 == 1 or done >= STEPS:
            img = pipe.render_frame(fit.params)
            traj.append((done, round(float(pipe.psnr(img, t)[0]), 2)))
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(json.dumps({"optimizer": opt, "steps": done, "seconds": round(dt, 2),
                      "its": round(done / dt), "psnr_db": traj, "status": fit.check()}), flush=True)
