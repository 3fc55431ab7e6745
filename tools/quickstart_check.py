#!/usr/bin/env python
"""The README quick start, shortened to 5,000 steps: a logged fit (JSONL),
a checkpoint, a resumed Fitter and one fused frame (run from the repo root)."""
import sys, time
sys.path.insert(0, ".")
import torch, synth
from paper_2403_08551_b200.pipeline import Fitter, Pipeline
from paper_2403_08551_b200 import gi
params = torch.from_numpy(synth.init_params(1, 70000)).cuda()[None].contiguous()
target = torch.from_numpy(synth.image(1, 768, 512)).cuda()[None].contiguous()
fit = Fitter(params, target)
t0 = time.time()
log = fit.fit(5000, log_every=1000, log="gpurun_out/qs_fit.jsonl")
print("fit 5000 steps", time.time() - t0, log[-1])
fit.save("gpurun_out/qs_ckpt.npz")
fit2 = Fitter.load("gpurun_out/qs_ckpt.npz", target)
img = Pipeline(70000, 768, 512).render_frame(fit2.params)
print("render ok", float(img.mean()))
