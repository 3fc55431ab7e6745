#!/usr/bin/env python
"""Diagnostic (for ncu): a few gi_render_frame calls and chained fit steps of
the fitted-proxy cloud.  CFG=C2 (default) or C3."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter, Pipeline  # noqa: E402

CFG = os.environ.get("CFG", "C2")
W, H, N, SEED = (2040, 1356, 100000, 2) if CFG == "C3" else (768, 512, 70000, 1)
pd = torch.from_numpy(synth.fitted_params(SEED, N)).cuda()[None].contiguous()
pipe = Pipeline(N, W, H, 1)
for _ in range(4):
    pipe.render_frame(pd)
t = torch.from_numpy(synth.image(SEED, W, H)).cuda()[None].contiguous()
fit = Fitter(pd.clone(), t)
for _ in range(4):
    fit.step()
torch.cuda.synchronize()
print("keys", pipe.frame_keys(), fit.n_keys())
