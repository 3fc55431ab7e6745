#!/usr/bin/env python
"""Diagnostic: a few gi_render_frame calls of the C2 fitted-proxy cloud (for ncu)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Pipeline  # noqa: E402

W, H, N = 768, 512, 70000
pd = torch.from_numpy(synth.fitted_params(1, N)).cuda()[None].contiguous()
pipe = Pipeline(N, W, H, 1)
for _ in range(4):
    pipe.render_frame(pd)
torch.cuda.synchronize()
print("keys", pipe.frame_keys())
