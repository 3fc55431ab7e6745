#!/usr/bin/env python
"""A few C2 frames through gi_render_frame only (for `ncu -k` captures of the
render kernel without the fit kernels around it)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Pipeline  # noqa: E402

p = torch.from_numpy(synth.init_params(1, 70000)).cuda()[None].contiguous()
pipe = Pipeline(70000, 768, 512, 1)
for _ in range(6):
    pipe.render_frame(p)
torch.cuda.synchronize()
print("ok")
