#!/usr/bin/env python
"""Diagnostic: how far the CUDA path sits from the parity bars (max pixel
error vs 2e-5, per-group gradient rel. L2 vs 1e-4) on the test cases, for the
fused fit kernels (gi_render_backward) and the render kernel.  Oracle = the
fp64 CPU reference (test infrastructure)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import gio  # noqa: E402
from paper_2403_08551_b200.pipeline import Pipeline  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_state import near_line_params  # noqa: E402

CASES = {"c1": (64, 64, 256, 0, False), "ragged": (70, 45, 300, 1, False),
         "c1_fitted": (64, 64, 256, 3, True), "c2_init": (768, 512, 70000, 1, False),
         "c2_fitted": (768, 512, 70000, 1, True), "c3_init": (2040, 1356, 100000, 2, False),
         "nearline_999_0.1": (96, 80, 300, 5, "nearline"),
         "clustered": (256, 192, 30000, 3, "clustered")}
for name, (W, H, n, seed, fitted) in CASES.items():
    if fitted == "nearline":
        p = near_line_params(1000, n, 0.999, 0.1)
    elif fitted == "clustered":
        p = synth.clustered_params(seed, n, W, H, clusters=4, frac=0.5, radius_px=6.0)
    else:
        p = synth.fitted_params(seed, n) if fitted else synth.init_params(seed, n)
    t = synth.image(seed, W, H)
    mode = gio.ALL_PAIRS if W * H * n <= 64 * 64 * 300 else gio.TILED
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, t, mode=mode)
    pipe = Pipeline(n, W, H, 1)
    pd = torch.from_numpy(p).cuda()[None].contiguous()
    img = pipe.render_frame(pd)[0].cpu().numpy()     # the fused frame (the bench's path)
    pipe.render(pd)
    pipe.backward(pd, target=torch.from_numpy(t).cuda()[None].contiguous())
    g = pipe.grads[0].cpu().numpy().astype(np.float64)
    errs = {k: np.linalg.norm(g[:, c] - ref_g[:, c]) / np.linalg.norm(ref_g[:, c])
            for k, c in (("mu", [0, 1]), ("l", [2, 3, 4]), ("c", [5, 6, 7]))}
    pix = float(np.abs(img - ref_img).max())
    pix_scaled = float((np.abs(img - ref_img) / np.maximum(1.0, np.abs(ref_img))).max())
    print(f"{name:16s} pixel max err {pix:.2e} ({pix / 2e-5:5.1%} of bar; scaled {pix_scaled:.1e})  grads "
          + "  ".join(f"{k} {v:.2e} ({v / 1e-4:5.1%})" for k, v in errs.items())
          + f"  loss rel {abs(float(pipe.loss[0]) - ref_loss) / ref_loss:.1e}", flush=True)
