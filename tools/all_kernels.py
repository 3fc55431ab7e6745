#!/usr/bin/env python
"""Diagnostic (for `ncu --set full -k regex:gi::`): every libgi kernel once on
C2-sized inputs (a 3-image launch for the two-pixel tile kernel) -- the gi_bin path (count, scan, scatter, segsort), render,
the unfused backward (alloc, tile, finalize, loss), Adam, Adan, decode,
encode, K-means, PSNR, the fused frame and fit steps."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200 import gi  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter, Pipeline, _bytes  # noqa: E402

W, H, N, SEED = 768, 512, 70000, 1
dev = torch.device("cuda")
p = torch.from_numpy(synth.init_params(SEED, N)).to(dev)[None].contiguous()
t = torch.from_numpy(synth.image(SEED, W, H)).to(dev)[None].contiguous()
pipe = Pipeline(N, W, H, 1)
pipe.render(p)                      # project, gi_bin (count, scan, scatter, segsort), render
pipe.backward(p, target=t)          # alloc, tile (gi_render_backward), finalize, loss
pipe.psnr(pipe.image, t)
pipe.render_frame(p)                # project + direct binning, render
m = torch.zeros_like(p)
v = torch.zeros_like(p)
gi.gi_adam_step(p.clone(), pipe.grads, m, v, N * 8, 1, 1e-3)
nn = torch.zeros_like(p)
gp = torch.zeros_like(p)
gi.gi_adan_step(p.clone(), pipe.grads, m, v, nn, gp, N * 8, 1, 1e-3)
data, gamma, beta, books = synth.payload(SEED, N)
meta = gi.codec_meta(N, gamma, beta, torch.from_numpy(books).to(dev))
dparams = torch.zeros(1, N, 8, dtype=torch.float32, device=dev)
gi.gi_vq_decode(torch.from_numpy(data).to(dev), meta, dparams)
pay = torch.zeros((N * 56 + 7) // 8 + 16, dtype=torch.uint8, device=dev)
eff = torch.zeros(N, 8, dtype=torch.float32, device=dev)
gi.gi_vq_encode(dparams[0], meta, pay, eff, flags=gi.GI_POS_NORMALIZED)
pts = dparams[0, :, 5:8].contiguous()
cent = pts[:8].clone()
assign = torch.zeros(N, dtype=torch.int32, device=dev)
gi.gi_kmeans_step(pts, cent, assign, _bytes(gi.gi_kmeans_workspace_bytes(8), dev))
fit = Fitter(p.clone(), t)
for _ in range(3):
    fit.step()                      # chained: tile kernel + finalize (+ next projection)
pb = p.repeat(3, 1, 1).contiguous()     # 3 images per launch: the two-pixel tile kernel
fb = Fitter(pb, t.repeat(3, 1, 1, 1).contiguous())
fb.step()
fa = Fitter(p.clone(), t, optimizer="adan")
fa.step()                           # finalize_kernel<true> (fused Adan)
torch.cuda.synchronize()
print("ok", pipe.keys(), fit.n_keys())
