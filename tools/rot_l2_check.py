#!/usr/bin/env python
"""Evidence for bench.py's L2-cold rotation (rot_ms): run under
  ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,
      lts__t_sector_hit_rate.pct -k regex:fused_tile_kernel
and compare the tile kernel's DRAM reads per launch in the two protocols:
  rot    -- 8 independent C2 fits stepped in turn inside one graph (no flush);
  flush  -- one fit, a 256 MB L2 flush before every single-step replay.
(One pass per kernel: the three metrics need no replay, so ncu does not
re-run a kernel on a cache the previous pass warmed.)"""
from __future__ import annotations

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "rot"
    W, H, n = 768, 512, 70000
    p = torch.from_numpy(synth.init_params(1, n)).cuda().view(1, n, 8).contiguous()
    t = torch.from_numpy(synth.image(1, W, H)).cuda().view(1, 3, H, W).contiguous()
    R = 8 if mode == "rot" else 1
    fits = [Fitter(p.clone(), t.clone()) for _ in range(R)]
    for f in fits:
        f.step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    gs = torch.cuda.Stream()
    gs.wait_stream(stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for f in fits:
            f.step()
    stream.wait_stream(gs)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3 if mode == "rot" else 16):
        if mode == "flush":
            flush.zero_()
        g.replay()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
