#!/usr/bin/env python
"""Diagnostic: fit step time of the chained / plain fused step, with and
without an L2 flush before each step (CUDA graph of one step, CUDA events)."""
from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter  # noqa: E402


def main():
    W, H, n = 768, 512, 70000
    reps = int(os.environ.get("REPS", "200"))
    p = torch.from_numpy(synth.init_params(1, n)).cuda().view(1, n, 8).contiguous()
    t = torch.from_numpy(synth.image(1, W, H)).cuda().view(1, 3, H, W).contiguous()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for chained in (True, False):
        fit = Fitter(p.clone(), t, chained=chained)
        fit.step()
        fit.capture(1)
        for _ in range(20):
            fit.replay()
        torch.cuda.synchronize()
        for fl in (True, False):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(reps)]
            for a, b in ev:
                if fl:
                    flush.zero_()
                a.record()
                fit.replay()
                b.record()
            torch.cuda.synchronize()
            ts = sorted(a.elapsed_time(b) * 1000 for a, b in ev)
            print(json.dumps({"chained": chained, "flush": fl, "us_median": round(ts[len(ts) // 2], 2),
                              "us_mean": round(sum(ts) / len(ts), 2)}), flush=True)


if __name__ == "__main__":
    main()
