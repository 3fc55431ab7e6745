#!/usr/bin/env python
"""Diagnostic: stage times of one C2 fit step (cold L2), chained and plain,
from a captured graph with external event nodes at the stage boundaries
(gi_fit_step's stage_events): project | tile kernel | finalize (+Adam, +next
projection when chained).  Event nodes separate the kernels, so there is no
PDL overlap inside this graph: the stages are each kernel alone."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter  # noqa: E402


def main():
    W, H, n = 768, 512, 70000
    reps = int(os.environ.get("REPS", "100"))
    fitted = os.environ.get("CLOUD", "init") == "fitted"
    p0 = synth.fitted_params(1, n) if fitted else synth.init_params(1, n)
    p = torch.from_numpy(p0).cuda().view(1, n, 8).contiguous()
    t = torch.from_numpy(synth.image(1, W, H)).cuda().view(1, 3, H, W).contiguous()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for chained in (True, False):
        fit = Fitter(p.clone(), t, chained=chained)
        fit.step()
        ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(6)]
        for e in ev:
            e.record(stream)
        torch.cuda.synchronize()
        g = fit.capture(1, stage_events=ev)
        for _ in range(10):
            g.replay()
        acc = np.zeros(5)
        for _ in range(reps):
            flush.zero_()
            g.replay()
            torch.cuda.synchronize()
            acc += [ev[i].elapsed_time(ev[i + 1]) * 1000 for i in range(5)]
        acc /= reps
        print(json.dumps({"chained": chained, "cloud": "fitted" if fitted else "init",
                          "project_us": round(acc[0], 2), "tile_us": round(acc[2], 2),
                          "finalize_us": round(acc[3], 2)}), flush=True)


if __name__ == "__main__":
    main()
