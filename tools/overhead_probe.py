#!/usr/bin/env python
"""Diagnostic: what a bench step costs besides the tile kernel.  Times, with
bench.py's protocol (L2 flush, events around one graph replay):
  empty  -- a graph holding one 1-element torch kernel (replay overhead);
  fit    -- the chained C2 fit step (the bench's `value` graph);
  fit x4 -- four chained steps in one graph, no flush between them (per step).
"""
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
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    s_ev = torch.cuda.Event(enable_timing=True)
    e_ev = torch.cuda.Event(enable_timing=True)

    def timed(g, do_flush=True):
        for _ in range(10):
            g.replay()
        tot = 0.0
        for _ in range(reps):
            if do_flush:
                flush.zero_()
            s_ev.record(stream)
            g.replay()
            e_ev.record(stream)
            torch.cuda.synchronize()
            tot += s_ev.elapsed_time(e_ev)
        return tot / reps * 1000.0

    x = torch.zeros(1, device=dev)
    s = torch.cuda.Stream()
    s.wait_stream(stream)
    g0 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g0, stream=s):
        x.add_(1.0)
    stream.wait_stream(s)
    out = {"empty_us": round(timed(g0), 2)}

    p = torch.from_numpy(synth.init_params(1, n)).to(dev).view(1, n, 8).contiguous()
    t = torch.from_numpy(synth.image(1, W, H)).to(dev).view(1, 3, H, W).contiguous()
    fit = Fitter(p.clone(), t)
    fit.step()
    g1 = fit.capture(1)
    out["fit_us"] = round(timed(g1), 2)
    g4 = fit.capture(4)
    out["fit_x4_per_step_us"] = round(timed(g4) / 4, 2)
    out["fit_x4_noflush_per_step_us"] = round(timed(g4, do_flush=False) / 4, 2)

    def eager(fn):
        for _ in range(10):
            fn()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            s_ev.record(stream)
            fn()
            e_ev.record(stream)
            torch.cuda.synchronize()
            tot += s_ev.elapsed_time(e_ev)
        return tot / reps * 1000.0

    out["fit_eager_us"] = round(eager(fit.step), 2)
    from paper_2403_08551_b200.pipeline import Pipeline
    pipe = Pipeline(n, W, H, 1)
    out["render_eager_us"] = round(eager(lambda: pipe.render_frame(p)), 2)
    gr = torch.cuda.CUDAGraph()
    s.wait_stream(stream)
    with torch.cuda.graph(gr, stream=s):
        pipe.render_frame(p)
    stream.wait_stream(s)
    out["render_graph_us"] = round(timed(gr), 2)
    # R independent fits (same seeded problem, separate buffers) stepped in
    # turn inside one graph: each step's working set (~35 MB) was evicted by
    # the other R-1 fits' steps (R x 35 MB > 2 x L2), so no flush is needed
    for R in (4, 8):
        fits = [Fitter(p.clone(), t.clone()) for _ in range(R)]
        for f in fits:
            f.step()
        torch.cuda.synchronize()
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        gR = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gR, stream=gs):
            for f in fits:
                f.step()
        stream.wait_stream(gs)
        out[f"fit_rot{R}_per_step_us"] = round(timed(gR, do_flush=False) / R, 2)
        out[f"fit_rot{R}_flushed_per_step_us"] = round(timed(gR) / R, 2)
        del fits, gR
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
