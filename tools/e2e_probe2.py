#!/usr/bin/env python
"""Diagnostic: the bench's pipelined e2e loop with parts switched off, to see
which part bounds it on a given box (H2D, L2 flush, loss read-back, host)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2403_08551_b200.pipeline import Fitter  # noqa: E402

W, H, N = 768, 512, 70000
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
t_host = synth.image(1, W, H)[None]
params = torch.from_numpy(synth.init_params(1, N)).to(dev)[None].contiguous()
pinned_t = torch.from_numpy(t_host).pin_memory()
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
tbuf = [torch.from_numpy(t_host).to(dev).contiguous() for _ in range(2)]
fit = Fitter(params.clone(), tbuf[0])
cs = torch.cuda.Stream()
ds = torch.cuda.Stream()
copied = [torch.cuda.Event() for _ in range(2)]
consumed = [torch.cuda.Event() for _ in range(2)]
ploss = torch.zeros(1000, dtype=torch.float32).pin_memory()


def run(K, h2d=True, fl=True, d2h=True):
    cs.wait_stream(stream)
    if h2d:
        with torch.cuda.stream(cs):
            tbuf[0].copy_(pinned_t, non_blocking=True)
            copied[0].record(cs)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.record(stream)
    for i in range(K):
        b = i & 1
        if h2d and i + 1 < K:
            if i >= 1:
                cs.wait_event(consumed[b ^ 1])
            with torch.cuda.stream(cs):
                tbuf[b ^ 1].copy_(pinned_t, non_blocking=True)
                copied[b ^ 1].record(cs)
        if fl:
            flush.zero_()
        if h2d:
            stream.wait_event(copied[b])
        fit.target = tbuf[b]
        if d2h == "mapped":
            fit.step(loss_out=ploss[i % 1000].data_ptr())
        else:
            fit.step()
        consumed[b].record(stream)
        if d2h is True:
            ds.wait_event(consumed[b])
            with torch.cuda.stream(ds):
                ploss[i % 1000].copy_(fit.loss[0], non_blocking=True)
    stream.wait_stream(cs)
    stream.wait_stream(ds)
    e.record(stream)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return K / (s.elapsed_time(e) / 1000), K / (t1 - t0), K / (t2 - t0)


fit.step()
for args in (dict(), dict(d2h="mapped"), dict(fl=False), dict(d2h=False), dict(h2d=False),
             dict(h2d=False, fl=False, d2h=False)):
    run(20, **args)
    dev_its, host_enq, host_tot = run(200, **args)
    print(args, "device it/s", round(dev_its), "host enqueue it/s", round(host_enq), "wall it/s", round(host_tot))
