#!/usr/bin/env python
"""Diagnostic: pinned H2D / D2H bandwidth for the e2e target size, one copy
vs the same bytes split over several streams."""
import torch

MB = 4.5
n = int(MB * (1 << 20) / 4)
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    chunk = (n + parts - 1) // parts
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        torch.cuda.synchronize()
        s.record()
        for _ in range(20):
            for i, st in enumerate(streams):
                st.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(st):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
            for st in streams:
                torch.cuda.current_stream().wait_stream(st)
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"H2D {MB} MB in {parts} part(s): {ms * 1000:.1f} us, {MB * (1 << 20) / ms / 1e6:.1f} GB/s")
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    h.copy_(d, non_blocking=True)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"D2H {MB} MB: {ms * 1000:.1f} us, {MB * (1 << 20) / ms / 1e6:.1f} GB/s")
