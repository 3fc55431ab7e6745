import torch, time
for mb in [1, 4.7, 16, 64]:
    n = int(mb * (1<<20) / 4)
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)/20
    print(f"H2D {mb} MB: {ms*1000:.1f} us, {mb*(1<<20)/ms/1e6:.1f} GB/s")
    s.record()
    for _ in range(20): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)/20
    print(f"D2H {mb} MB: {ms*1000:.1f} us, {mb*(1<<20)/ms/1e6:.1f} GB/s")
