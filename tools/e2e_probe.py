import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import synth
from paper_2403_08551_b200.pipeline import Fitter
W, H, N = 768, 512, 70000
dev = torch.device('cuda')
p = torch.from_numpy(synth.init_params(1, N)).to(dev)[None].contiguous()
t_host = synth.image(1, W, H)[None]
target = torch.from_numpy(t_host).to(dev).contiguous()
pinned = torch.from_numpy(t_host).pin_memory()
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
fit = Fitter(p.clone(), target)
stream = torch.cuda.current_stream()
def run(mode, K=200, do_flush=True):
    cs = torch.cuda.Stream()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); s.record()
    for i in range(K):
        if mode == 'copy':
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                target.view(-1).copy_(pinned.view(-1), non_blocking=True)
            stream.wait_stream(cs)
        if do_flush: flush.zero_()
        fit.step()
    e.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(mode, 'flush' if do_flush else 'noflush', 'device it/s', round(K / (s.elapsed_time(e) / 1000)), 'host it/s', round(K / (t1 - t0)))
for m in ('none', 'copy'):
    for f in (True, False):
        run(m, do_flush=f)
# host cost of one step() call alone
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(200): fit.step()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print('enqueue us/step', (t1 - t0) / 200 * 1e6, 'total us/step', (t2 - t0) / 200 * 1e6)
