import sys, json, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2403_08551_b200.pipeline import Pipeline
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def timed(g, reps=50):
    ev=[(torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a,b in ev:
        flush.zero_(); a.record(); g.replay(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a,b in ev)[reps//2]
for W,H,N,B in ((2040,1356,100000,1),(768,512,70000,16),(768,512,70000,64)):
    p=torch.from_numpy(np.stack([synth.init_params(2+b,N) for b in range(B)])).cuda().contiguous()
    pipe=Pipeline(N,W,H,B); pipe.render_frame(p)
    s=torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream()); g=torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s): pipe.render_frame(p)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(5): g.replay()
    ms=timed(g); print(json.dumps({"W":W,"B":B,"image_fps":round(B*1000/ms)}), flush=True)
