import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, synth
from oracle import gio
from paper_2403_08551_b200.pipeline import Fitter, Pipeline
import importlib.util
spec = importlib.util.spec_from_file_location("tg", "tests/test_gpu_parity.py"); tg = importlib.util.module_from_spec(spec); spec.loader.exec_module(tg)
seed=3
rng = np.random.default_rng(2000 + seed)
B = int(rng.integers(2, 5)); W, H = int(rng.integers(8, 160)), int(rng.integers(8, 120)); n = int(rng.integers(1, 800))
ps = np.stack([tg.fuzz_regime(gio, tg.fuzz_params(rng, n), W, H) for _ in range(B)]); ts = np.stack([synth.image(50 + 7 * seed + b, W, H) for b in range(B)])
print("B,W,H,n",B,W,H,n)
fit = Fitter(torch.from_numpy(ps).cuda().contiguous(), torch.from_numpy(ts).cuda().contiguous()); fit.step(); torch.cuda.synchronize()
gg = fit.grads.cpu().numpy().astype(np.float64)
for b in range(B):
    ref_img, ref_loss, ref_g = gio.loss_and_grads(ps[b], ts[b], mode=gio.ALL_PAIRS)
    f1 = Fitter(torch.from_numpy(ps[b:b+1]).cuda().contiguous(), torch.from_numpy(ts[b:b+1]).cuda().contiguous()); f1.step(); torch.cuda.synchronize()
    g1 = f1.grads[0].cpu().numpy().astype(np.float64)
    for name, cols in tg.GROUPS.items():
        den = np.linalg.norm(ref_g[:, cols])
        print(b, name, "batched rel", np.linalg.norm(gg[b][:, cols]-ref_g[:, cols])/den, "single rel", np.linalg.norm(g1[:, cols]-ref_g[:, cols])/den, "batched==single", np.array_equal(gg[b][:,cols], g1[:,cols]), "maxpix", np.abs(ref_img).max(), "loss", ref_loss)
    worst = np.argsort(-np.abs(gg[b][:,0]-ref_g[:,0]))[:3]
    for w in worst: print("  g", w, ps[b][w], gg[b][w,:2], ref_g[w,:2])
