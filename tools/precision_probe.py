#!/usr/bin/env python
"""Diagnostic: gradient / pixel error of the CUDA path against the fp64
oracle on near-line (highly anisotropic) Gaussians and on unrestricted fuzz
clouds, with the worst individual Gaussians listed (parameters + per-Gaussian
relative error) -- to locate where fp32 loses the 1e-4 bar."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import gio  # noqa: E402
from paper_2403_08551_b200.pipeline import Pipeline  # noqa: E402

GROUPS = {"mu": [0, 1], "l": [2, 3, 4], "c": [5, 6, 7]}


def near_line(seed, n, W, H, rho=0.999, smin=0.2):
    """Gaussians with correlation rho and minor-axis sigma smin (px): Sigma =
    R diag(smaj^2, smin^2) R^T with random angle, smaj in [2, 8]; L = chol."""
    rng = np.random.default_rng(seed)
    p = synth.init_params(seed, n).astype(np.float64)
    for i in range(n):
        smaj = rng.uniform(2.0, 8.0)
        th = rng.uniform(0, np.pi)
        c, s = np.cos(th), np.sin(th)
        R = np.array([[c, -s], [s, c]])
        S = R @ np.diag([smaj ** 2, smin ** 2]) @ R.T
        l1 = np.sqrt(S[0, 0])
        l2 = S[1, 0] / l1
        l3 = np.sqrt(S[1, 1] - l2 * l2)
        sg = rng.choice([-1.0, 1.0], size=2)
        p[i, 2] = sg[0] * l1 - 0.5
        p[i, 3] = sg[0] * l2
        p[i, 4] = sg[1] * l3 - 0.5
    return p.astype(np.float32)


def fuzz_unrestricted(seed, n):
    rng = np.random.default_rng(seed)
    p = synth.init_params(int(rng.integers(1 << 30)), n) if rng.random() < 0.5 else \
        synth.fitted_params(int(rng.integers(1 << 30)), n)
    k = rng.random(n)
    p[k < 0.05, 2] = -0.5
    p[(k >= 0.05) & (k < 0.1), 4] = -0.5
    neg = (k >= 0.1) & (k < 0.2)
    m = int(neg.sum())
    p[neg, 2] = -rng.uniform(0.0, 3.0, size=m)
    p[neg, 3] = rng.uniform(-3.0, 3.0, size=m)
    p[neg, 4] = -rng.uniform(0.0, 3.0, size=m)
    edge = (k >= 0.2) & (k < 0.3)
    p[edge, 0:2] = rng.choice([-4.0, 4.0], size=(int(edge.sum()), 2)) * \
        rng.uniform(0.5, 1.0, size=(int(edge.sum()), 2))
    huge = (k >= 0.3) & (k < 0.32)
    p[huge, 2] = rng.uniform(10, 60, size=int(huge.sum()))
    p[huge, 4] = rng.uniform(10, 60, size=int(huge.sum()))
    p[(k >= 0.32) & (k < 0.4), 5:8] *= -1.0
    return p.astype(np.float32)


def run(name, p, W, H, tgt, show=3):
    n = len(p)
    mode = gio.ALL_PAIRS if W * H * n <= 20_000_000 else gio.TILED
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=mode)
    pipe = Pipeline(n, W, H, 1)
    pd = torch.from_numpy(p).cuda()[None].contiguous()
    img = pipe.render_frame(pd)[0].cpu().numpy()
    pipe.render(pd)
    pipe.backward(pd, target=torch.from_numpy(tgt).cuda()[None].contiguous())
    g = pipe.grads[0].cpu().numpy().astype(np.float64)
    errs = {k: np.linalg.norm(g[:, c] - ref_g[:, c]) / max(np.linalg.norm(ref_g[:, c]), 1e-300)
            for k, c in GROUPS.items()}
    pix = float(np.abs(img - ref_img).max())
    peak = float(np.abs(ref_img).max())
    print(f"{name:18s} n={n:6d} peak|C|={peak:7.2f} pix {pix:.2e}  "
          + "  ".join(f"{k} {v:.2e}" for k, v in errs.items())
          + f"  loss rel {abs(float(pipe.loss[0]) - ref_loss) / max(ref_loss, 1e-30):.1e}", flush=True)
    # contribution of each Gaussian to the group error
    for k, c in GROUPS.items():
        d = np.linalg.norm(g[:, c] - ref_g[:, c], axis=1)
        den = np.linalg.norm(ref_g[:, c])
        worst = np.argsort(-d)[:show]
        for i in worst:
            rel_i = d[i] / max(np.linalg.norm(ref_g[i, c]), 1e-300)
            print(f"   {k:2s} g{i:6d} share {d[i] / den:.2e} self-rel {rel_i:.2e} "
                  f"params {np.array2string(p[i], precision=3, max_line_width=200)}")
    return errs, pix


if __name__ == "__main__":
    for smin in (0.5, 0.2, 0.1):
        for rho_seed in range(2):
            W, H, n = 96, 80, 200
            p = near_line(100 + rho_seed, n, W, H, smin=smin)
            run(f"nearline s={smin} #{rho_seed}", p, W, H, synth.image(rho_seed, W, H))
    for seed in range(12):
        rng = np.random.default_rng(1000 + seed)
        W, H = int(rng.integers(1, 200)), int(rng.integers(1, 150))
        n = int(rng.integers(1, 1500))
        p = fuzz_unrestricted(5000 + seed, n)
        run(f"fuzz #{seed}", p, W, H, synth.image(seed, W, H), show=1)
