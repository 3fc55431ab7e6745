"""Image-batch data parallelism (SURVEY §8(e), configs[3]).

Independent image fits shard naturally: rank r of G takes images
{r, r + G, ...} and fits them batched in ONE launch per stage (image index in
blockIdx.y / folded into the tile id).  Nothing crosses GPUs during the fit;
the only collective is the all-gather of per-image PSNR at the end (NCCL over
NVLink on GPUs; gloo in the CPU tests).  Plumbing only: every step of the fit
runs in libgi kernels.
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def shard(n_images: int, world: int, rank: int) -> list[int]:
    """Round-robin image indices owned by `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, int(n_images), world))


def gather_psnr(local: torch.Tensor, n_images: int, world: int, rank: int) -> torch.Tensor:
    """All-gather per-image PSNR (fp32) and return it in global image order.

    Ranks own different numbers of images when world does not divide
    n_images, so every rank contributes a buffer padded to the largest share.
    """
    per = (int(n_images) + world - 1) // world
    buf = torch.full((per,), float("nan"), dtype=torch.float32, device=local.device)
    buf[: local.numel()] = local.to(torch.float32)
    if world == 1:
        parts = [buf]
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
    out = torch.empty(int(n_images), dtype=torch.float32, device=local.device)
    for r in range(world):
        idx = shard(n_images, world, r)
        out[idx] = parts[r][: len(idx)]
    return out


def fit_sharded(n_images: int, steps: int, n_gauss: int, width: int, height: int,
                seed0: int = 100, device=None):
    """configs[3]: fit this rank's share of `n_images` synthetic images for
    `steps` fused Adam steps (one batched launch per stage), then gather the
    per-image PSNR.  Returns (psnr[n_images] on every rank, my image ids)."""
    import synth
    from . import gi
    from .pipeline import Fitter, Pipeline
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        raise RuntimeError("init the process group first")
    dev = device or torch.device("cuda", local)
    mine = shard(n_images, world, rank)
    if not mine:
        local_psnr = torch.zeros(0, device=dev)
    else:
        params = torch.from_numpy(
            np.stack([synth.init_params(seed0 + i, n_gauss) for i in mine])).to(dev)
        target = torch.from_numpy(
            np.stack([synth.image(seed0 + i, width, height) for i in mine])).to(dev)
        fit = Fitter(params.contiguous(), target.contiguous())
        for _ in range(steps):
            fit.step()
        if fit.check() != gi.GI_OK:
            raise RuntimeError("fit status not OK")
        pipe = Pipeline(n_gauss, width, height, len(mine), device=dev)
        img = pipe.render_frame(fit.params)
        local_psnr = pipe.psnr(img, fit.target).clone()
    return gather_psnr(local_psnr, n_images, world, rank), mine


if __name__ == "__main__":
    # torchrun --nproc-per-node G -m paper_2403_08551_b200.dist [n_images steps]
    import sys
    n_img = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    rank, world, local = env_rank_world()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    ps, mine = fit_sharded(n_img, steps, 70000, 768, 512)
    if rank == 0:
        print({"images": n_img, "ranks": world, "mean_psnr": float(ps.mean()), "psnr": ps.tolist()})
    if world > 1:
        dist.destroy_process_group()
