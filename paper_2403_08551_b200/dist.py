"""Multi-GPU plumbing: image-batch data parallelism (SURVEY §8(e),
configs[3]) and single-image spatial sharding (NEXT-4, §8(f)).

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
        # NCCL gathers device buffers; gloo (CPU tests, several ranks sharing
        # one GPU in the multi-rank tests) gathers host-staged copies
        staged = buf.cpu() if buf.is_cuda and dist.get_backend() == "gloo" else buf
        parts = [torch.empty_like(staged) for _ in range(world)]
        dist.all_gather(parts, staged)
        parts = [p.to(local.device) for p in parts]
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


# ------------------------------------------------------------------ NEXT-4
def row_windows(tile_rows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous tile-row windows (row0, rows) of one image, one per rank,
    covering [0, tile_rows) exactly once, sizes differing by at most one."""
    if world < 1:
        raise ValueError("world")
    base, extra = divmod(int(tile_rows), world)
    out, r0 = [], 0
    for r in range(world):
        rows = base + (1 if r < extra else 0)
        out.append((r0, rows))
        r0 += rows
    return out


class SpatialFitter:
    """Single-image spatial sharding (NEXT-4): every rank holds all Gaussians
    (replicated params and Adam state), renders and back-propagates only its
    tile rows (gi_fit_grads), the per-Gaussian gradients and the loss are
    summed across ranks (the one real exchange of the path: NCCL all_reduce on
    GPUs, gloo in the CPU tests), and every rank applies the same Adam update
    (gi_adam_step), so the replicas stay bit-identical.

    grad_fn(params, row0, rows) -> (grads, loss) may replace the libgi call
    (CPU tests of the collective plumbing).

    adam_fn(params, grads, m, v, t, lr) may replace gi_adam_step (with
    grad_fn: the CPU tests' stand-in; the product path takes neither).  The
    learning rate is gi_lr_at's schedule (the library's definition, R17).

    Measurement status: NEXT-4 has only run with G ranks on ONE GPU (two
    processes, host barriers); it is unmeasured across GPUs.  Each step has
    two host synchronisations + process-group barriers, ~tens of us against a
    ~80 us C3 step on one B200, so at G = 2 it is likely SLOWER than one GPU
    until those become device-side flags in peer memory (not built: a flag
    barrier cannot be exercised with one GPU).

    exchange="peer" (GPU ranks of one node): instead of all_reduce + Adam,
    every rank writes its window's gradients and loss into an IPC-mapped
    exchange buffer (gi_peer_alloc / gi_peer_open, handles swapped over the
    process group) and gi_peer_adam_step sums the G buffers in rank order and
    applies Adam in one kernel, reading the peers' gradients over NVLink.  The
    process group only carries the handles and the two barriers per step."""

    def __init__(self, params: torch.Tensor, target: torch.Tensor, rank: int = 0, world: int = 1,
                 k: float = 3.0, key_capacity: int | None = None, lr0: float = 1e-3,
                 half_every: int = 20000, grad_fn=None, flags: int = 0, exchange: str = "nccl",
                 adam_fn=None):
        self.rank, self.world = int(rank), int(world)
        self.params = params.contiguous()
        self.target = target.contiguous()
        self.grads = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.params.device)
        self.t = 0
        self.lr0, self.half_every = lr0, half_every
        H, W = target.shape[-2], target.shape[-1]
        self.n = self.params.shape[-2]
        self.window = row_windows((H + 15) // 16, self.world)[self.rank]
        self.grad_fn = grad_fn
        self.adam_fn = adam_fn
        if (grad_fn is None) != (adam_fn is None):
            raise ValueError("grad_fn and adam_fn replace the libgi calls together (CPU tests)")
        self.flags = flags
        from . import gi
        self.gi = gi
        if grad_fn is None:
            from .pipeline import _bytes, default_capacity
            self.f = gi.frame(W, H, 1, k)
            self.cap = int(key_capacity) if key_capacity else default_capacity(self.n, 1)
            self.ws = _bytes(gi.gi_fit_workspace_bytes(self.n, self.cap, self.f), self.params.device)
        if exchange not in ("nccl", "peer"):
            raise ValueError("exchange must be 'nccl' or 'peer'")
        self.exchange = exchange
        if exchange == "peer":
            if grad_fn is not None:
                raise ValueError("the peer exchange runs on libgi device buffers")
            self.count = self.params.numel()
            self.buf, handle = self.gi.gi_peer_alloc(4 * (self.count + 1))
            handles = [handle]
            if self.world > 1:
                handles = [None] * self.world
                dist.all_gather_object(handles, handle)
            self.peers = [self.buf if r == self.rank else self.gi.gi_peer_open(handles[r])
                          for r in range(self.world)]

    def close(self):
        """Unmap the peers' exchange buffers and free this rank's (peer mode)."""
        if getattr(self, "exchange", "nccl") == "peer" and self.buf:
            if self.world > 1:
                torch.cuda.synchronize()
                dist.barrier()
            for r, ptr in enumerate(self.peers):
                if r != self.rank:
                    self.gi.gi_peer_close(ptr)
            self.gi.gi_peer_free(self.buf)
            self.buf = 0

    def local_grads(self):
        r0, rows = self.window
        if self.grad_fn is not None:
            g, l = self.grad_fn(self.params, r0, rows)
            self.grads.copy_(g)
            self.loss.copy_(l)
            return
        self.gi.gi_fit_grads(self.params, self.grads, self.target, self.n, self.f, self.flags, r0,
                             rows, self.cap, self.ws, self.loss)

    def _peer_step(self):
        r0, rows = self.window
        # this rank's window gradients + loss into its exchange buffer
        self.gi.gi_fit_grads(self.params, self.buf, self.target, self.n, self.f, self.flags, r0,
                             rows, self.cap, self.ws, self.buf + 4 * self.count)
        if self.world > 1:                 # every rank's buffer complete
            torch.cuda.synchronize()
            dist.barrier()
        self.t += 1
        lr = self.gi.gi_lr_at(self.t, self.lr0, self.half_every)
        self.gi.gi_peer_adam_step(self.params, self.m, self.v, self.peers, self.count, self.t, lr,
                                  n_loss=1, loss_out=self.loss)
        if self.world > 1:                 # every peer read done before the next overwrite
            torch.cuda.synchronize()
            dist.barrier()

    def step(self):
        if self.exchange == "peer":
            self._peer_step()
            return
        self.local_grads()
        if self.world > 1:
            dist.all_reduce(self.grads, op=dist.ReduceOp.SUM)
            dist.all_reduce(self.loss, op=dist.ReduceOp.SUM)
        self.t += 1
        lr = self.gi.gi_lr_at(self.t, self.lr0, self.half_every)
        if self.adam_fn is not None:
            self.adam_fn(self.params, self.grads, self.m, self.v, self.t, lr)
        else:
            self.gi.gi_adam_step(self.params, self.grads, self.m, self.v, self.params.numel(),
                                 self.t, lr)


if __name__ == "__main__":
    # torchrun --nproc-per-node G -m paper_2403_08551_b200.dist [n_images steps]
    import sys
    n_img = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    n_g = int(sys.argv[3]) if len(sys.argv) > 3 else 70000
    W = int(sys.argv[4]) if len(sys.argv) > 4 else 768
    H = int(sys.argv[5]) if len(sys.argv) > 5 else 512
    rank, world, local = env_rank_world()
    dev = torch.device("cuda", local % torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(dev)
        # GI_DIST_BACKEND=gloo: several ranks on one GPU (tests); NCCL otherwise
        dist.init_process_group(os.environ.get("GI_DIST_BACKEND", "nccl"))
    ps, mine = fit_sharded(n_img, steps, n_g, W, H, device=dev)
    if rank == 0:
        import json
        print(json.dumps({"images": n_img, "ranks": world, "mean_psnr": float(ps.mean()),
                          "psnr": ps.tolist()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
