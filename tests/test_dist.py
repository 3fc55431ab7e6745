"""Multi-process host logic of the image-batch data parallelism on CPU
(gloo, world size 2): sharding covers every image exactly once, and the PSNR
all-gather returns every image's value in global order on every rank."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_08551_b200.dist import gather_psnr, shard


def test_shard_partitions():
    for n in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            seen = sorted(i for r in range(world) for i in shard(n, world, r))
            assert seen == list(range(n))
            sizes = [len(shard(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_images, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(n_images, world, rank)
    local = torch.tensor([100.0 + i for i in mine], dtype=torch.float32)   # fake per-image PSNR
    out = gather_psnr(local, n_images, world, rank)
    q.put((rank, out.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_images", [64, 7])
def test_psnr_all_gather_gloo_world2(n_images):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_images, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [100.0 + i for i in range(n_images)]
    assert res[0] == want and res[1] == want


def test_gather_single_rank():
    out = gather_psnr(torch.tensor([1.0, 2.0, 3.0]), 3, 1, 0)
    assert out.tolist() == [1.0, 2.0, 3.0]


# ----------------------------------------------------------------- NEXT-4
from paper_2403_08551_b200.dist import SpatialFitter, row_windows   # noqa: E402


def test_row_windows_partition():
    for rows in (1, 5, 32, 85):
        for world in (1, 2, 3, 8):
            w = row_windows(rows, world)
            assert len(w) == world
            cover = [r for (r0, n) in w for r in range(r0, r0 + n)]
            assert cover == list(range(rows))
            assert max(n for _, n in w) - min(n for _, n in w) <= 1


TY = 32


def _fake_grads(params, r0, rows):
    # a per-window share that sums to the whole image's over any partition
    return torch.sin(params) * (rows / TY) * (1.0 + 0.0 * r0), torch.tensor([rows / TY])


def _torch_adam(params, grads, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    # CPU stand-in for gi_adam_step in the collective-plumbing tests (the
    # textbook update; the product path runs libgi's kernel)
    m.mul_(b1).add_(grads, alpha=1 - b1)
    v.mul_(b2).addcmul_(grads, grads, value=1 - b2)
    params.sub_(lr * (m / (1 - b1 ** t)) / ((v / (1 - b2 ** t)).sqrt() + eps))


def _spatial_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    p = torch.randn(1, 50, 8)
    t = torch.zeros(1, 3, 16 * TY, 64)
    fit = SpatialFitter(p.clone(), t, rank, world, grad_fn=_fake_grads, adam_fn=_torch_adam)
    for _ in range(3):
        fit.step()
    q.put((rank, fit.params.clone(), float(fit.loss[0]), fit.window))
    dist.barrier()
    dist.destroy_process_group()


def test_spatial_sharding_gloo_world2():
    # the rank windows partition the rows, the all-reduced gradient and loss
    # equal the single-process ones and the replicas stay identical
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spatial_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (pp, l, w)) for r, pp, l, w in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    torch.manual_seed(0)
    p = torch.randn(1, 50, 8)
    ref = SpatialFitter(p.clone(), torch.zeros(1, 3, 16 * TY, 64), 0, 1, grad_fn=_fake_grads, adam_fn=_torch_adam)
    for _ in range(3):
        ref.step()
    assert res[0][2] == (0, TY // 2) and res[1][2] == (TY // 2, TY // 2)
    assert torch.equal(res[0][0], res[1][0])
    assert torch.allclose(res[0][0], ref.params, atol=1e-6)
    assert abs(res[0][1] - 1.0) < 1e-6
