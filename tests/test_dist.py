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
