"""The world > 1 code paths on the one GPU this pool gives: bench.py and
dist.fit_sharded launched by torchrun with 2 ranks sharing cuda:0 over gloo
(GI_DIST_BACKEND=gloo; host-staged collectives).  The ranks' kernels never
wait on one another -- image fits are independent -- so this
exercises the plumbing (value aggregation over ranks, max-over-ranks timing,
image sharding, the PSNR gather in global image order), not scaling."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(args, nproc, timeout=900):
    env = dict(os.environ, GI_DIST_BACKEND="gloo", PYTHONPATH=ROOT)
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
               "--master-port", str(_port())] + args
    else:
        cmd = [sys.executable] + args
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]      # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_two_ranks():
    K = 5
    d = _run(["bench.py", "--gpus", "2", "--steps", str(K), "--warmup", "3", "--quick",
              "--no-cpu-baseline"], 2)
    assert d["n_gpus"] == 2 and d["steps"] == K and d["scaling"] == "weak"
    assert len(d["rank_ms"]) == 2 and all(ms > 0 for ms in d["rank_ms"])
    t = max(d["rank_ms"])                               # max over ranks
    assert d["value"] == pytest.approx(2 * K / (t / 1000.0), rel=1e-9)
    assert d["ms_per_step"] == pytest.approx(t / K, rel=1e-9)
    assert len(d["psnr_db_after_fit_steps"]) == 2
    b = d["batched"]
    assert b["images_total"] == 4 and b["psnr_images"] == 4
    assert d["gpu_launches"] == K * d["gpu_launches_per_step"] > 0


def test_fit_sharded_two_ranks_matches_one():
    # 5 images over 2 ranks (3 + 2, round-robin) vs all 5 in one process: the
    # gathered PSNR is in global image order and bitwise equal (per-image fits
    # in a batched launch do not depend on the batch's other images)
    args = ["-m", "paper_2403_08551_b200.dist", "5", "20", "3000", "160", "96"]
    two = _run(args, 2)
    one = _run(args, 1)
    assert two["ranks"] == 2 and one["ranks"] == 1
    assert len(two["psnr"]) == 5
    assert two["psnr"] == one["psnr"]
