"""CUDA path vs the fp64 oracle at the states the method really produces and
on the inputs round 1's tests narrowed away, plus the workspace-state
contracts of the chained fit step.

* near-line Gaussians (correlation +-0.99 / +-0.999, minor-axis sigma 0.2 and
  0.1 px): any L with a non-zero diagonal is valid (Eq. 1), so the
  1e-4 gradient bar (north_star) holds for them too;
* a FITTED cloud: 2000 steps of the paper's fitting loop (L2 loss P:298,
  Adam with the P:381 schedule, reading R16/R17) run by the ORACLE from the
  paper's init (App. C) on a C2-density frame -- no input of the
  comparison comes from the CUDA path;
* direct binning: the per-tile key sets the timed fused paths build (counts
  and slab contents) bit-exact against the oracle's binning (R9);
* the fused optimiser: bitwise the arithmetic of gi_adam_step, which is
  checked against the oracle's Adam elementwise;
* re-priming after chained steps (gi_fit_prime / gi_fit_reset clear the
  pending keys a chained step leaves).
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
PIX_TOL = 2e-5
GRAD_TOL = 1e-4
GROUPS = {"mu": [0, 1], "l": [2, 3, 4], "c": [5, 6, 7]}


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def group_err(g, ref):
    return {k: np.linalg.norm(g[..., c] - ref[..., c]) / max(np.linalg.norm(ref[..., c]), 1e-300)
            for k, c in GROUPS.items()}


def near_line_params(seed, n, rho, smin):
    """Gaussians with correlation +-rho and minor-axis sigma smin (pixels):
    Sigma = [[sx^2, r sx sy], [r sx sy, sy^2]], sy/sx in [1/4, 4], scaled so
    the smaller eigenvalue is smin^2; L = chol(Sigma) with random signs on
    the diagonal (L L^T is unchanged), stored raw (l_ii - 1/2, R4).  Positions
    and colours from the paper's init."""
    rng = np.random.default_rng(seed)
    p = synth.init_params(seed, n).astype(np.float64)
    r = rng.uniform(0.25, 4.0, size=n)
    sgn = rng.choice([-1.0, 1.0], size=n)
    lam = (1 + r * r - np.sqrt((1 - r * r) ** 2 + 4 * rho * rho * r * r)) / 2   # sx = 1
    sx = smin / np.sqrt(lam)
    sy = r * sx
    l1 = sx
    l2 = sgn * rho * sy
    l3 = sy * np.sqrt(1 - rho * rho)
    d1 = rng.choice([-1.0, 1.0], size=n)
    d3 = rng.choice([-1.0, 1.0], size=n)
    p[:, 2] = d1 * l1 - 0.5
    p[:, 3] = d1 * l2
    p[:, 4] = d3 * l3 - 0.5
    return p.astype(np.float32)


@pytest.mark.parametrize("rho,smin", [(0.999, 0.2), (0.99, 0.2), (0.999, 0.1), (0.99, 0.1)])
def test_near_line_gaussians(gi, gio, rho, smin):
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 96, 80, 300
    p = near_line_params(int(rho * 1000) + int(smin * 10), n, rho, smin)
    # the construction really is near-line: |corr| and the minor axis as asked
    l1e, l2, l3e = p[:, 2] + 0.5, p[:, 3], p[:, 4] + 0.5
    S = np.stack([l1e * l1e, l1e * l2, l2 * l2 + l3e * l3e], 1).astype(np.float64)
    corr = S[:, 1] / np.sqrt(S[:, 0] * S[:, 2])
    assert np.allclose(np.abs(corr), rho, atol=1e-4)
    tgt = synth.image(5, W, H)
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    pipe = Pipeline(n, W, H, 1, device=DEV)
    img = pipe.render_frame(to_dev(p)[None].contiguous())[0].cpu().numpy()
    assert np.abs(img - ref_img).max() <= PIX_TOL
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    errs = group_err(fit.grads[0].cpu().numpy().astype(np.float64), ref_g)
    assert max(errs.values()) <= GRAD_TOL, errs
    assert abs(float(fit.loss[0]) - ref_loss) <= 1e-5 * ref_loss


# ---------------------------------------------------------------- fitted cloud
FIT_W, FIT_H, FIT_N, FIT_STEPS = 256, 192, 8750, 2000   # C2's density: 70k / (768 x 512)


@pytest.fixture(scope="module")
def fitted(gio):
    """The paper's fitting loop run by the oracle: init (App. C) -> 2000 Adam
    steps (lr 1e-3) on the L2 loss, fp64 arithmetic with the
    parameters and moments held in fp32 between steps."""
    p = synth.init_params(77, FIT_N)
    tgt = synth.image(77, FIT_W, FIT_H)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for t in range(1, FIT_STEPS + 1):
        _, _, g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
        po, mo, vo = gio.adam(p, g.astype(np.float32), m, v, t, gio.lr_at(t))
        p, m, v = po.astype(np.float32), mo.astype(np.float32), vo.astype(np.float32)
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
    return dict(p=p, tgt=tgt, img=ref_img, loss=ref_loss, g=ref_g)


def test_fitted_cloud_is_fitted(gio, fitted):
    # the state differs from the init the other tests use: a fitted loss,
    # denser tiles, Gaussians that went anisotropic / signed
    p0 = synth.init_params(77, FIT_N)
    _, l0, _ = gio.loss_and_grads(p0, fitted["tgt"], mode=gio.TILED)
    assert fitted["loss"] < 0.05 * l0
    p = fitted["p"]
    assert (p[:, 2] + 0.5 < 0).any() or (p[:, 4] + 0.5 < 0).any() or np.abs(p[:, 3]).max() > 1.0


def test_fitted_cloud_project_bin(gi, gio, fitted):
    from paper_2403_08551_b200.pipeline import Pipeline
    p = fitted["p"]
    pipe = Pipeline(FIT_N, FIT_W, FIT_H, 1, device=DEV)
    pipe.render(to_dev(p)[None].contiguous())
    torch.cuda.synchronize()
    kt, kg, rng = gio.bin(p, FIT_W, FIT_H)
    K = len(kt)
    assert pipe.keys() == K
    assert np.array_equal(pipe.key_tile[:K].cpu().numpy().view(np.uint32), kt)
    assert np.array_equal(pipe.key_gid[:K].cpu().numpy().view(np.uint32), kg)
    assert np.array_equal(pipe.tile_range[:len(rng)].cpu().numpy().view(np.uint32), rng)
    assert np.abs(pipe.image[0].cpu().numpy() - fitted["img"]).max() <= PIX_TOL


def test_fitted_cloud_frame_and_fit_step(gi, gio, fitted):
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    p, tgt = fitted["p"], fitted["tgt"]
    pipe = Pipeline(FIT_N, FIT_W, FIT_H, 1, device=DEV)
    img = pipe.render_frame(to_dev(p)[None].contiguous())[0].cpu().numpy()
    assert np.abs(img - fitted["img"]).max() <= PIX_TOL
    for chained in (True, False):
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), chained=chained)
        fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        errs = group_err(fit.grads[0].cpu().numpy().astype(np.float64), fitted["g"])
        assert max(errs.values()) <= GRAD_TOL, errs
        assert abs(float(fit.loss[0]) - fitted["loss"]) <= 1e-5 * fitted["loss"]


def test_fitted_cloud_direct_binning(gi, gio, fitted):
    _check_direct_binning(gi, gio, fitted["p"][None], FIT_W, FIT_H)


# ---------------------------------------------------------------- direct binning
def _bin_state(gi, fit):
    """(counts [B*T], per-tile sorted gid lists or None if the tile streams)."""
    tc, stride, sl, scap = gi.gi_fit_bin_view(fit.fit_ws, fit.n, fit.cap, fit.f)
    base = fit.fit_ws.data_ptr()
    words = fit.fit_ws.view(torch.int32)
    T = gi.gi_num_tiles(fit.f)
    BT = T * fit.B
    counts = words[(tc - base) // 4:(tc - base) // 4 + BT * stride:stride].cpu().numpy()
    counts = counts.view(np.uint32).astype(np.int64)
    slab = words[(sl - base) // 4:(sl - base) // 4 + BT * scap].cpu().numpy().view(np.uint32)
    lists = []
    for g in range(BT):
        c = int(counts[g])
        lists.append(np.sort(slab[g * scap:g * scap + c]) if c <= scap else None)
    return counts, lists, scap


def _check_direct_binning(gi, gio, ps, W, H, key_capacity=None):
    from paper_2403_08551_b200.pipeline import Fitter
    B, n = ps.shape[0], ps.shape[1]
    tgt = np.stack([synth.image(b, W, H) for b in range(B)])
    fit = Fitter(to_dev(ps).contiguous(), to_dev(tgt).contiguous(), key_capacity=key_capacity)
    gi.gi_fit_prime(fit.params, fit.n, fit.f, fit.flags, fit.cap, fit.fit_ws)
    torch.cuda.synchronize()
    counts, lists, scap = _bin_state(gi, fit)
    T = gi.gi_num_tiles(fit.f)
    streamed = 0
    for b in range(B):
        kt, kg, rng = gio.bin(ps[b], W, H)
        ref_counts = np.diff(rng.astype(np.int64))
        assert np.array_equal(counts[b * T:(b + 1) * T], ref_counts)
        for t in range(T):
            got = lists[b * T + t]
            if got is None:
                streamed += 1
                continue
            ref = kg[rng[t]:rng[t + 1]] + b * n  # ascending gid (R9); batch-global ids
            assert np.array_equal(got, ref), (b, t)
    return fit, streamed, scap


@pytest.mark.parametrize("cfg", ["c1", "ragged", "c2_init", "c2_fitted_proxy", "batch3"])
def test_direct_binning_slabs_bitexact(gi, gio, cfg):
    W, H, n, B, fitted = {"c1": (64, 64, 256, 1, False), "ragged": (70, 45, 300, 1, False),
                          "c2_init": (768, 512, 70000, 1, False),
                          "c2_fitted_proxy": (768, 512, 70000, 1, True),
                          "batch3": (130, 70, 900, 3, True)}[cfg]
    gen = synth.fitted_params if fitted else synth.init_params
    ps = np.stack([gen(40 + b, n) for b in range(B)])
    _check_direct_binning(gi, gio, ps, W, H)


def huge_params(seed, n, every=5):
    """The paper's init with every `every`-th Gaussian blown up to sigma 6-40 px
    (boxes of up to ~15 x 15 tiles: single Gaussians with more keys than a
    warp has lanes, several of them per warp) and its colour scaled down."""
    rng = np.random.default_rng(seed)
    p = synth.init_params(seed, n)
    idx = np.arange(0, n, every)
    s = rng.uniform(6.0, 40.0, size=len(idx)).astype(np.float32)
    p[idx, 2] = s - 0.5
    p[idx, 3] = rng.uniform(-0.5, 0.5, size=len(idx)).astype(np.float32) * s
    p[idx, 4] = rng.uniform(0.3, 1.0, size=len(idx)).astype(np.float32) * s - 0.5
    p[idx, 5:8] *= 0.05
    return p


def test_huge_gaussians(gi, gio):
    # > 32-key Gaussians: the flat key emission of post_project_warp (prime and
    # the chained finalize) bit-exact against the oracle's binning, and the
    # finalize's long slot ranges in the gradients, frame and chained step
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 256, 192, 2000
    p = huge_params(11, n)
    r = gio.project(p, W, H)
    tt = np.asarray(r["touched"])
    assert tt.max() > 64 and (tt > 32).sum() > 50
    _check_direct_binning(gi, gio, p[None], W, H)
    tgt = synth.image(11, W, H)
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
    pipe = Pipeline(n, W, H, 1, device=DEV)
    img = pipe.render_frame(to_dev(p)[None].contiguous())[0].cpu().numpy()
    assert np.abs(img - ref_img).max() <= PIX_TOL
    for chained in (True, False):
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), chained=chained)
        fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        errs = group_err(fit.grads[0].cpu().numpy().astype(np.float64), ref_g)
        assert max(errs.values()) <= GRAD_TOL, errs
        assert abs(float(fit.loss[0]) - ref_loss) <= 1e-5 * ref_loss
    # the chained finalize's projection + binning of the updated cloud equals a prime of it
    a = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    for _ in range(3):
        a.step()
    b = Fitter(a.params.clone(), to_dev(tgt)[None].contiguous())
    gi.gi_fit_prime(b.params, b.n, b.f, b.flags, b.cap, b.fit_ws)
    torch.cuda.synchronize()
    ca, la, _ = _bin_state(gi, a)
    cb, lb, _ = _bin_state(gi, b)
    assert np.array_equal(ca, cb)
    assert all((x is None and y is None) or np.array_equal(x, y) for x, y in zip(la, lb))


def test_direct_binning_small_slabs():
    # slabs so small (GI_SLAB_MIN=0, capacity 6 keys per tile) that many tiles
    # overflow: the counts stay exact, in-slab tiles exact, the overflowing
    # ones are counted as streamed; fresh process (the minimum is read once)
    import os
    import subprocess
    import sys
    code = """
import sys, numpy as np, synth
sys.path.insert(0, "tests")
import test_gpu_state as T
from oracle import gio
from paper_2403_08551_b200 import gi
gi.load()
gio.build()
fit, streamed, scap = T._check_direct_binning(gi, gio, synth.fitted_params(9, 3000)[None], 128, 96,
                                              key_capacity=48 * 6)
assert scap == 6 and streamed > 0, (scap, streamed)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GI_SLAB_MIN="0", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_chained_projection_equals_prime(gi):
    # the next step's projection + binning done inside finalize equals a fresh
    # gi_fit_prime of the updated params, record for record and key set for key set
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 200, 150, 5000
    p = synth.init_params(3, n)
    tgt = synth.image(3, W, H)
    a = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    for _ in range(3):
        a.step()
    b = Fitter(a.params.clone(), to_dev(tgt)[None].contiguous())
    gi.gi_fit_prime(b.params, b.n, b.f, b.flags, b.cap, b.fit_ws)
    torch.cuda.synchronize()
    ca, la, _ = _bin_state(gi, a)
    cb, lb, _ = _bin_state(gi, b)
    assert np.array_equal(ca, cb)
    assert all((x is None and y is None) or np.array_equal(x, y) for x, y in zip(la, lb))
    nproj = n * 12                            # 48-B records at the start of fit_ws
    assert torch.equal(a.fit_ws[:nproj], b.fit_ws[:nproj])


# ---------------------------------------------------------------- re-priming
def test_unchain_reprime_matches_fresh(gi):
    # chained steps, params edited, unchain() -> step(): bitwise what a fresh
    # non-chained fitter does from the same params / moments / step counter.
    # Before gi_fit_prime cleared the pending keys, each Gaussian was staged twice.
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 160, 120, 4000
    p = synth.init_params(11, n)
    tgt = to_dev(synth.image(11, W, H))[None].contiguous()
    a = Fitter(to_dev(p)[None].contiguous(), tgt)
    for _ in range(3):
        a.step()
    a.params[..., 5:8] += 0.01               # an external writer of params
    a.unchain()
    b = Fitter(a.params.clone(), tgt, chained=False)
    b.m.copy_(a.m)
    b.v.copy_(a.v)
    b.step_counter.copy_(a.step_counter)
    a.step()
    b.step()
    torch.cuda.synchronize()
    assert a.check() == gi.GI_OK and b.check() == gi.GI_OK
    assert torch.equal(a.loss, b.loss)
    assert torch.equal(a.grads, b.grads)
    assert torch.equal(a.params, b.params)
    assert torch.equal(a.m, b.m) and torch.equal(a.v, b.v)


def test_replaced_buffers_after_steps(gi):
    # Fitter's prepared step call (gi.FitStepCall) follows buffers replaced
    # between steps: new params / moment tensors are the ones stepped
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 160, 120, 4000
    p = synth.init_params(12, n)
    tgt = to_dev(synth.image(12, W, H))[None].contiguous()
    a = Fitter(to_dev(p)[None].contiguous(), tgt)
    for _ in range(2):
        a.step()
    a.params = a.params.clone()
    a.m, a.v = a.m.clone(), a.v.clone()
    a.unchain()
    b = Fitter(a.params.clone(), tgt, chained=False)
    b.m.copy_(a.m)
    b.v.copy_(a.v)
    b.step_counter.copy_(a.step_counter)
    a.step()
    b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.params, b.params) and torch.equal(a.m, b.m) and torch.equal(a.v, b.v)


def test_non_chained_and_render_after_chained(gi):
    # gi_fit_step (non-chained) clears the pending keys itself; gi_render_frame
    # on that workspace needs gi_fit_reset first (documented in gi.h)
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 128, 96, 2500
    p = synth.init_params(12, n)
    tgt = to_dev(synth.image(12, W, H))[None].contiguous()
    a = Fitter(to_dev(p)[None].contiguous(), tgt)
    for _ in range(2):
        a.step()
    b = Fitter(a.params.clone(), tgt, chained=False)
    b.m.copy_(a.m)
    b.v.copy_(a.v)
    b.step_counter.copy_(a.step_counter)
    gi.gi_fit_step(a.params, a.grads, a.m, a.v, a.target, a.n, a.f, a.flags, a.cap, a.fit_ws,
                   a.step_counter, loss=a.loss, status_flags=a.status, **a.hyper)
    b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.params, b.params) and torch.equal(a.grads, b.grads)
    # chained again, then reset -> render_frame on the same workspace
    c = Fitter(to_dev(p)[None].contiguous(), tgt)
    c.step()
    gi.gi_fit_reset(c.n, c.f, c.cap, c.fit_ws)
    img = torch.zeros(1, 3, H, W, dtype=torch.float32, device=DEV)
    gi.gi_render_frame(c.params, c.n, c.f, c.flags, c.cap, c.fit_ws, img)
    ref = Pipeline(n, W, H, 1, device=DEV).render_frame(c.params).clone()
    torch.cuda.synchronize()
    assert torch.equal(img, ref)


# ---------------------------------------------------------------- fused Adam
def test_fused_adam_is_adam_step(gi, gio):
    # p, m, v of every fused step (t = 1..5, and across the lr halving at
    # 20001) are bitwise gi_adam_step applied to that step's gradients
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 128, 96, 3000
    p = synth.init_params(21, n)
    tgt = to_dev(synth.image(21, W, H))[None].contiguous()
    for start, chained in ((0, True), (19998, False), (19998, True)):
        fit = Fitter(to_dev(p)[None].contiguous(), tgt, chained=chained)
        rng = np.random.default_rng(start)
        if start:
            fit.m.copy_(to_dev((rng.normal(size=(1, n, 8)) * 1e-3).astype(np.float32)))
            fit.v.copy_(to_dev((rng.uniform(size=(1, n, 8)) * 1e-5).astype(np.float32)))
            fit.step_counter.fill_(start)
        for t in range(start + 1, start + 6):
            p0, m0, v0 = fit.params.clone(), fit.m.clone(), fit.v.clone()
            fit.step()
            lr = gi.gi_lr_at(t, 1e-3, 20000)
            gi.gi_adam_step(p0, fit.grads, m0, v0, p0.numel(), t, lr, 0.9, 0.999, 1e-8)
            torch.cuda.synchronize()
            assert fit.steps_done() == t
            assert torch.equal(fit.params, p0), t
            assert torch.equal(fit.m, m0) and torch.equal(fit.v, v0), t


@pytest.mark.parametrize("step", [1, 2, 3, 4, 5, 20001])
def test_adam_step_nonzero_state_vs_oracle(gi, gio, step):
    # c.4: updated p, m, v within 1e-6 relative elementwise (floor 1e-12),
    # from shared non-zero state.  Relative to the terms each result sums
    # (reading R34): m = b1 m + (1 - b1) g can cancel to ~0, and fp32 then
    # owes 1e-6 of |b1 m| + |(1 - b1) g|, not of the cancelled sum
    rng = np.random.default_rng(100 + step)
    n = 8 * 1024 + 5
    p = rng.normal(size=n).astype(np.float32)
    g = (rng.normal(size=n) * 10.0 ** rng.uniform(-5, 0, size=n)).astype(np.float32)
    m = (rng.normal(size=n) * 1e-2).astype(np.float32)
    v = (rng.uniform(size=n) * 1e-3).astype(np.float32)
    lr = gio.lr_at(step)
    pt, mt, vt = to_dev(p), to_dev(m), to_dev(v)
    gi.gi_adam_step(pt, to_dev(g), mt, vt, n, step, lr)
    po, mo, vo = gio.adam(p, g, m, v, step, lr)
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    gd = g.astype(np.float64)
    scale = {"p": np.abs(p) + np.abs(po - p), "m": np.abs(b1 * m) + np.abs((1 - b1) * gd),
             "v": np.abs(b2 * v) + (1 - b2) * gd * gd}
    for name, got, ref in (("p", pt, po), ("m", mt, mo), ("v", vt, vo)):
        got = got.cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= 1e-6 * scale[name] + 1e-12), name


# ---------------------------------------------------------------- clustered cloud
def test_clustered_cloud(gi, gio):
    # half of 30k Gaussians in 4 discs of 6 px: tiles of up to ~4,100 keys,
    # past the 1,024-key slab (streamed) and every sort buffer -- parity and
    # bitwise chained == plain hold on the slow paths too
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 256, 192, 30000
    p = synth.clustered_params(3, n, W, H, clusters=4, frac=0.5, radius_px=6.0)
    tgt = synth.image(3, W, H)
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
    kt, kg, rng = gio.bin(p, W, H)
    assert np.diff(rng.astype(np.int64)).max() > 1024
    pipe = Pipeline(n, W, H, 1, device=DEV)
    pipe.render(to_dev(p)[None].contiguous())
    torch.cuda.synchronize()
    K = len(kt)
    assert pipe.keys() == K
    assert np.array_equal(pipe.key_gid[:K].cpu().numpy().view(np.uint32), kg)
    scale = np.maximum(1.0, np.abs(ref_img))           # R26: sums far above 1
    assert np.all(np.abs(pipe.image[0].cpu().numpy() - ref_img) <= PIX_TOL * scale)
    img = Pipeline(n, W, H, 1, device=DEV).render_frame(to_dev(p)[None].contiguous())
    assert np.all(np.abs(img[0].cpu().numpy() - ref_img) <= PIX_TOL * scale)
    outs = []
    for chained in (True, False):
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), chained=chained)
        fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        streamed, _ = fit.seg_stats()
        assert streamed > 0
        errs = group_err(fit.grads[0].cpu().numpy().astype(np.float64), ref_g)
        assert max(errs.values()) <= GRAD_TOL, errs
        assert abs(float(fit.loss[0]) - ref_loss) <= 1e-5 * ref_loss
        for _ in range(2):
            fit.step()
        torch.cuda.synchronize()
        outs.append((fit.params.clone(), fit.loss.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_nonfinite_colour_propagates(gi):
    # a NaN colour must not vanish in the fixed-point forward: the pixels of
    # that Gaussian's tiles come out NaN (as an fp32 sum would), and a fit
    # step raises the non-finite status
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 64, 64, 256
    p = synth.init_params(4, n)
    p[7, 5] = np.nan
    img = Pipeline(n, W, H, 1, device=DEV).render_frame(to_dev(p)[None].contiguous())
    torch.cuda.synchronize()
    assert torch.isnan(img).any()
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(synth.image(4, W, H))[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_ENONFINITE


@pytest.mark.parametrize("optimizer", ["adam", "adan"])
def test_fit_trajectory_band(gi, gio, optimizer):
    # SURVEY c.3: long fitting trajectories are chaotic in fp32 vs fp64, so
    # they are pinned by a band: C1 (64x64, 256 Gaussians, the paper's init),
    # 2000 steps of the paper's loop on the GPU (chained fused steps) and in
    # the oracle (fp64 steps, state rounded to fp32 between steps, as stored);
    # final PSNR within 0.1 dB, and both fits far above the start
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n, steps = 64, 64, 256, 2000
    p0 = synth.init_params(0, n)
    tgt = synth.image(0, W, H)
    fit = Fitter(to_dev(p0)[None].contiguous(), to_dev(tgt)[None].contiguous(), optimizer=optimizer)
    fit.capture(100)
    for _ in range(steps // 100):
        fit.replay()
    pipe = Pipeline(n, W, H, 1, device=DEV)
    img = pipe.render_frame(fit.params)
    gpu_psnr = float(pipe.psnr(img, to_dev(tgt)[None].contiguous())[0])
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK and fit.steps_done() == steps
    p = p0.copy()
    z = np.zeros_like(p)
    st = dict(m=z.copy(), v=z.copy(), n=z.copy(), gp=z.copy())
    for t in range(1, steps + 1):
        _, _, g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
        g = g.astype(np.float32)
        if optimizer == "adam":
            po, mo, vo = gio.adam(p, g, st["m"], st["v"], t, gio.lr_at(t))
            st.update(m=mo.astype(np.float32), v=vo.astype(np.float32))
        else:
            po, mo, vo, no = gio.adan(p, g, st["m"], st["v"], st["n"], st["gp"], t, gio.lr_at(t))
            st.update(m=mo.astype(np.float32), v=vo.astype(np.float32), n=no.astype(np.float32),
                      gp=g)
        p = po.astype(np.float32)
    ref_psnr = gio.psnr(gio.render(p, W, H, mode=gio.ALL_PAIRS), tgt)
    start = gio.psnr(gio.render(p0, W, H, mode=gio.ALL_PAIRS), tgt)
    assert ref_psnr > start + 5.0 and gpu_psnr > start + 5.0, (start, ref_psnr, gpu_psnr)
    assert abs(gpu_psnr - ref_psnr) <= 0.1, (gpu_psnr, ref_psnr)


# ---------------------------------------------------------------- checkpoint / log
@pytest.mark.parametrize("optimizer", ["adam", "adan"])
def test_checkpoint_resume_bitwise(gi, tmp_path, optimizer):
    # save after 15 steps, resume in a new Fitter, 15 more: bitwise the 30-step fit
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 160, 120, 3000
    p = to_dev(synth.init_params(21, n))[None].contiguous()
    tgt = to_dev(synth.image(21, W, H))[None].contiguous()
    a = Fitter(p.clone(), tgt, optimizer=optimizer)
    for _ in range(30):
        a.step()
    b = Fitter(p.clone(), tgt, optimizer=optimizer)
    for _ in range(15):
        b.step()
    path = str(tmp_path / "ckpt.npz")
    b.save(path)
    c = Fitter.load(path, tgt)
    assert c.optimizer == optimizer and c.steps_done() == 15
    for _ in range(15):
        c.step()
    torch.cuda.synchronize()
    assert c.check() == gi.GI_OK
    assert torch.equal(a.params, c.params) and torch.equal(a.m, c.m) and torch.equal(a.v, c.v)
    assert torch.equal(a.step_counter, c.step_counter)
    if optimizer == "adan":
        assert torch.equal(a.n_acc, c.n_acc) and torch.equal(a.grad_prev, c.grad_prev)


def test_fit_loop_jsonl_log(gi, tmp_path):
    # Fitter.fit: graph replays of log_every steps, a JSON line per log point
    # (step, loss, PSNR, it/s); the same params as stepping eagerly
    import json
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 160, 120, 3000
    p = to_dev(synth.init_params(22, n))[None].contiguous()
    tgt = to_dev(synth.image(22, W, H))[None].contiguous()
    a = Fitter(p.clone(), tgt)
    log = tmp_path / "fit.jsonl"
    rec = a.fit(250, log_every=100, log=str(log))
    lines = [json.loads(x) for x in log.read_text().splitlines()]
    assert [r["step"] for r in lines] == [100, 200, 250] == [r["step"] for r in rec]
    assert lines[0]["loss"][0] > lines[-1]["loss"][0] > 0
    assert lines[-1]["psnr_db"][0] > lines[0]["psnr_db"][0]
    assert all(r["it_per_s"] > 0 for r in lines)
    b = Fitter(p.clone(), tgt)
    for _ in range(250):
        b.step()
    torch.cuda.synchronize()
    assert torch.equal(a.params, b.params) and torch.equal(a.m, b.m)


def test_streamed_8bit_target_fit(gi):
    # the bench's e2e loop: each step's target uploaded as 8-bit RGB on a copy
    # stream (gi_target_upload_rgb8), expanded on the compute stream
    # (gi_target_from_rgb8), then the chained step -- bitwise a plain fit on
    # the same (8-bit rounded) target
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 160, 120, 3000
    p = to_dev(synth.init_params(23, n))[None].contiguous()
    t = synth.image(23, W, H)
    t8 = np.ascontiguousarray(np.clip(np.rint(t * 255.0), 0, 255).astype(np.uint8).transpose(1, 2, 0))
    tq = to_dev((t8.astype(np.float32) / np.float32(255)).transpose(2, 0, 1))[None].contiguous()
    ref = Fitter(p.clone(), tq.clone())
    for _ in range(6):
        ref.step()
    host = torch.from_numpy(t8).pin_memory()
    stage = [torch.empty(t8.shape, dtype=torch.uint8, device=DEV) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    stream = torch.cuda.current_stream()
    for e in ready + free:
        e.record(stream)
    tbuf = torch.zeros_like(tq)
    a = Fitter(p.clone(), tbuf)
    cs = torch.cuda.Stream()
    cs.wait_stream(stream)
    gi.gi_target_upload_rgb8(host, stage[0], a.f, None, ready[0], cs)
    for i in range(6):
        b = i & 1
        if i + 1 < 6:
            gi.gi_target_upload_rgb8(host, stage[b ^ 1], a.f, free[b ^ 1] if i >= 1 else None,
                                     ready[b ^ 1], cs)
        gi.gi_target_from_rgb8(stage[b], a.f, tbuf, ready[b], free[b], stream)
        a.step()
    stream.wait_stream(cs)
    torch.cuda.synchronize()
    assert torch.equal(tbuf, tq)
    assert torch.equal(a.params, ref.params) and torch.equal(a.m, ref.m) and torch.equal(a.v, ref.v)
