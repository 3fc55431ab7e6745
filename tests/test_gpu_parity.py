"""CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Bars (north_star):
  * keys, ranges, offsets, tile counts, boxes, decode: bit-exact
  * pixels: max |gpu - oracle| <= 2e-5 on unclamped output
  * gradients: ||g_gpu - g_ref|| / ||g_ref|| <= 1e-4 per group (mu, l, c')
  * Adam: elementwise, tolerance derived from fp32 rounding of each term
Configs: C1 64x64/256 (all-pairs oracle), ragged frames, C2 768x512/70k at the
paper's init and at the 3x "fitted" proxy (tiled oracle, full frame), C3
2040x1356/100k (full frame), batches of images per launch.
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

CASES = {
    "c1": (64, 64, 256, 0, False),
    "ragged": (70, 45, 300, 1, False),
    "tiny": (5, 3, 4, 2, False),
    "c1_fitted": (64, 64, 256, 3, True),
    "c2_init": (768, 512, 70000, 1, False),
    "c2_fitted": (768, 512, 70000, 1, True),
}


def params_for(n, seed, fitted):
    return synth.fitted_params(seed, n) if fitted else synth.init_params(seed, n)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def run_gpu(gi, params_b, W, H, flags=0, target_b=None, dL=None):
    from paper_2403_08551_b200.pipeline import Pipeline
    B, n = params_b.shape[0], params_b.shape[1]
    pipe = Pipeline(n, W, H, B, device=DEV)
    p = to_dev(params_b)
    pipe.render(p, flags)
    img = pipe.image.clone()
    out = dict(pipe=pipe, image=img.cpu().numpy())
    if target_b is not None or dL is not None:
        pipe.backward(p, target=None if target_b is None else to_dev(target_b),
                      dL_dimage=None if dL is None else to_dev(dL), flags=flags)
        out["grads"] = pipe.grads.cpu().numpy().astype(np.float64)
        out["loss"] = pipe.loss.cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    assert pipe.check() == gi.GI_OK
    return out


def group_err(g, ref):
    errs = {}
    for name, cols in GROUPS.items():
        den = np.linalg.norm(ref[..., cols])
        errs[name] = np.linalg.norm(g[..., cols] - ref[..., cols]) / max(den, 1e-300)
    return errs


@pytest.fixture(scope="module", params=list(CASES))
def case(request, gio):
    W, H, n, seed, fitted = CASES[request.param]
    p = params_for(n, seed, fitted)
    tgt = synth.image(seed, W, H)
    mode = gio.ALL_PAIRS if W * H * n <= 64 * 64 * 300 else gio.TILED
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=mode)
    return dict(name=request.param, W=W, H=H, n=n, p=p, tgt=tgt, ref_img=ref_img,
                ref_loss=ref_loss, ref_g=ref_g)


def test_project_and_bin_bitexact(gi, gio, case):
    W, H, p = case["W"], case["H"], case["p"]
    out = run_gpu(gi, p[None], W, H)
    pipe = out["pipe"]
    pr = gio.project(p, W, H)
    touched = u32(pipe.tiles_touched)[: case["n"]]
    assert np.array_equal(touched, pr["touched"])
    rec = pipe.proj.view(-1, 12).cpu().numpy()
    bx = rec[:, 7].view(np.uint32)
    by = rec[:, 11].view(np.uint32)
    valid = pr["touched"] > 0
    box = np.stack([bx & 0xffff, bx >> 16, by & 0xffff, by >> 16], 1).astype(np.int32)
    assert np.array_equal(box[valid], pr["box"][valid])
    # split centre reproduces the fp64 centre to fp32 rounding of the fraction
    ix = rec[:, 0].view(np.int32).astype(np.float64)
    iy = rec[:, 1].view(np.int32).astype(np.float64)
    assert np.abs(ix + rec[:, 2] - pr["mu"][:, 0]).max() < 1e-6
    assert np.abs(iy + rec[:, 3] - pr["mu"][:, 1]).max() < 1e-6
    kt, kg, rng = gio.bin(p, W, H)
    K = len(kt)
    assert pipe.keys() == K
    assert np.array_equal(u32(pipe.key_tile)[:K], kt)
    assert np.array_equal(u32(pipe.key_gid)[:K], kg)
    assert np.array_equal(u32(pipe.tile_range)[: len(rng)], rng)


def test_render_parity(gi, gio, case):
    out = run_gpu(gi, case["p"][None], case["W"], case["H"])
    err = np.abs(out["image"][0] - case["ref_img"]).max()
    assert err <= PIX_TOL, err


def test_render_frame_fused_parity(gi, gio, case):
    # fused path: counts in projection, ordering inside the render kernel
    from paper_2403_08551_b200.pipeline import Pipeline
    pipe = Pipeline(case["n"], case["W"], case["H"], 1, device=DEV)
    img = pipe.render_frame(to_dev(case["p"][None]))
    torch.cuda.synchronize()
    assert np.abs(img[0].cpu().numpy() - case["ref_img"]).max() <= PIX_TOL
    kt, _, _ = gio.bin(case["p"], case["W"], case["H"])
    assert pipe.frame_keys() == len(kt)


def test_loss_and_backward_parity(gi, gio, case):
    out = run_gpu(gi, case["p"][None], case["W"], case["H"], target_b=case["tgt"][None])
    errs = group_err(out["grads"][0], case["ref_g"])
    assert max(errs.values()) <= GRAD_TOL, errs
    assert abs(out["loss"][0] - case["ref_loss"]) <= 1e-5 * max(case["ref_loss"], 1e-3)


def test_backward_explicit_upstream(gi, gio):
    W, H, n = 70, 45, 300
    p = synth.init_params(4, n)
    rng = np.random.default_rng(4)
    dL = rng.normal(size=(3, H, W)).astype(np.float32)
    ref = gio.backward(p, dL.astype(np.float64), W, H)
    out = run_gpu(gi, p[None], W, H, dL=dL[None])
    errs = group_err(out["grads"][0], ref)
    assert max(errs.values()) <= GRAD_TOL, errs


def test_normalized_positions(gi, gio):
    # decode path: params[0:2] already in (-1, 1) (GI_POS_NORMALIZED)
    W, H, n = 96, 80, 400
    p = synth.init_params(5, n)
    p[:, :2] = np.tanh(p[:, :2].astype(np.float64)).astype(np.float32)
    tgt = synth.image(5, W, H)
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, pos_mode=gio.POS_NORMALIZED,
                                                  mode=gio.ALL_PAIRS)
    out = run_gpu(gi, p[None], W, H, flags=gi.GI_POS_NORMALIZED, target_b=tgt[None])
    assert np.abs(out["image"][0] - ref_img).max() <= PIX_TOL
    errs = group_err(out["grads"][0], ref_g)
    assert max(errs.values()) <= GRAD_TOL, errs


def test_batched_launch(gi, gio):
    # B images per launch: tile ids img*T + t, gids img*N + n
    W, H, n, B = 100, 60, 500, 3
    pb = np.stack([synth.init_params(10 + b, n) for b in range(B)])
    tb = np.stack([synth.image(10 + b, W, H) for b in range(B)])
    out = run_gpu(gi, pb, W, H, target_b=tb)
    pipe = out["pipe"]
    T = gio.n_tiles(W, H)
    kts, kgs = [], []
    for b in range(B):
        img, loss, g = gio.loss_and_grads(pb[b], tb[b], mode=gio.ALL_PAIRS)
        assert np.abs(out["image"][b] - img).max() <= PIX_TOL
        assert max(group_err(out["grads"][b], g).values()) <= GRAD_TOL
        assert abs(out["loss"][b] - loss) <= 1e-5 * max(loss, 1e-3)
        kt, kg, _ = gio.bin(pb[b], W, H)
        kts.append(kt + b * T)
        kgs.append(kg + b * n)
    kt, kg = np.concatenate(kts), np.concatenate(kgs)
    assert pipe.keys() == len(kt)
    assert np.array_equal(u32(pipe.key_tile)[: len(kt)], kt)
    assert np.array_equal(u32(pipe.key_gid)[: len(kg)], kg)


@pytest.mark.parametrize("n", [3000, 9000])
def test_long_segments(gi, gio, n):
    # segments of ~1.3k keys (bitonic path) and > 2048 keys (in-order rebuild
    # path), through gi_bin, the fused render and the fused fit step
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H = 48, 48
    p = synth.fitted_params(20 + n, n)
    tgt = synth.image(20, W, H)
    kt, kg, rng = gio.bin(p, W, H)
    assert np.diff(rng).max() > (2048 if n == 9000 else 256)
    out = run_gpu(gi, p[None], W, H, target_b=tgt[None])
    pipe = out["pipe"]
    assert np.array_equal(u32(pipe.key_gid)[: len(kg)], kg)
    assert np.array_equal(u32(pipe.tile_range)[: len(rng)], rng)
    img, loss, g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
    # ~3500 overlapping terms per pixel push C to ~6: the 2e-5 bar is stated
    # on a [0, 1] scale (north_star), so it is applied to C / max(1, max|C|)
    tol = PIX_TOL * max(1.0, float(np.abs(img).max()))
    assert np.abs(out["image"][0] - img).max() <= tol
    assert max(group_err(out["grads"][0], g).values()) <= GRAD_TOL
    fimg = pipe.render_frame(to_dev(p[None]))
    assert np.abs(fimg[0].cpu().numpy() - img).max() <= tol
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert abs(float(fit.loss[0]) - loss) <= 1e-5 * loss
    assert max(group_err(fit.grads[0].cpu().numpy().astype(np.float64), g).values()) <= GRAD_TOL


def test_c3_render_sampled(gi, gio):
    # C3 (DIV2K-shaped 2040x1356, 100k) full frame, in the bench launch shape
    W, H, n = 2040, 1356, 100000
    p = synth.init_params(2, n)
    out = run_gpu(gi, p[None], W, H)
    ref = gio.render(p, W, H, mode=gio.TILED)
    assert np.abs(out["image"][0] - ref).max() <= PIX_TOL
    kt, kg, rng = gio.bin(p, W, H)
    assert out["pipe"].keys() == len(kt)
    assert np.array_equal(u32(out["pipe"].key_gid)[: len(kg)], kg)


def test_edge_cases(gi, gio):
    from paper_2403_08551_b200.pipeline import Pipeline
    # all Gaussians culled (l1 + 1/2 == 0): empty lists, zero image, zero grads
    p = synth.init_params(6, 50)
    p[:, 2] = -0.5
    out = run_gpu(gi, p[None], 40, 30, target_b=synth.image(6, 40, 30)[None])
    assert out["pipe"].keys() == 0
    assert not out["image"].any() and not out["grads"].any()
    # one huge Gaussian covering every tile of a ragged frame
    p = np.array([[0.0, 0.0, 200.0, 5.0, 150.0, 0.5, -0.25, 1.0]], np.float32)
    tgt = synth.image(7, 100, 37)
    ref_img, _, ref_g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    out = run_gpu(gi, p[None], 100, 37, target_b=tgt[None])
    assert out["pipe"].keys() == gio.n_tiles(100, 37)
    assert np.abs(out["image"][0] - ref_img).max() <= PIX_TOL
    assert max(group_err(out["grads"][0], ref_g).values()) <= GRAD_TOL
    # 1x1 frame
    p = synth.init_params(8, 3)
    ref = gio.render(p, 1, 1)
    out = run_gpu(gi, p[None], 1, 1)
    assert np.abs(out["image"][0] - ref).max() <= PIX_TOL
    # n = 0
    pipe = Pipeline(0, 32, 32, 1, device=DEV)
    pipe.render(torch.zeros(1, 1, 8, device=DEV))
    torch.cuda.synchronize()
    assert pipe.keys() == 0 and not pipe.image.any()
    # capacity overflow is reported, not a crash
    p = synth.fitted_params(9, 2000)
    pipe = Pipeline(2000, 128, 128, 1, key_capacity=64, device=DEV)
    pipe.render(to_dev(p))
    assert pipe.check() == gi.GI_ECAPACITY


def fuzz_params(rng, n):
    """Seeded mix of the paper's init, the 3x fitted proxy and degenerate
    Gaussians: culled (l1 or l3 + 1/2 == 0), negative diagonals, centres at
    the border, huge boxes, negative colours."""
    p = synth.init_params(int(rng.integers(1 << 30)), n) if rng.random() < 0.5 else \
        synth.fitted_params(int(rng.integers(1 << 30)), n)
    k = rng.random(n)
    p[k < 0.05, 2] = -0.5
    p[(k >= 0.05) & (k < 0.1), 4] = -0.5
    # signed (negative) diagonals, any off-diagonal: near-singular and
    # near-line Gaussians included (|l_ii + 1/2| down to 0, |l2| up to 3)
    neg = (k >= 0.1) & (k < 0.2)
    m = int(neg.sum())
    p[neg, 2] = -rng.uniform(0.0, 3.0, size=m)
    p[neg, 3] = rng.uniform(-3.0, 3.0, size=m)
    p[neg, 4] = -rng.uniform(0.0, 3.0, size=m)
    edge = (k >= 0.2) & (k < 0.3)
    p[edge, 0:2] = rng.choice([-4.0, 4.0], size=(int(edge.sum()), 2)) * rng.uniform(0.5, 1.0, size=(int(edge.sum()), 2))
    huge = (k >= 0.3) & (k < 0.32)
    p[huge, 2] = rng.uniform(10, 60, size=int(huge.sum()))
    p[huge, 4] = rng.uniform(10, 60, size=int(huge.sum()))
    p[(k >= 0.32) & (k < 0.4), 5:8] *= -1.0
    return p.astype(np.float32)


def pix_ok(img, ref):
    """The 2e-5 bar is stated on the [0, 1] scale; random clouds can sum to
    pixel values of ~10, where fp32 accumulation alone moves the sum by a few
    ulp of the value, so the fuzz cases scale the bar by max(1, |ref|)."""
    return np.all(np.abs(img - ref) <= PIX_TOL * np.maximum(1.0, np.abs(ref)))


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_small_frames(gi, gio, seed):
    # random frames (ragged, tiny, wider than tall), cloud sizes and
    # degenerate Gaussians: keys bit-exact, fused frame and fused fit step
    # gradients vs the oracle (no memory checker on this pool: parity on many
    # small random cases is the bounds check)
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(1, 200)), int(rng.integers(1, 150))
    n = int(rng.integers(1, 1500))
    p = fuzz_params(rng, n)
    tgt = synth.image(seed, W, H)
    pipe = run_gpu(gi, p[None], W, H)["pipe"]
    kt, kg, _ = gio.bin(p, W, H)
    K = len(kt)
    assert pipe.keys() == K
    assert np.array_equal(u32(pipe.key_tile)[:K], kt)
    assert np.array_equal(u32(pipe.key_gid)[:K], kg)
    mode = gio.ALL_PAIRS if W * H * n <= 20_000_000 else gio.TILED
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=mode)
    fp = Pipeline(n, W, H, 1, device=DEV)
    img = fp.render_frame(to_dev(p)[None].contiguous())
    torch.cuda.synchronize()
    assert pix_ok(img[0].cpu().numpy(), ref_img)
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    assert abs(float(fit.loss[0]) - ref_loss) <= 1e-5 * max(ref_loss, 1e-12)
    gg = fit.grads[0].cpu().numpy().astype(np.float64)
    for name, cols in GROUPS.items():
        den = np.linalg.norm(ref_g[:, cols])
        num = np.linalg.norm(gg[:, cols] - ref_g[:, cols])
        assert num <= GRAD_TOL * den + 1e-12, (name, num, den)
    assert np.all(np.isfinite(fit.params.cpu().numpy()))


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_batched(gi, gio, seed):
    # 2-4 different random images per launch: each image's frame and fused
    # fit-step gradients vs the oracle run on that image alone
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    rng = np.random.default_rng(2000 + seed)
    B = int(rng.integers(2, 5))
    W, H = int(rng.integers(8, 160)), int(rng.integers(8, 120))
    n = int(rng.integers(1, 800))
    ps = np.stack([fuzz_params(rng, n) for _ in range(B)])
    ts = np.stack([synth.image(50 + 7 * seed + b, W, H) for b in range(B)])
    fp = Pipeline(n, W, H, B, device=DEV)
    img = fp.render_frame(to_dev(ps).contiguous()).cpu().numpy()
    fit = Fitter(to_dev(ps).contiguous(), to_dev(ts).contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    gg = fit.grads.cpu().numpy().astype(np.float64)
    for b in range(B):
        ref_img, ref_loss, ref_g = gio.loss_and_grads(ps[b], ts[b], mode=gio.ALL_PAIRS)
        assert pix_ok(img[b], ref_img)
        assert abs(float(fit.loss[b]) - ref_loss) <= 1e-5 * ref_loss
        for name, cols in GROUPS.items():
            den = np.linalg.norm(ref_g[:, cols])
            assert np.linalg.norm(gg[b][:, cols] - ref_g[:, cols]) <= GRAD_TOL * den + 1e-12, name


def test_adam_parity(gi, gio):
    rng = np.random.default_rng(12)
    n = 4096 + 3                               # float4 body + scalar tail
    p = rng.normal(size=n).astype(np.float32)
    g = (rng.normal(size=n) * 10.0 ** rng.uniform(-6, 1, size=n)).astype(np.float32)
    m = (rng.normal(size=n) * 0.01).astype(np.float32)
    v = (rng.uniform(0, 1, size=n) * 1e-3).astype(np.float32)
    for step, lr in [(1, 1e-3), (7, 1e-3), (20001, 5e-4)]:
        pt, gt, mt, vt = to_dev(p), to_dev(g), to_dev(m), to_dev(v)
        flag = torch.zeros(1, dtype=torch.int32, device=DEV)
        gi.gi_adam_step(pt, gt, mt, vt, n, step, lr, nonfinite_flag=flag)
        po, mo, vo = gio.adam(p, g, m, v, step, lr)
        b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
        gd = g.astype(np.float64)
        tol_m = 1e-6 * (np.abs(b1 * m) + np.abs((1 - b1) * gd)) + 1e-12
        tol_v = 1e-6 * (np.abs(b2 * v) + np.abs((1 - b2) * gd * gd)) + 1e-12
        upd = np.abs(po - p.astype(np.float64))
        tol_p = 1e-6 * (np.abs(p) + upd) + 1e-12
        assert np.all(np.abs(mt.cpu().numpy() - mo) <= tol_m)
        assert np.all(np.abs(vt.cpu().numpy() - vo) <= tol_v)
        assert np.all(np.abs(pt.cpu().numpy() - po) <= tol_p)
        assert int(flag.item()) == 0
    # non-finite detection
    pt = to_dev(p); gt = to_dev(np.full(n, np.nan, np.float32))
    flag = torch.zeros(1, dtype=torch.int32, device=DEV)
    gi.gi_adam_step(pt, gt, to_dev(m), to_dev(v), n, 1, 1e-3, nonfinite_flag=flag)
    assert gi.gi_check(None, 0, flag) == gi.GI_ENONFINITE


@pytest.mark.parametrize("bits,n", [(6, 70000), (8, 1001), (6, 1)])
def test_vq_decode_bitexact(gi, gio, bits, n):
    data, gamma, beta, books = synth.payload(bits, n, bits=bits)
    ref = gio.vq_decode(data, n, gamma, beta, books, bits=bits)
    out = torch.zeros(n, 8, dtype=torch.float32, device=DEV)
    bk = to_dev(books)
    meta = gi.codec_meta(n, gamma, beta, bk, bits=bits)
    gi.gi_vq_decode(to_dev(data), meta, out)
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_decode_then_render(gi, gio):
    # C5 path: payload -> decode -> project(GI_POS_NORMALIZED) -> bin -> render
    from paper_2403_08551_b200.pipeline import Pipeline
    n, W, H = 4500, 768, 512
    data, gamma, beta, books = synth.payload(3, n)
    ref_p = gio.vq_decode(data, n, gamma, beta, books)
    ref = gio.render(ref_p, W, H, pos_mode=gio.POS_NORMALIZED, mode=gio.TILED)
    params = torch.zeros(1, n, 8, dtype=torch.float32, device=DEV)
    bk = to_dev(books)                      # keep alive: the meta holds the raw pointer
    gi.gi_vq_decode(to_dev(data), gi.codec_meta(n, gamma, beta, bk), params)
    pipe = Pipeline(n, W, H, 1, device=DEV)
    img = pipe.render(params, gi.GI_POS_NORMALIZED)
    assert np.abs(img[0].cpu().numpy() - ref).max() <= PIX_TOL


@pytest.mark.parametrize("n", [4500, 70000])
def test_decode_render_frame_fused(gi, gio, n):
    # configs[4] in two kernels (decode fused into the projection): image and
    # decoded params bitwise those of gi_vq_decode -> gi_render_frame, and the
    # image within the pixel bar of the oracle's decode -> render
    from paper_2403_08551_b200.pipeline import Pipeline
    W, H = 768, 512
    data, gamma, beta, books = synth.payload(4, n)
    bk = to_dev(books)
    meta = gi.codec_meta(n, gamma, beta, bk)
    pay = to_dev(data)
    p_ref = torch.zeros(1, n, 8, dtype=torch.float32, device=DEV)
    gi.gi_vq_decode(pay, meta, p_ref)
    a = Pipeline(n, W, H, 1, device=DEV)
    img_ref = a.render_frame(p_ref, gi.GI_POS_NORMALIZED).clone()
    b = Pipeline(n, W, H, 1, device=DEV)
    p_out = torch.full((1, n, 8), float("nan"), dtype=torch.float32, device=DEV)
    for _ in range(2):                      # counters left zeroed for the next frame
        img = b.decode_render_frame(pay, meta, p_out).clone()
        torch.cuda.synchronize()
        assert torch.equal(img, img_ref)
        assert torch.equal(p_out, p_ref)
    b.decode_render_frame(pay, meta)        # params output is optional
    torch.cuda.synchronize()
    assert torch.equal(b.image, img_ref)
    assert b.frame_keys() == a.frame_keys()
    if n <= 4500:
        ref_p = gio.vq_decode(data, n, gamma, beta, books)
        ref = gio.render(ref_p, W, H, pos_mode=gio.POS_NORMALIZED, mode=gio.TILED)
        assert np.abs(img[0].cpu().numpy() - ref).max() <= PIX_TOL
    with pytest.raises(RuntimeError):       # one image per payload
        bad = Pipeline(n, W, H, 2, device=DEV)
        bad.decode_render_frame(pay, meta)


def test_fit_step_matches_oracle(gi, gio):
    # one fused device step (project, bin, fwd+L2+bwd, Adam) from a fresh state
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 64, 64, 256
    p = synth.init_params(0, n)
    tgt = synth.image(0, W, H)
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK and fit.steps_done() == 1
    img, loss, g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    assert abs(float(fit.loss[0]) - loss) <= 1e-5 * loss
    gg = fit.grads[0].cpu().numpy().astype(np.float64)
    assert max(group_err(gg, g).values()) <= GRAD_TOL
    # Adam step 1 from zero state, on the oracle's gradients: p - lr g/(|g|+eps);
    # compare where the oracle gradient is well above the gradient error
    z = np.zeros_like(p)
    po, _, _ = gio.adam(p, g.astype(np.float32), z, z, 1, 1e-3)
    got = fit.params[0].cpu().numpy().astype(np.float64)
    big = np.abs(g) > 1e-3 * np.sqrt(np.mean(g ** 2, axis=0, keepdims=True))
    assert big.mean() > 0.9
    assert np.all(np.abs(got - po)[big] <= 1e-6 * np.abs(po)[big] + 1e-9)


def test_fit_graph_loss_decreases(gi):
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 128, 96, 2000
    p = synth.init_params(1, n)
    tgt = synth.image(1, W, H)
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    l0 = float(fit.loss[0])
    fit.capture(10)
    for _ in range(30):
        fit.replay()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    assert fit.steps_done() == 1 + 300        # capture records, it does not execute
    assert float(fit.loss[0]) < 0.5 * l0


def test_determinism_and_counter_reuse(gi):
    # the fused paths leave their per-tile counters zeroed for the next call;
    # repeated frames and two identical fits must agree bit for bit (no
    # atomics on values, fixed reduction orders)
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 256, 192, 8000
    p = synth.init_params(31, n)
    tgt = synth.image(31, W, H)
    pipe = Pipeline(n, W, H, 1, device=DEV)
    a = pipe.render_frame(to_dev(p[None])).clone()
    b = pipe.render_frame(to_dev(p[None])).clone()
    assert torch.equal(a, b)
    outs = []
    for chained in (True, False):     # the chained path must equal the plain one bitwise
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), chained=chained)
        for _ in range(5):
            fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        outs.append((fit.params.clone(), fit.loss.clone(), fit.grads.clone()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][2], outs[1][2])


def test_adan_parity(gi, gio):
    # NEXT-1: elementwise Adan vs the fp64 oracle over three steps (the
    # gradient-difference term is live from step 2).  Every step starts both
    # sides from the same state -- the oracle's, rounded to fp32 as it is
    # stored, copied to the GPU (c.4 "one step from shared inputs"; no GPU
    # value is fed to the oracle).  Bar (c.4, R34): 1e-6 relative to the terms
    # each result sums.
    rng = np.random.default_rng(13)
    n = 8 * 1000
    p = rng.normal(size=n).astype(np.float32)
    z = np.zeros(n, np.float32)
    dev = {k: to_dev(z) for k in ("m", "v", "n", "gp")}
    pt = to_dev(p)
    o = dict(p=p.copy(), m=z.copy(), v=z.copy(), n=z.copy(), gp=z.copy())
    b1, b2, b3 = (float(np.float32(x)) for x in (0.98, 0.92, 0.99))
    for step in (1, 2, 3):
        g = (rng.normal(size=n) * 10.0 ** rng.uniform(-4, 1, size=n)).astype(np.float32)
        po, mo, vo, no = gio.adan(o["p"], g, o["m"], o["v"], o["n"], o["gp"], step, 1e-3)
        pt.copy_(to_dev(o["p"]))
        for k in ("m", "v", "n", "gp"):
            dev[k].copy_(to_dev(o[k]))
        gi.gi_adan_step(pt, to_dev(g), dev["m"], dev["v"], dev["n"], dev["gp"], n, step, 1e-3)
        gd = g.astype(np.float64)
        d = gd - o["gp"] if step > 1 else np.zeros(n)
        sc = {"p": np.abs(o["p"]) + np.abs(po - o["p"]),
              "m": np.abs(b1 * o["m"]) + np.abs((1 - b1) * gd),
              "v": np.abs(b2 * o["v"]) + np.abs((1 - b2) * d),
              "n": np.abs(b3 * o["n"]) + (1 - b3) * (gd + b2 * d) ** 2}
        for name, got, ref in (("p", pt, po), ("m", dev["m"], mo), ("v", dev["v"], vo),
                               ("n", dev["n"], no)):
            got = got.cpu().numpy().astype(np.float64)
            assert np.all(np.abs(got - ref) <= 1e-6 * sc[name] + 1e-12), (step, name)
        assert np.array_equal(dev["gp"].cpu().numpy(), g)
        o = dict(p=po.astype(np.float32), m=mo.astype(np.float32), v=vo.astype(np.float32),
                 n=no.astype(np.float32), gp=g.copy())


def test_fit_step_adan(gi, gio):
    # fused Adan fit step: gradients and the first update vs the oracle
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 64, 64, 256
    p = synth.init_params(0, n)
    tgt = synth.image(0, W, H)
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), optimizer="adan")
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK and fit.steps_done() == 1
    img, loss, g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    assert max(group_err(fit.grads[0].cpu().numpy().astype(np.float64), g).values()) <= GRAD_TOL
    z = np.zeros_like(p)
    po, _, _, _ = gio.adan(p, g.astype(np.float32), z, z, z, z, 1, 1e-3)
    got = fit.params[0].cpu().numpy().astype(np.float64)
    big = np.abs(g) > 1e-3 * np.sqrt(np.mean(g ** 2, axis=0, keepdims=True))
    assert np.all(np.abs(got - po)[big] <= 1e-6 * np.abs(po)[big] + 1e-9)
    for _ in range(20):
        fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK and float(fit.loss[0]) < loss


def test_adan_fused_matches_kernel_sequence(gi, gio):
    # NEXT-1: the Adan update fused into finalize -- plain (3 kernels) and
    # chained (2 kernels) -- is bitwise the standalone sequence
    # gi_render_backward -> gi_adan_step over 4 steps
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    W, H, n = 96, 64, 600
    p = synth.init_params(5, n)
    tgt = synth.image(5, W, H)
    res = []
    for chained in (True, False):
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(),
                     optimizer="adan", chained=chained)
        for _ in range(4):
            fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK and fit.steps_done() == 4
        res.append(fit.params.clone())
    assert torch.equal(res[0], res[1])
    pipe = Pipeline(n, W, H, 1, device=DEV)
    pt = to_dev(p)[None].contiguous()
    st = {k: torch.zeros_like(pt) for k in ("m", "v", "n", "gp")}
    t_dev = to_dev(tgt)[None].contiguous()
    for step in range(1, 5):
        pipe.render(pt)
        pipe.backward(pt, target=t_dev)
        gi.gi_adan_step(pt, pipe.grads, st["m"], st["v"], st["n"], st["gp"], n * 8, step, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(pt, res[1])


def test_c3_backward_and_fit_step(gi, gio):
    # configs[2] at full size: fused forward + L2 + backward and one fused fit
    # step (the launch shape of a C3 fit) against the oracle, full gradient
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 2040, 1356, 100000
    p = synth.init_params(2, n)
    tgt = synth.image(2, W, H)
    img, loss, g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
    out = run_gpu(gi, p[None], W, H, target_b=tgt[None])
    assert np.abs(out["image"][0] - img).max() <= PIX_TOL
    assert max(group_err(out["grads"][0], g).values()) <= GRAD_TOL
    assert abs(out["loss"][0] - loss) <= 1e-5 * loss
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    assert abs(float(fit.loss[0]) - loss) <= 1e-5 * loss
    assert max(group_err(fit.grads[0].cpu().numpy().astype(np.float64), g).values()) <= GRAD_TOL


def test_batched_fit_step(gi, gio):
    # configs[3] pattern: 4 images in one fused fit step, per-image parity
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n, B = 160, 96, 1500, 4
    pb = np.stack([synth.init_params(40 + b, n) for b in range(B)])
    tb = np.stack([synth.image(40 + b, W, H) for b in range(B)])
    fit = Fitter(to_dev(pb).contiguous(), to_dev(tb).contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    for b in range(B):
        img, loss, g = gio.loss_and_grads(pb[b], tb[b], mode=gio.ALL_PAIRS)
        assert abs(float(fit.loss[b]) - loss) <= 1e-5 * loss
        assert max(group_err(fit.grads[b].cpu().numpy().astype(np.float64), g).values()) <= GRAD_TOL


def rs_params(seed, n, scale=1.0):
    # NEXT-3: init-like rotation-scaling cloud (theta ~ U(-pi, pi), s ~ U[0,1) x scale)
    p = synth.init_params(seed, n)
    rng = np.random.default_rng(500 + seed)
    p[:, 2] = rng.uniform(-np.pi, np.pi, size=n).astype(np.float32)
    p[:, 3:5] = (rng.uniform(0.0, 1.0, size=(n, 2)) * scale).astype(np.float32)
    return p


@pytest.mark.parametrize("W,H,n,scale", [(64, 64, 256, 1.0), (70, 45, 300, 2.5), (768, 512, 70000, 1.0)])
def test_rs_parity(gi, gio, W, H, n, scale):
    RS = gi.GI_COV_RS
    p = rs_params(n, n, scale)
    tgt = synth.image(n % 7, W, H)
    mode = gio.ALL_PAIRS if W * H * n <= 64 * 64 * 300 else gio.TILED
    img, loss, g = gio.loss_and_grads(p, tgt, pos_mode=RS, mode=mode)
    out = run_gpu(gi, p[None], W, H, flags=RS, target_b=tgt[None])
    pr = gio.project(p, W, H, pos_mode=RS)
    rec = out["pipe"].proj.view(-1, 12).cpu().numpy()
    bx, by = rec[:, 7].view(np.uint32), rec[:, 11].view(np.uint32)
    valid = pr["touched"] > 0
    box = np.stack([bx & 0xffff, bx >> 16, by & 0xffff, by >> 16], 1).astype(np.int32)
    assert np.array_equal(box[valid], pr["box"][valid])
    kt, kg, _ = gio.bin(p, W, H, pos_mode=RS)
    assert np.array_equal(u32(out["pipe"].key_gid)[: len(kg)], kg)
    assert np.abs(out["image"][0] - img).max() <= PIX_TOL
    assert max(group_err(out["grads"][0], g).values()) <= GRAD_TOL
    assert abs(out["loss"][0] - loss) <= 1e-5 * max(loss, 1e-3)


def test_rs_fit_steps(gi, gio):
    # fused, chained and Adan fit steps in RS mode: gradients of step 1 vs the
    # oracle; chained == plain bitwise over 4 steps
    from paper_2403_08551_b200.pipeline import Fitter
    RS = gi.GI_COV_RS
    W, H, n = 96, 64, 600
    p = rs_params(3, n)
    tgt = synth.image(3, W, H)
    _, loss, g = gio.loss_and_grads(p, tgt, pos_mode=RS, mode=gio.ALL_PAIRS)
    res = []
    for kw in (dict(chained=True), dict(chained=False), dict(optimizer="adan")):
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), flags=RS, **kw)
        fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        assert abs(float(fit.loss[0]) - loss) <= 1e-5 * loss
        assert max(group_err(fit.grads[0].cpu().numpy().astype(np.float64), g).values()) <= GRAD_TOL
        for _ in range(3):
            fit.step()
        torch.cuda.synchronize()
        res.append(fit.params.clone())
    assert torch.equal(res[0], res[1])


@pytest.mark.parametrize("nt", ["256", "128"])
@pytest.mark.parametrize("per_tile", [2, 40])
def test_direct_binning_overflow(per_tile, nt):
    # slab capacity below the per-tile key count (GI_SLAB_MIN=0 lets the
    # capacity set the slab): overflowing tiles stream their keys in gid order
    # from all Gaussians, so frames, gradients and updates are bitwise those
    # of a roomy slab (and match the oracle); run in a fresh process
    import os
    import subprocess
    import sys
    code = f"""
import numpy as np, torch, synth
from oracle import gio
from paper_2403_08551_b200 import gi
from paper_2403_08551_b200.pipeline import Fitter, Pipeline
W, H, n = 96, 64, 600
p = synth.fitted_params(3, n)
tgt = synth.image(3, W, H)
TT = (W // 16) * (H // 16)
small = TT * {per_tile}
pd = torch.from_numpy(p).cuda()[None].contiguous()
big = 4 * TT * 600
a = Pipeline(n, W, H, 1, key_capacity=big).render_frame(pd).clone()
b = Pipeline(n, W, H, 1, key_capacity=small).render_frame(pd).clone()
torch.cuda.synchronize()
assert torch.equal(a, b)
ref_img, loss, g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
assert np.abs(b[0].cpu().numpy() - ref_img).max() <= 2e-5
res = []
for cap in (big, small):
    fit = Fitter(pd.clone(), torch.from_numpy(tgt).cuda()[None].contiguous(), key_capacity=cap)
    fit.step()
    torch.cuda.synchronize()
    gg = fit.grads[0].cpu().numpy().astype(np.float64)
    for cols in ([0, 1], [2, 3, 4], [5, 6, 7]):
        e = np.linalg.norm(gg[:, cols] - g[:, cols]) / np.linalg.norm(g[:, cols])
        assert e <= 1e-4, (cols, e)
    streamed = fit.seg_stats()[0]
    assert streamed == 0 if cap == big else (streamed > 0 or {per_tile} >= 40), streamed
    for _ in range(3):
        fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    res.append((fit.params.clone(), fit.loss.clone(), fit.n_keys()))
assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
assert res[0][2] == res[1][2]
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GI_SLAB_MIN="0", GI_TILE3_NT=nt, PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_partial_slot_overflow(gi, gio):
    # Gaussians touching ~20 tiles with a tiny key capacity: their backward
    # partial slots do not fit, so their tiles accumulate atomically; the
    # gradients still match the oracle
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 96, 64, 300
    p = synth.init_params(4, n)
    rng = np.random.default_rng(44)
    p[:, 2] = rng.uniform(6.0, 10.0, n).astype(np.float32)
    p[:, 4] = rng.uniform(3.0, 6.0, n).astype(np.float32)
    p[:, 5:8] *= np.float32(0.05)
    tgt = synth.image(4, W, H)
    _, loss, g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    for cap in (None, 48):
        fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), key_capacity=cap)
        fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        assert abs(float(fit.loss[0]) - loss) <= 1e-5 * loss
        assert max(group_err(fit.grads[0].cpu().numpy().astype(np.float64), g).values()) <= GRAD_TOL


@pytest.mark.parametrize("bits,stages,codebook,pos_mode", [(6, 2, 8, 0), (5, 3, 16, 0),
                                                           (8, 2, 8, 1), (4, 1, 256, 0)])
def test_vq_encode_bitexact(gi, gio, bits, stages, codebook, pos_mode):
    # NEXT-2 encoder: codes, packed bytes and dequantised parameters equal the
    # oracle's bit for bit; GPU decode of the GPU payload returns them too
    n = 5003
    rng = np.random.default_rng(bits * 100 + stages)
    p = synth.fitted_params(bits, n)
    if pos_mode:
        p[:, :2] = rng.uniform(-1, 1, (n, 2)).astype(np.float32)
    gamma = np.float32([0.06, 0.05, 0.06]) * np.float32(64.0 / (1 << bits))
    beta = np.float32([-1.5, -1.6, -1.5])
    books = rng.normal(0, 0.3, (stages, codebook, 3)).astype(np.float32)
    ref = gio.vq_encode(p, gamma, beta, books, bits, stages, codebook, pos_mode)
    data = synth.pack_records(ref["pos16"].astype(np.uint16), ref["codes"], ref["idx"], bits,
                              codebook)
    bk = to_dev(books)                      # keep alive: meta holds the raw pointer
    meta = gi.codec_meta(n, gamma, beta, bk, bits=bits, stages=stages, codebook=codebook)
    payload = torch.full((data.size + 8,), 0xAB, dtype=torch.uint8, device=DEV)
    eff = torch.zeros(n, 8, dtype=torch.float32, device=DEV)
    gi.gi_vq_encode(to_dev(p), meta, payload, eff, flags=gi.GI_POS_NORMALIZED if pos_mode else 0)
    torch.cuda.synchronize()
    assert np.array_equal(eff.cpu().numpy().view(np.uint32), ref["eff"].view(np.uint32))
    assert np.array_equal(payload[: data.size].cpu().numpy(), data)
    dec = torch.zeros(n, 8, dtype=torch.float32, device=DEV)
    gi.gi_vq_decode(payload, meta, dec)
    assert torch.equal(dec, eff)


def test_kmeans_step_parity(gi, gio):
    # NEXT-2 codebook init: 5 Lloyd iterations on colours (stage 1) and on
    # the stage-1 residuals (stage 2) vs the oracle; assignments bit-exact,
    # centroids within 1 fp32 ulp-scale (fixed-point vs fp64 summation)
    n, B = 70000, 8
    p = synth.fitted_params(9, n)
    cols = np.ascontiguousarray(p[:, 5:8])
    init = cols[:: n // B][:B].copy()
    ws = torch.zeros(gi.gi_kmeans_workspace_bytes(B), dtype=torch.uint8, device=DEV)
    pts = to_dev(cols)
    cent = to_dev(init)
    asg = torch.zeros(n, dtype=torch.int32, device=DEV)
    ref_c = init.copy()
    for it in range(5):
        ref_c_prev = ref_c
        ref_c, ref_a, _ = gio.kmeans(cols, ref_c_prev, iters=1)
        gi.gi_kmeans_step(pts, cent, asg, ws)
        torch.cuda.synchronize()
        got_c = cent.cpu().numpy()
        assert np.array_equal(asg.cpu().numpy().view(np.uint32), ref_a), it
        assert np.allclose(got_c, ref_c, rtol=3e-7, atol=1e-8), it
        cent = to_dev(ref_c)          # continue both from the oracle's centroids


def test_qat_step_parity(gi, gio):
    # NEXT-2 QAT step vs the oracle's composition (straight-through LSQ+
    # gradients, Adam, EMA codebooks, Eq. 10): quantised cloud bit-exact,
    # gradients per group <= 1e-4, losses, gamma/beta gradients, the updated
    # parameters and codebooks
    from paper_2403_08551_b200.pipeline import QatFitter
    W, H, n = 96, 64, 600
    rng = np.random.default_rng(21)
    p = synth.fitted_params(21, n)
    tgt = synth.image(21, W, H)
    gamma = np.float32([0.05, 0.04, 0.05])
    beta = np.float32([-1.0, -1.2, -1.0])
    books = rng.normal(0, 0.3, (2, 8, 3)).astype(np.float32)
    st = dict(m=np.zeros((n, 8), np.float32), v=np.zeros((n, 8), np.float32), gamma=gamma,
              beta=beta, qm=np.zeros(6, np.float32), qv=np.zeros(6, np.float32), books=books,
              ema_n=np.ones((2, 8), np.float32), ema_s=books.copy())
    ref = gio.qat_step(p, tgt, st, 1, 1e-4, lam=1.0, decay=0.99, mode=gio.ALL_PAIRS)
    q = QatFitter(to_dev(p), to_dev(tgt)[None].contiguous(), gamma, beta, to_dev(books), lr=1e-4)
    q.step()
    torch.cuda.synchronize()
    assert q.check() == gi.GI_OK
    assert np.array_equal(q.eff.cpu().numpy().view(np.uint32), ref["eff"].view(np.uint32))
    errs = group_err(q.grads.cpu().numpy().astype(np.float64), ref["grads"])
    assert max(errs.values()) <= GRAD_TOL, errs
    L = q.losses.cpu().numpy().astype(np.float64)
    assert abs(L[1] - ref["l_rec"]) <= 1e-5 * ref["l_rec"]
    assert abs(L[2] - ref["l_c"]) <= 1e-6 * ref["l_c"]
    assert abs(L[0] - ref["loss"]) <= 1e-5 * ref["loss"]
    dq = np.concatenate([ref["dgamma"], ref["dbeta"]])
    assert np.allclose(L[3:], dq, rtol=1e-4, atol=1e-9 * np.abs(dq).max())
    got = q.params.cpu().numpy().astype(np.float64)
    g = ref["grads"]
    big = np.abs(g) > 1e-3 * np.sqrt(np.mean(g ** 2, axis=0, keepdims=True))
    assert np.all(np.abs(got - ref["params"])[big] <= 1e-6 * np.abs(ref["params"])[big] + 1e-9)
    assert np.allclose(q.books.cpu().numpy(), ref["state"]["books"], atol=1e-6)
    assert np.allclose(q.ema_n.cpu().numpy(), ref["state"]["ema_n"], rtol=1e-6)
    assert np.allclose(q.ema_s.cpu().numpy(), ref["state"]["ema_s"], atol=1e-6)
    # a captured graph of QAT steps keeps running and the loss falls
    q.capture(10)
    for _ in range(5):
        q.replay()
    torch.cuda.synchronize()
    assert q.check() == gi.GI_OK and float(q.losses[0]) < ref["loss"]


def test_spatial_windows_batch2(gi, gio):
    # NEXT-4 windows on a 2-image launch: per image, the windows add up to
    # the whole image
    from paper_2403_08551_b200.dist import row_windows
    from paper_2403_08551_b200.pipeline import _bytes, default_capacity
    W, H, n, B = 80, 64, 400, 2
    p = np.stack([params_for(n, 11 + b, True) for b in range(B)])
    tgt = np.stack([synth.image(11 + b, W, H) for b in range(B)])
    f = gi.frame(W, H, B)
    cap = default_capacity(n, B)
    ws = _bytes(gi.gi_fit_workspace_bytes(n, cap, f), DEV)
    pd, td = to_dev(p).contiguous(), to_dev(tgt).contiguous()
    acc = torch.zeros(B, n, 8, dtype=torch.float64, device=DEV)
    lsum = torch.zeros(B, dtype=torch.float64, device=DEV)
    for (r0, rows) in row_windows(H // 16, 3):
        gr = torch.zeros(B, n, 8, dtype=torch.float32, device=DEV)
        lo = torch.zeros(B, dtype=torch.float32, device=DEV)
        gi.gi_fit_grads(pd, gr, td, n, f, 0, r0, rows, cap, ws, lo)
        torch.cuda.synchronize()
        acc += gr.double()
        lsum += lo.double()
    for b in range(B):
        _, loss, g = gio.loss_and_grads(p[b], tgt[b], mode=gio.TILED)
        assert max(group_err(acc[b].cpu().numpy(), g).values()) <= GRAD_TOL
        assert abs(float(lsum[b]) - loss) <= 1e-5 * loss


@pytest.mark.parametrize("parts", [2, 3])
def test_spatial_windows_sum_to_whole(gi, gio, parts):
    # NEXT-4: gradients and loss of tile-row windows covering the image add up
    # to the whole image's (and to the oracle's); the ranks of a sharded fit
    # are simulated one after another on this GPU
    from paper_2403_08551_b200.dist import row_windows
    from paper_2403_08551_b200.pipeline import _bytes, default_capacity
    W, H, n = 96, 80, 700
    p = params_for(n, 5, True)
    tgt = synth.image(5, W, H)
    _, loss, g = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    f = gi.frame(W, H, 1)
    cap = default_capacity(n, 1)
    ws = _bytes(gi.gi_fit_workspace_bytes(n, cap, f), DEV)
    pd, td = to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous()
    acc = torch.zeros(1, n, 8, dtype=torch.float64, device=DEV)
    lsum = 0.0
    for (r0, rows) in row_windows(H // 16, parts):
        gr = torch.zeros(1, n, 8, dtype=torch.float32, device=DEV)
        lo = torch.zeros(1, dtype=torch.float32, device=DEV)
        gi.gi_fit_grads(pd, gr, td, n, f, 0, r0, rows, cap, ws, lo)
        torch.cuda.synchronize()
        acc += gr.double()
        lsum += float(lo[0])
    whole = torch.zeros(1, n, 8, dtype=torch.float32, device=DEV)
    lw = torch.zeros(1, dtype=torch.float32, device=DEV)
    gi.gi_fit_grads(pd, whole, td, n, f, 0, 0, -1, cap, ws, lw)
    torch.cuda.synchronize()
    a = acc[0].cpu().numpy()
    assert max(group_err(a, whole[0].cpu().numpy().astype(np.float64)).values()) <= 1e-6
    assert max(group_err(a, g).values()) <= GRAD_TOL
    assert abs(lsum - float(lw[0])) <= 1e-6 * float(lw[0])
    assert abs(lsum - loss) <= 1e-5 * loss


def test_spatial_fitter_single_rank(gi, gio):
    # NEXT-4 driver with one rank = gi_fit_grads + gi_adam_step: follows the
    # fused fit step (same Adam up to its approximate reciprocal / sqrt)
    from paper_2403_08551_b200.dist import SpatialFitter
    from paper_2403_08551_b200.pipeline import Fitter
    W, H, n = 64, 64, 256
    p = synth.init_params(0, n)
    tgt = synth.image(0, W, H)
    a = SpatialFitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    b = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous(), chained=False)
    for _ in range(3):
        a.step()
        b.step()
    torch.cuda.synchronize()
    assert torch.allclose(a.params, b.params, rtol=1e-5, atol=1e-7)
    assert abs(float(a.loss[0]) - float(b.loss[0])) <= 1e-5 * float(b.loss[0])


def test_peer_adam_step_local(gi):
    # NEXT-4 exchange kernel with G local buffers: the rank-order sum followed
    # by Adam is bitwise gi_adam_step on that sum; the loss tail is summed
    rng = np.random.default_rng(41)
    count = 8 * 1001
    p0 = to_dev(rng.normal(size=count).astype(np.float32))
    bufs = [to_dev(rng.normal(size=count + 2).astype(np.float32)) for _ in range(3)]
    for G in (1, 3):
        p, m, v = p0.clone(), torch.zeros_like(p0), torch.zeros_like(p0)
        q, mq, vq = p0.clone(), torch.zeros_like(p0), torch.zeros_like(p0)
        loss = torch.zeros(2, device=DEV)
        for step in (1, 2):
            gi.gi_peer_adam_step(p, m, v, [b.data_ptr() for b in bufs[:G]], count, step, 1e-3,
                                 n_loss=2, loss_out=loss)
            gsum = bufs[0][:count].clone()
            for b in bufs[1:G]:
                gsum += b[:count]
            gi.gi_adam_step(q, gsum, mq, vq, count, step, 1e-3)
        torch.cuda.synchronize()
        assert torch.equal(p, q) and torch.equal(m, mq) and torch.equal(v, vq)
        lsum = bufs[0][count:].clone()
        for b in bufs[1:G]:
            lsum += b[count:]
        assert torch.equal(loss, lsum)
    ptr, handle = gi.gi_peer_alloc(4096)
    assert len(handle) == 64
    gi.gi_peer_free(ptr)


def _peer_worker(rank, world, port, p, tgt, steps, q):
    import os
    import torch.distributed as dist
    from paper_2403_08551_b200.dist import SpatialFitter
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)                   # both ranks on the one GPU: the IPC plumbing
    f = SpatialFitter(torch.from_numpy(p).cuda()[None].contiguous(),
                      torch.from_numpy(tgt).cuda()[None].contiguous(), rank=rank, world=world,
                      exchange="peer")
    for _ in range(steps):
        f.step()
    torch.cuda.synchronize()
    q.put((rank, f.params.cpu().numpy(), float(f.loss[0])))
    f.close()
    dist.destroy_process_group()


def test_spatial_peer_exchange_two_processes(gi, gio):
    # NEXT-4 over peer memory end to end: two processes (gloo for the handle
    # exchange and the barriers; both on this GPU -- no kernel waits on the
    # other process) run 3 peer-exchange steps; both replicas equal, bitwise,
    # the same 3 steps computed in one process (window gradients of both row
    # windows -> gi_peer_adam_step over the two buffers)
    import socket
    import torch.multiprocessing as mp
    from paper_2403_08551_b200.dist import row_windows
    from paper_2403_08551_b200.pipeline import _bytes, default_capacity
    W, H, n, steps = 96, 64, 600, 3
    p = synth.init_params(12, n)
    tgt = synth.image(12, W, H)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, p, tgt, steps, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict((r, (pp, ll)) for r, pp, ll in (q.get(timeout=300) for _ in range(2)))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert np.array_equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]
    # single-process reference
    f = gi.frame(W, H, 1)
    cap = default_capacity(n, 1)
    ws = _bytes(gi.gi_fit_workspace_bytes(n, cap, f), DEV)
    prm = to_dev(p)[None].contiguous()
    m, v = torch.zeros_like(prm), torch.zeros_like(prm)
    t_dev = to_dev(tgt)[None].contiguous()
    bufs = [torch.zeros(n * 8 + 1, device=DEV) for _ in range(2)]
    loss = torch.zeros(1, device=DEV)
    wins = row_windows((H + 15) // 16, 2)
    for step in range(1, steps + 1):
        for b, (r0, rows) in zip(bufs, wins):
            gi.gi_fit_grads(prm, b, t_dev, n, f, 0, r0, rows, cap, ws, b[n * 8:])
        gi.gi_peer_adam_step(prm, m, v, [b.data_ptr() for b in bufs], n * 8, step, 1e-3,
                             n_loss=1, loss_out=loss)
    torch.cuda.synchronize()
    assert np.array_equal(prm[0].cpu().numpy(), res[0][0][0])
    assert float(loss[0]) == res[0][1]
    # and it fits: the loss after 3 steps is the whole image's (up to fp32 order)
    _, ref_loss, _ = gio.loss_and_grads(p, tgt, mode=gio.ALL_PAIRS)
    assert res[0][1] < 1.01 * ref_loss


def test_new_entry_edge_cases(gi, gio):
    # gi_decode_render_frame with no records: a zero frame; chained Adan on a
    # 2-image launch equals the plain fused Adan step bitwise over 3 steps
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    books = to_dev(np.zeros((2, 8, 3), np.float32))
    meta = gi.codec_meta(0, [0.1] * 3, [0.0] * 3, books)
    pipe = Pipeline(0, 40, 24, 1, device=DEV)
    pipe.image.fill_(1.0)
    pipe.decode_render_frame(torch.zeros(8, dtype=torch.uint8, device=DEV), meta)
    torch.cuda.synchronize()
    assert not pipe.image.any()
    W, H, n = 80, 48, 300
    ps = np.stack([synth.init_params(20 + b, n) for b in range(2)])
    ts = np.stack([synth.image(20 + b, W, H) for b in range(2)])
    res = []
    for chained in (True, False):
        fit = Fitter(to_dev(ps).contiguous(), to_dev(ts).contiguous(), optimizer="adan",
                     chained=chained)
        for _ in range(3):
            fit.step()
        torch.cuda.synchronize()
        assert fit.check() == gi.GI_OK
        res.append(fit.params.clone())
    assert torch.equal(res[0], res[1])


def test_render_one_pixel_variant():
    # the round-1 one-pixel-per-thread render kernel (GI_RENDER3=0
    # GI_RENDER2=0, the A/B baseline) stays within the pixel bar: C2 init and
    # a ragged frame, fused frame vs the oracle, in a fresh process
    import os
    import subprocess
    import sys
    code = """
import numpy as np, torch, synth
from oracle import gio
from paper_2403_08551_b200.pipeline import Pipeline
for W, H, n, seed in ((768, 512, 70000, 1), (70, 45, 300, 1)):
    p = synth.init_params(seed, n)
    ref = gio.render(p, W, H, mode=gio.TILED)
    img = Pipeline(n, W, H, 1).render_frame(torch.from_numpy(p).cuda()[None].contiguous())
    err = float(np.abs(img[0].cpu().numpy() - ref).max())
    assert err <= 2e-5, err
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GI_RENDER2="0", GI_RENDER3="0", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


VARIANTS = {
    "tile3_256": {"GI_TILE3_NT": "256", "GI_RENDER3": "1"},
    "tile3_128": {"GI_TILE3_NT": "128", "GI_RENDER3": "1"},
    "round1_onepixel": {"GI_TILE3": "0", "GI_TILE2": "0", "GI_RENDER2": "0"},
    "round1_twopixel": {"GI_TILE3": "0", "GI_TILE2": "1"},
}


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_tile_kernel_variants(variant):
    # every fused tile kernel (Gaussian-parallel at 256 / 128 threads, the
    # round-1 one- and two-pixel kernels) and render kernel in a fresh
    # process with the choice forced: C2 init frame + fused fit-step
    # gradients, a 3-image launch and a tile past every sort buffer vs the
    # oracle
    import os
    import subprocess
    import sys
    code = """
import numpy as np, torch, synth
from oracle import gio
from paper_2403_08551_b200.pipeline import Fitter
big = synth.init_params(6, 1500)
big[:, 2] += 3.0                    # boxes ~ 20 px: ~1,500 keys per tile, past the
big[:, 4] += 3.0                    # two-pixel kernel's 1,024-key sort buffer
big[:, 5:8] *= 0.002
cases = [(768, 512, [synth.init_params(1, 70000)], [synth.image(1, 768, 512)]),
         (96, 70, [synth.fitted_params(s, 900) for s in (3, 4, 5)],
          [synth.image(s, 96, 70) for s in (3, 4, 5)]),
         (32, 32, [big], [synth.image(6, 32, 32)])]
from paper_2403_08551_b200.pipeline import Pipeline
for W, H, ps, ts in cases:
    pd = torch.from_numpy(np.stack(ps)).cuda().contiguous()
    fit = Fitter(pd.clone(), torch.from_numpy(np.stack(ts)).cuda().contiguous())
    fit.step()
    g = fit.grads.cpu().numpy().astype(np.float64)
    img = Pipeline(ps[0].shape[0], W, H, len(ps)).render_frame(pd).cpu().numpy()
    for b in range(len(ps)):
        mode = gio.TILED if W * H > 10000 else gio.ALL_PAIRS
        ref_img, loss, rg = gio.loss_and_grads(ps[b], ts[b], mode=mode)
        assert np.all(np.abs(img[b] - ref_img) <= 2e-5 * np.maximum(1.0, np.abs(ref_img)))
        assert abs(float(fit.loss[b]) - loss) <= 1e-5 * loss
        for cols in ([0, 1], [2, 3, 4], [5, 6, 7]):
            e = np.linalg.norm(g[b][:, cols] - rg[:, cols]) / np.linalg.norm(rg[:, cols])
            assert e <= 1e-4, (b, cols, e)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, **VARIANTS[variant])
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_next_edge_cases(gi, gio):
    # NEXT-2/4 entry points on empty and tiny inputs
    from paper_2403_08551_b200.pipeline import QatFitter, _bytes, default_capacity
    books = to_dev(np.zeros((2, 8, 3), np.float32))
    meta = gi.codec_meta(0, [0.1] * 3, [0.0] * 3, books)
    gi.gi_vq_encode(torch.zeros(1, 8, device=DEV), meta,
                    torch.zeros(8, dtype=torch.uint8, device=DEV), torch.zeros(1, 8, device=DEV))
    ws = torch.zeros(gi.gi_kmeans_workspace_bytes(8), dtype=torch.uint8, device=DEV)
    cent = to_dev(np.arange(24, dtype=np.float32).reshape(8, 3))
    gi.gi_kmeans_step(torch.zeros(0, 3, device=DEV), cent, None, ws)
    torch.cuda.synchronize()
    assert torch.equal(cent.cpu(), torch.arange(24, dtype=torch.float32).view(8, 3))
    # one Gaussian: QAT step against the oracle
    p = synth.fitted_params(2, 1)
    tgt = synth.image(2, 20, 12)
    st = dict(m=np.zeros((1, 8), np.float32), v=np.zeros((1, 8), np.float32),
              gamma=np.float32([0.05] * 3), beta=np.float32([-1.0] * 3),
              qm=np.zeros(6, np.float32), qv=np.zeros(6, np.float32),
              books=np.zeros((2, 8, 3), np.float32), ema_n=np.ones((2, 8), np.float32),
              ema_s=np.zeros((2, 8, 3), np.float32))
    ref = gio.qat_step(p, tgt, st, 1, 1e-4, mode=gio.ALL_PAIRS)
    q = QatFitter(to_dev(p), to_dev(tgt)[None].contiguous(), [0.05] * 3, [-1.0] * 3, books)
    q.step()
    torch.cuda.synchronize()
    assert np.array_equal(q.eff.cpu().numpy().view(np.uint32), ref["eff"].view(np.uint32))
    assert abs(float(q.losses[1]) - ref["l_rec"]) <= 1e-5 * ref["l_rec"]
    # a zero-row window contributes nothing
    f = gi.frame(64, 48, 1)
    pp = to_dev(synth.init_params(3, 100))[None].contiguous()
    cap = default_capacity(100, 1)
    fws = _bytes(gi.gi_fit_workspace_bytes(100, cap, f), DEV)
    gr = torch.ones(1, 100, 8, device=DEV)
    lo = torch.ones(1, device=DEV)
    gi.gi_fit_grads(pp, gr, to_dev(synth.image(3, 64, 48))[None].contiguous(), 100, f, 0, 1, 0,
                    cap, fws, lo)
    torch.cuda.synchronize()
    assert not gr.any() and float(lo[0]) == 0.0


def test_target_from_rgb8(gi):
    # 8-bit RGB targets (the paper's datasets): interleaved u8 -> planar
    # fp32 u / 255, bit-exact against the definition (IEEE fp32 division)
    rng = np.random.default_rng(8)
    for W, H, B in ((768, 512, 1), (70, 45, 3), (5, 3, 2)):
        rgb = rng.integers(0, 256, size=(B, H, W, 3), dtype=np.uint8)
        rgb.reshape(-1)[:2] = (0, 255)
        ref = np.ascontiguousarray((rgb.astype(np.float32) / np.float32(255)).transpose(0, 3, 1, 2))
        out = torch.full((B, 3, H, W), float("nan"), device=DEV)
        gi.gi_target_from_rgb8(to_dev(rgb), gi.frame(W, H, B), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32)), (W, H, B)
        # from host memory: upload on a copy stream, expansion on the compute
        # stream after the upload's event -- same bits
        host = torch.from_numpy(rgb).pin_memory()
        stage = torch.empty(rgb.shape, dtype=torch.uint8, device=DEV)
        out2 = torch.full((B, 3, H, W), float("nan"), device=DEV)
        cs = torch.cuda.Stream()
        ready, done = torch.cuda.Event(), torch.cuda.Event()
        ready.record(torch.cuda.current_stream())
        done.record(torch.cuda.current_stream())
        fr = gi.frame(W, H, B)
        gi.gi_target_upload_rgb8(host, stage, fr, None, ready, cs)
        gi.gi_target_from_rgb8(stage, fr, out2, ready, done)
        torch.cuda.synchronize()
        assert np.array_equal(out2.cpu().numpy().view(np.uint32), ref.view(np.uint32)), (W, H, B)


@pytest.mark.parametrize("W,H", [(32767, 40), (40, 32767)])
def test_max_frame_dims(gi, gio, W, H):
    # the largest frame gi_frame accepts along each axis (ragged: 32767 = 2047
    # tiles + 15 px): 16-bit box words at their limit, 2,048 x 3 tiles (the
    # >= 3,072-tile kernels); frame, fused fit-step gradients and loss vs the oracle
    from paper_2403_08551_b200.pipeline import Fitter, Pipeline
    n = 4000
    p = synth.init_params(31, n)
    tgt = synth.image(31, W, H)
    ref_img, ref_loss, ref_g = gio.loss_and_grads(p, tgt, mode=gio.TILED)
    pipe = Pipeline(n, W, H, 1, device=DEV)
    img = pipe.render_frame(to_dev(p)[None].contiguous())[0].cpu().numpy()
    assert np.abs(img - ref_img).max() <= PIX_TOL
    fit = Fitter(to_dev(p)[None].contiguous(), to_dev(tgt)[None].contiguous())
    fit.step()
    torch.cuda.synchronize()
    assert fit.check() == gi.GI_OK
    assert max(group_err(fit.grads[0].cpu().numpy().astype(np.float64), ref_g).values()) <= GRAD_TOL
    assert abs(float(fit.loss[0]) - ref_loss) <= 1e-5 * ref_loss
