"""Pins for the fp64 oracle (``-m "not gpu"``): worked examples, closed forms,
brute force and finite differences -- never a retyped copy of its formula.

Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
Each pin is chosen so that a plausible slip in the oracle (dropped term, wrong
sign or index, transposed operand, wrong box rounding) fails at least one.
"""
import math

import numpy as np
import pytest

import synth

NORM = 1  # pos_mode: params[0:2] are normalised positions u in (-1, 1)


def one(u, l, c, extra=None):
    p = np.array([[u[0], u[1], l[0], l[1], l[2], c[0], c[1], c[2]]], np.float32)
    if extra is not None:
        p = np.concatenate([p, np.asarray(extra, np.float32)], 0)
    return p


# ------------------------------------------------------------- Eq. 1 / Eq. 5
def test_covariance_worked_examples(gio):
    # S:52-53 (Eq. 1): raw (0.5,0,0.5) -> L = I -> Sigma = I;
    # raw (1.5,1,0.5) -> L = [[2,0],[1,1]] -> Sigma = [[4,2],[2,2]]
    pr = gio.project(one((0, 0), (0.5, 0, 0.5), (1, 1, 1)), 10, 10, pos_mode=NORM)
    assert np.array_equal(pr["sigma"][0], [1.0, 0.0, 1.0])
    pr = gio.project(one((0, 0), (1.5, 1.0, 0.5), (1, 1, 1)), 10, 10, pos_mode=NORM)
    assert np.array_equal(pr["sigma"][0], [4.0, 2.0, 2.0])
    # inverse of [[4,2],[2,2]] = [[0.5,-0.5],[-0.5,1]] (det 4)
    assert np.array_equal(pr["sinv"][0], [0.5, -0.5, 1.0])


def test_inverse_multiply_back(gio):
    # Sigma Sigma^-1 = I for random SPD matrices (invariant)
    rng = np.random.default_rng(5)
    for _ in range(200):
        L = np.array([[rng.uniform(0.2, 3), 0], [rng.uniform(-2, 2), rng.uniform(0.2, 3)]])
        S = L @ L.T
        si = gio.inverse2([S[0, 0], S[0, 1], S[1, 1]])
        Si = np.array([[si[0], si[1]], [si[1], si[2]]])
        assert np.allclose(S @ Si, np.eye(2), atol=1e-12)


def test_sigma_worked_examples(gio):
    # S:115-117 (Eq. 5): Sigma = I, d = 0 -> 0; d = (1,1) -> 1.0;
    # Sigma = [[4,2],[2,2]], d = (1,0) -> 0.25
    assert gio.eval_sigma([1, 0, 1], 0, 0) == 0.0
    assert gio.eval_sigma([1, 0, 1], 1, 1) == 1.0
    assert gio.eval_sigma([0.5, -0.5, 1.0], 1, 0) == 0.25
    # off-diagonal enters twice (d^T S d) -- catches a dropped factor 2
    assert gio.eval_sigma([0.5, -0.5, 1.0], 1, 1) == 0.5 * (0.5 - 1.0 + 1.0)


def test_position_map(gio):
    # S:70 (App. C, reading R2): mu_raw = (0,0) at 768x512 -> (384, 256)
    pr = gio.project(one((0, 0), (0.5, 0, 0.5), (1, 1, 1)), 768, 512)
    assert np.array_equal(pr["mu"][0], [384.0, 256.0])
    # u = (0.5, -0.5) at 100x100 -> (75, 25); exact in normalised mode,
    # through tanh(atanh(.)) within the fp32 rounding of the logit
    pr = gio.project(one((0.5, -0.5), (0.5, 0, 0.5), (1, 1, 1)), 100, 100, pos_mode=NORM)
    assert np.array_equal(pr["mu"][0], [75.0, 25.0])
    lg = np.float32(math.atanh(0.5))
    pr = gio.project(one((lg, -lg), (0.5, 0, 0.5), (1, 1, 1)), 100, 100)
    assert np.allclose(pr["mu"][0], [75.0, 25.0], atol=1e-5)


# ------------------------------------------------------------ box (R6, R7)
def test_box_closed_form(gio):
    # Sigma = I, k = 3: pixels whose centre x + 1/2 is within 3 of mu.
    # mu = 50 -> x + .5 in [47, 53] -> x in [47, 52]   (R7; NOT S:133's [47,53])
    pr = gio.project(one((0, 0), (0.5, 0, 0.5), (1, 1, 1)), 100, 100, pos_mode=NORM)
    assert list(pr["box"][0]) == [47, 52, 47, 52]
    # mu = 50.5 (W = 101) -> x in [47, 53]
    pr = gio.project(one((0, 0), (0.5, 0, 0.5), (1, 1, 1)), 101, 101, pos_mode=NORM)
    assert list(pr["box"][0]) == [47, 53, 47, 53]
    # S:135 anisotropic Sigma = [[16,0],[0,1]]: half extents (12, 3)
    pr = gio.project(one((0, 0), (3.5, 0, 0.5), (1, 1, 1)), 101, 101, pos_mode=NORM)
    assert list(pr["box"][0]) == [38, 62, 47, 53]
    # y extent uses sqrt(Syy) = sqrt(l2^2 + l3^2): l2 = 3, l3e = 4 -> 5 -> 15 px
    pr = gio.project(one((0, 0), (0.5, 3.0, 3.5), (1, 1, 1)), 101, 101, pos_mode=NORM)
    assert list(pr["box"][0]) == [47, 53, 35, 65]


def test_box_brute_force(gio):
    # box == {pixels with |x + 1/2 - mu_x| <= k sqrt(Sxx)} (and same in y),
    # checked against a brute-force scan in exact rational-ish fp64.
    rng = np.random.default_rng(11)
    W, H = 37, 29
    p = synth.init_params(3, 300)
    p[:, 2:5] = rng.uniform(-0.4, 2.0, size=(300, 3)).astype(np.float32)
    pr = gio.project(p, W, H, k=3.0)
    for i in range(300):
        mu = pr["mu"][i]
        S = pr["sigma"][i]
        rx, ry = 3.0 * math.sqrt(S[0]), 3.0 * math.sqrt(S[2])
        xs = [x for x in range(W) if abs(x + 0.5 - mu[0]) <= rx]
        ys = [y for y in range(H) if abs(y + 0.5 - mu[1]) <= ry]
        b = pr["box"][i]
        if not xs or not ys:
            assert b[0] > b[1]
            continue
        # fp32 recipe may differ from this fp64 scan only at exact ties
        assert abs(b[0] - xs[0]) <= 0 or abs(xs[0] + 0.5 - mu[0] + rx) < 1e-4
        assert abs(b[1] - xs[-1]) <= 0 or abs(xs[-1] + 0.5 - mu[0] - rx) < 1e-4
        assert abs(b[2] - ys[0]) <= 0 or abs(ys[0] + 0.5 - mu[1] + ry) < 1e-4
        assert abs(b[3] - ys[-1]) <= 0 or abs(ys[-1] + 0.5 - mu[1] - ry) < 1e-4


def test_box_cull_and_offscreen(gio):
    # R8: l1 + 0.5 == 0 culls; S:134 centre outside the frame by > k std -> empty
    pr = gio.project(one((0, 0), (-0.5, 0, 0.5), (1, 1, 1)), 64, 64, pos_mode=NORM)
    assert pr["touched"][0] == 0 and pr["box"][0][0] > pr["box"][0][1]
    # (u in [-1, 1] keeps mu inside the frame, so "outside" = on the border
    # with a support that reaches no pixel centre: mu = W, k |l1e| = 0.3 < 0.5)
    pr = gio.project(one((1.0, 0), (-0.4, 0, 0.0), (1, 1, 1)), 1000, 64, pos_mode=NORM)
    assert pr["touched"][0] == 0
    pr = gio.project(one((1.0, 0), (-0.3, 0, 0.0), (1, 1, 1)), 1000, 64, pos_mode=NORM)
    assert list(pr["box"][0][:2]) == [999, 999]     # k |l1e| = 0.6 >= 0.5
    # signed diagonal (l1 + 0.5 < 0) is allowed: |l1e| sets the extent (R8)
    pr = gio.project(one((0, 0), (-1.5, 0, 0.5), (1, 1, 1)), 100, 100, pos_mode=NORM)
    assert list(pr["box"][0]) == [47, 52, 47, 52]


# ------------------------------------------------------------------ binning
@pytest.mark.parametrize("tile", [1, 8, 13, 16])
def test_bin_two_methods_agree(gio, tile):
    for seed, (W, H, n) in enumerate([(64, 64, 256), (70, 45, 300), (33, 17, 50)]):
        p = synth.init_params(seed, n)
        a = gio.bin(p, W, H, tile=tile, method=0)
        b = gio.bin(p, W, H, tile=tile, method=1)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        kt, kg, rng = b
        # every (tile, gid) pair present exactly once; ascending gid within a tile
        pr = gio.project(p, W, H, tile=tile)
        TX = (W + tile - 1) // tile
        want = sorted((ty * TX + tx, i) for i in range(n) for (tx0, tx1, ty0, ty1) in [pr["rect"][i]]
                      for ty in range(ty0, ty1 + 1) for tx in range(tx0, tx1 + 1))
        assert [tuple(v) for v in zip(kt.tolist(), kg.tolist())] == want
        assert rng[0] == 0 and rng[-1] == len(kt)
        assert int(pr["touched"].sum()) == len(kt)


# ------------------------------------------------------------ Eq. 7 render
def test_centred_gaussian_returns_colour(gio):
    # sigma = 0 at the pixel centre -> C = c' exactly (W = 64, x = 31:
    # mu = (1 - 1/64) * 32 = 31.5 = 31 + 1/2)
    c = (0.3125, -0.75, 1.5)
    p = one((-0.015625, -0.015625), (0.7, 0.3, 0.2), c)
    for mode in (gio.ALL_PAIRS, gio.TILED, gio.DENSE):
        img = gio.render(p, 64, 64, pos_mode=NORM, mode=mode)
        assert tuple(img[:, 31, 31]) == c


def test_lattice_sum_equals_gaussian_integral(gio):
    # Dense sum over the pixel lattice of exp(-sigma) = integral of the
    # Gaussian = 2 pi sqrt(det Sigma) = 2 pi l1e l3e (Poisson summation,
    # aliasing ~ exp(-2 pi^2 s^2) < 1e-18 for min axis s >= 1.5 px).
    for (l1, l2, l3, ux, uy) in [(1.5, 0.5, 1.3, 0.01, -0.02), (2.2, -1.0, 1.0, 0.1, 0.05),
                                 (1.0, 0.0, 1.0, -0.03, 0.07)]:
        p = one((ux, uy), (l1, l2, l3), (1.0, 0.0, 0.0))
        img = gio.render(p, 96, 96, pos_mode=NORM, mode=gio.DENSE)
        want = 2 * math.pi * (float(np.float32(l1)) + 0.5) * (float(np.float32(l3)) + 0.5)
        assert abs(img[0].sum() / want - 1) < 1e-12
        assert img[1].sum() == 0.0 and img[2].sum() == 0.0


def test_separable_box_sum(gio):
    # l2 = 0: exp(-sigma) = exp(-dx^2 / 2 l1e^2) exp(-dy^2 / 2 l3e^2), so the
    # boxed sum factorises into two 1-D sums over the box ranges.
    p = one((0.013, -0.021), (0.875, 0.0, 0.375), (1.0, 0.0, 0.0))   # l1e 1.375, l3e .875
    W, H = 64, 48
    pr = gio.project(p, W, H, pos_mode=NORM)
    x0, x1, y0, y1 = pr["box"][0]
    mx, my = pr["mu"][0]
    sx = sum(math.exp(-((x + 0.5 - mx) ** 2) / (2 * 1.375 ** 2)) for x in range(x0, x1 + 1))
    sy = sum(math.exp(-((y + 0.5 - my) ** 2) / (2 * 0.875 ** 2)) for y in range(y0, y1 + 1))
    img = gio.render(p, W, H, pos_mode=NORM, mode=gio.ALL_PAIRS)
    assert abs(img[0].sum() - sx * sy) < 1e-13


@pytest.mark.parametrize("tile", [1, 8, 13, 16])
def test_tiled_equals_all_pairs_bitwise(gio, tile):
    # north_star: tiled-versus-all-pairs equality (same terms, same order)
    for seed, (W, H, n) in enumerate([(64, 64, 256), (70, 45, 300)]):
        p = synth.init_params(seed, n)
        a = gio.render(p, W, H, tile=tile, mode=gio.ALL_PAIRS)
        b = gio.render(p, W, H, tile=tile, mode=gio.TILED)
        assert np.array_equal(a, b)
        # and the result does not depend on the tile size (R6 per-pixel predicate)
        c = gio.render(p, W, H, tile=16, mode=gio.ALL_PAIRS)
        assert np.array_equal(a, c)


def test_render_invariances(gio):
    # permutation (order-free Eq. 7), linearity in c',
    # empty region exactly 0
    p = synth.init_params(7, 200)
    a = gio.render(p, 48, 48)
    perm = np.random.default_rng(1).permutation(200)
    b = gio.render(p[perm], 48, 48)
    assert np.abs(a - b).max() < 1e-12
    q = p.copy(); q[:, 5:8] *= 2.0
    assert np.array_equal(gio.render(q, 48, 48), 2.0 * a)
    q = p.copy(); q[:, 5:8] = 0.0; q[0, 5:8] = (1, 2, 3)
    img = gio.render(q[:1], 48, 48)
    x0, x1, y0, y1 = gio.project(q[:1], 48, 48)["box"][0]
    mask = np.zeros((48, 48), bool); mask[y0:y1 + 1, x0:x1 + 1] = True
    assert np.all(img[:, ~mask] == 0.0) and np.all(img[:, mask] > 0.0)


def test_render_truncation_bound(gio):
    # |boxed - dense| <= |c'| exp(-4.5)-ish per Gaussian at k = 3
    p = one((0.1, -0.05), (0.6, 0.2, 0.3), (1.0, 1.0, 1.0))
    a = gio.render(p, 32, 32, pos_mode=NORM, mode=gio.ALL_PAIRS)
    d = gio.render(p, 32, 32, pos_mode=NORM, mode=gio.DENSE)
    assert np.abs(a - d).max() <= math.exp(-4.5) + 1e-12


# -------------------------------------------------------- loss / metrics
def test_mse_worked_example(gio):
    # x^ = 0.5, x = 0 -> loss 0.25, upstream 2 * 0.5 / count
    img = np.full((3, 1, 1), 0.5)
    loss, g = gio.mse(img, np.zeros((3, 1, 1), np.float32))
    assert loss == 0.25
    assert np.allclose(g, 1.0 / 3.0, rtol=0, atol=1e-16)


def test_psnr_worked_examples(gio):
    # identical -> capped 100 dB; MSE 0.01 -> 20 dB
    x = np.full(300, 0.5)
    assert gio.psnr(x, x.astype(np.float32)) == 100.0
    y = np.full(300, 0.75, np.float32)       # exact in fp32; MSE = 1/16 -> 12.0412 dB
    assert abs(gio.psnr(x, y) - 10 * math.log10(16)) < 1e-12
    y = np.full(300, 0.6, np.float32)
    assert abs(gio.psnr(x, y) - 20.0) < 1e-5


# ------------------------------------------------------------- Appendix A
def test_backward_worked_example(gio):
    # S:174 (App. A.1): Sigma = I, d = (1, 0), c' = (1,1,1),
    # upstream (1,0,0): dc'_r = e^-0.5; dL/dsigma = -e^-0.5;
    # dsigma/dSigma = -1/2 [[1,0],[0,0]] -> G = [[e^-.5/2, 0], [0, 0]]
    # -> dl1 = 2 g1 l1 = e^-0.5 (l1e = 1), dl2 = dl3 = 0;
    # dmu_pix = dL/dsigma * (-Sigma^-1 d) = (e^-0.5, 0); x (W/2 = 1) in norm mode
    p = one((-0.5, -0.5), (0.5, 0.0, 0.5), (1.0, 1.0, 1.0))   # mu = (0.5, 0.5) at 2x2
    g = np.zeros((3, 2, 2)); g[0, 0, 1] = 1.0                  # pixel (x=1, y=0)
    out = gio.backward(p, g, 2, 2, pos_mode=NORM)[0]
    e = math.exp(-0.5)
    want = [e, 0.0, e, 0.0, 0.0, e, 0.0, 0.0]
    assert np.allclose(out, want, rtol=1e-15, atol=1e-300)
    # d = 0 -> dc' = upstream, dmu = 0
    g = np.zeros((3, 2, 2)); g[:, 0, 0] = (0.25, 0.5, 0.75)
    out = gio.backward(p, g, 2, 2, pos_mode=NORM)[0]
    assert list(out[5:]) == [0.25, 0.5, 0.75] and out[0] == 0.0 and out[1] == 0.0


def test_chol_backward_worked_and_printed_formulas(gio):
    # G = I, l = (1,0,1) -> (2,0,2)
    assert list(gio.chol_backward([1, 0, 1], 1.0, 0.0, 1.0)) == [2.0, 0.0, 2.0]
    # dl1 and dl3 as printed; dl2 per R14 (P:627 misprint),
    # adjudicated by finite differences of <G, Sigma(l)> below
    G = np.array([0.3, -0.7, 1.1]); l = np.array([1.3, 0.4, 0.9])

    def f(l1, l2, l3):
        S = np.array([l1 * l1, l1 * l2, l2 * l2 + l3 * l3])
        return G[0] * S[0] + 2 * G[1] * S[1] + G[2] * S[2]   # Frobenius <G, Sigma>
    h = 1e-6
    fd = [(f(*(l + h * e)) - f(*(l - h * e))) / (2 * h) for e in np.eye(3)]
    got = gio.chol_backward(G, *l)
    assert np.allclose(got, fd, rtol=1e-8)
    paper_dl2 = 2 * G[1] * l[0] + G[1] * l[1]   # P:627 as printed
    assert abs(paper_dl2 - fd[1]) > 0.1           # the misprint is real


def _fd_grads(gio, p, target, mode, pos_mode=0, h=1e-3, idx=None):
    W, H = target.shape[2], target.shape[1]
    n = p.shape[0]
    out = np.zeros((n, 8))
    base_box = gio.project(p, W, H, pos_mode=pos_mode)["box"]
    for i in range(n) if idx is None else idx:
        for j in range(8):
            hp = np.float32(p[i, j] + h * max(1.0, abs(float(p[i, j]))))
            hm = np.float32(p[i, j] - h * max(1.0, abs(float(p[i, j]))))
            q1 = p.copy(); q1[i, j] = hp
            q2 = p.copy(); q2[i, j] = hm
            if mode != gio.DENSE:
                b1 = gio.project(q1, W, H, pos_mode=pos_mode)["box"]
                b2 = gio.project(q2, W, H, pos_mode=pos_mode)["box"]
                if not (np.array_equal(b1, base_box) and np.array_equal(b2, base_box)):
                    out[i, j] = np.nan      # truncated function jumps: not comparable
                    continue
            l1, _ = gio.mse(gio.render(q1, W, H, pos_mode=pos_mode, mode=mode), target)
            l2, _ = gio.mse(gio.render(q2, W, H, pos_mode=pos_mode, mode=mode), target)
            out[i, j] = (l1 - l2) / (float(hp) - float(hm))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_backward_matches_finite_differences_dense(gio, seed):
    # analytic grads of L2 o render vs central FD (dense: smooth)
    rng = np.random.default_rng(100 + seed)
    n, W, H = int(rng.integers(1, 6)), 12, 10
    p = synth.init_params(seed, n)
    p[:, 2:5] = rng.uniform(-0.2, 1.5, size=(n, 3)).astype(np.float32)
    p[:, 5:8] = rng.uniform(-1, 1, size=(n, 3)).astype(np.float32)
    target = rng.uniform(0, 1, size=(3, H, W)).astype(np.float32)
    for pos_mode in (0, 1):
        q = p.copy()
        if pos_mode == 1:
            q[:, 0:2] = np.tanh(q[:, 0:2])
        img = gio.render(q, W, H, pos_mode=pos_mode, mode=gio.DENSE)
        _, g = gio.mse(img, target)
        an = gio.backward(q, g, W, H, pos_mode=pos_mode, mode=gio.DENSE)
        fd = _fd_grads(gio, q, target, gio.DENSE, pos_mode=pos_mode, h=1e-4)
        err = np.abs(an - fd) / np.maximum(np.abs(fd), 1e-6)
        assert err.max() < 1e-5, (pos_mode, err.max())


def test_backward_matches_finite_differences_boxed(gio):
    # boxed (the truncated function actually optimised): FD where the
    # perturbation leaves every box unchanged
    rng = np.random.default_rng(7)
    n, W, H = 5, 14, 11
    p = synth.init_params(21, n)
    p[:, 5:8] = rng.uniform(-1, 1, size=(n, 3)).astype(np.float32)
    target = rng.uniform(0, 1, size=(3, H, W)).astype(np.float32)
    img = gio.render(p, W, H)
    _, g = gio.mse(img, target)
    an = gio.backward(p, g, W, H)
    fd = _fd_grads(gio, p, target, gio.ALL_PAIRS, h=1e-4)
    ok = ~np.isnan(fd)
    assert ok.sum() > 30
    err = np.abs(an[ok] - fd[ok]) / np.maximum(np.abs(fd[ok]), 1e-6)
    assert err.max() < 1e-5


def test_backward_zero_upstream_and_outside_box(gio):
    # zero upstream -> 0; upstream outside the box -> exactly 0
    p = one((0, 0), (0.5, 0.0, 0.5), (1, 1, 1))
    out = gio.backward(p, np.zeros((3, 40, 40)), 40, 40, pos_mode=NORM)
    assert np.all(out == 0.0)
    g = np.zeros((3, 40, 40)); g[:, 0, 0] = 1.0     # far outside the 6x6 box
    out = gio.backward(p, g, 40, 40, pos_mode=NORM)
    assert np.all(out == 0.0)


# ------------------------------------------------------------------- Adam
def test_lr_schedule(gio):
    # P:381 "initial learning rate of 1e-3, halved every 20000 steps" (R17)
    assert gio.lr_at(1) == 1e-3 and gio.lr_at(20000) == 1e-3
    assert gio.lr_at(20001) == 5e-4 and gio.lr_at(40000) == 5e-4
    assert gio.lr_at(40001) == 2.5e-4 and gio.lr_at(50000) == 2.5e-4


def test_adam_closed_forms(gio):
    rng = np.random.default_rng(3)
    p = rng.normal(size=1000).astype(np.float32)
    g = rng.normal(size=1000).astype(np.float32)
    z = np.zeros(1000, np.float32)
    lr, eps = 1e-3, 1e-8
    # step 1 from m = v = 0: bias-corrected m^ = g, v^ = g^2 ->
    # p' = p - lr g / (|g| + eps)
    po, mo, vo = gio.adam(p, g, z, z, 1, lr)
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    gd = g.astype(np.float64)
    want = p.astype(np.float64) - float(np.float32(lr)) * gd / (np.abs(gd) + float(np.float32(eps)))
    assert np.allclose(po, want, rtol=1e-13, atol=1e-15)
    assert np.allclose(mo, (1 - b1) * gd, rtol=1e-14)
    assert np.allclose(vo, (1 - b2) * gd ** 2, rtol=1e-14)
    # S:251 zero gradients from step 1 -> p unchanged
    po, mo, vo = gio.adam(p, z, z, z, 1, lr)
    assert np.array_equal(po, p.astype(np.float64)) and not mo.any() and not vo.any()
    # a constant gradient keeps m^ = g and v^ = g^2 at every step t:
    # m_t = (1 - b1^t) g, v_t = (1 - b2^t) g^2 -> the same step as at t = 1
    for t in (2, 7, 30):
        m = ((1 - b1 ** (t - 1)) * gd).astype(np.float32)
        v = ((1 - b2 ** (t - 1)) * gd ** 2).astype(np.float32)
        po, mo, vo = gio.adam(p, g, m, v, t, lr)
        assert np.allclose(po, want, rtol=1e-6, atol=1e-9)


# ------------------------------------------------------------ codec decode
def test_half_decoding(gio):
    # IEEE binary16 bit patterns ("16-bit float precision")
    cases = {0x3C00: 1.0, 0xB800: -0.5, 0x0001: 2.0 ** -24, 0x7BFF: 65504.0,
             0x3555: 0.333251953125, 0x0000: 0.0, 0x8000: -0.0, 0x0400: 2.0 ** -14}
    for bits, val in cases.items():
        assert gio.half_to_double(bits) == val


def test_decode_hand_assembled_record(gio):
    # One 56-bit record written out by hand from SPEC.md:404 (MSB first):
    # x = 0x3C00 (1.0), y = 0xB800 (-0.5), codes 44, 0, 63 (6 bits), indices 3, 5
    bits = ("0011110000000000" "1011100000000000" "101100" "000000" "111111" "011" "101")
    assert len(bits) == 56
    data = np.frombuffer(int(bits, 2).to_bytes(7, "big"), np.uint8)
    gamma = np.array([0.1, 0.25, 0.5], np.float32)
    beta = np.array([-3.2, 1.0, -2.0], np.float32)
    books = np.zeros((2, 8, 3), np.float32)
    books[0, 3] = (0.5, 0.25, -1.0)
    books[1, 5] = (0.125, 0.5, 0.75)
    out = gio.vq_decode(data, 1, gamma, beta, books)[0]
    assert out[0] == 1.0 and out[1] == -0.5
    # b = 6, gamma = 0.1, beta = -3.2, code 44 -> 1.2 (Eq. 8)
    assert abs(out[2] - 1.2) < 1e-6
    assert out[3] == np.float32(1.0) and out[4] == np.float32(63 * 0.5 - 2.0)
    # Eq. 9: c' = C1[3] + C2[5]
    assert list(out[5:]) == [0.625, 0.75, -0.25]
    # and the shared input generator packs the same bytes
    pk = synth.pack_records(np.array([[0x3C00, 0xB800]], np.uint16), np.array([[44, 0, 63]]),
                            np.array([[3, 5]]), 6, 8)
    assert bytes(pk) == bytes(data)


def test_decode_rvq_exact_codeword_and_size(gio):
    # c' equals C1[3] and C2[0] = 0 -> exact reconstruction
    books = np.zeros((2, 8, 3), np.float32)
    books[0, 3] = (0.3, -0.2, 0.9)
    pk = synth.pack_records(np.array([[0, 0]], np.uint16), np.array([[0, 0, 0]]),
                            np.array([[3, 0]]), 6, 8)
    out = gio.vq_decode(pk, 1, np.ones(3, np.float32), np.zeros(3, np.float32), books)[0]
    assert np.array_equal(out[5:], books[0, 3])
    # 56 bits per Gaussian at b = 6, M = 2, B = 8
    assert synth.record_bits(6, 2, 8) == 56
    data, ga, be, bo = synth.payload(0, 30000)
    assert data.size == 30000 * 7
    # a record straddling byte boundaries (b = 8 -> 62-bit records) round-trips
    pos = np.array([[0x3C00, 0x0001], [0xB800, 0x7BFF], [0x1234, 0x4321]], np.uint16)
    codes = np.array([[255, 0, 17], [1, 2, 3], [200, 100, 50]])
    idx = np.array([[7, 1], [0, 6], [3, 3]])
    pk = synth.pack_records(pos, codes, idx, 8, 8)
    assert pk.size == (3 * 62 + 7) // 8
    books = np.arange(48, dtype=np.float32).reshape(2, 8, 3)
    out = gio.vq_decode(pk, 3, np.ones(3, np.float32), np.zeros(3, np.float32), books, bits=8)
    assert np.array_equal(out[:, 2:5], codes.astype(np.float32))
    assert np.array_equal(out[:, 5:], books[0, idx[:, 0]] + books[1, idx[:, 1]])
    assert out[1, 1] == 65504.0 and out[0, 1] == 2.0 ** -24


# ------------------------------------------------------------------- Adan
def test_adan_closed_forms(gio):
    # NEXT-1 (P:381 Adan; update rule of the cited Adan reference, R28)
    rng = np.random.default_rng(9)
    p = rng.normal(size=500).astype(np.float32)
    g = rng.normal(size=500).astype(np.float32)
    z = np.zeros(500, np.float32)
    lr = 1e-3
    b1, b2, b3 = (float(np.float32(x)) for x in (0.98, 0.92, 0.99))
    gd = g.astype(np.float64)
    # zero gradients from step 1 -> unchanged
    po, mo, vo, no = gio.adan(p, z, z, z, z, z, 1, lr)
    assert np.array_equal(po, p.astype(np.float64)) and not mo.any() and not no.any()
    # constant gradient g from step 1: d = 0, m^ = g, n^ = g^2 -> p - lr g/(|g|+eps)
    want = p.astype(np.float64) - float(np.float32(lr)) * gd / (np.abs(gd) + float(np.float32(1e-8)))
    for t in (1, 2, 9):
        m = ((1 - b1 ** (t - 1)) * gd).astype(np.float32)
        n = ((1 - b3 ** (t - 1)) * gd ** 2).astype(np.float32)
        po, mo, vo, no = gio.adan(p, g, m, z, n, g if t > 1 else z, t, lr)
        assert np.allclose(po, want, rtol=1e-6, atol=1e-9)
        assert not vo.any()
    # the gradient-difference term: g1 = 0 then g2 = a gives, by hand,
    # step = lr sign(a) [1/(1+b1) + b2/(1+b2)] (1+b3)^(1/2) / (1+b2)  (eps -> 0)
    a = np.array([0.7, -2.0, 1e-3], np.float32)
    z3 = np.zeros(3, np.float32)
    p3 = np.zeros(3, np.float32)
    _, m1, v1, n1 = gio.adan(p3, z3, z3, z3, z3, z3, 1, lr, eps=0.0)
    po, _, _, _ = gio.adan(p3, a, m1.astype(np.float32), v1.astype(np.float32),
                           n1.astype(np.float32), z3, 2, lr, eps=0.0)
    k = (1 / (1 + b1) + b2 / (1 + b2)) * math.sqrt(1 + b3) / (1 + b2)
    assert abs(k - 0.7231) < 1e-3
    assert np.allclose(po, -float(np.float32(lr)) * np.sign(a) * k, rtol=1e-12)
    # f(x) = x^2 from x0 = 1, lr = 1e-2, 500 steps -> |x| < 1e-2
    x = np.ones(1, np.float32)
    st = [np.zeros(1, np.float32) for _ in range(4)]      # m, v, n, g_prev
    for t in range(1, 501):
        gg = (2 * x).astype(np.float32)
        xo, mo, vo, no = gio.adan(x, gg, st[0], st[1], st[2], st[3], t, 1e-2)
        x = xo.astype(np.float32)
        st = [mo.astype(np.float32), vo.astype(np.float32), no.astype(np.float32), gg]
    assert abs(float(x[0])) < 1e-2


# ---------------------------------------------- NEXT-3: rotation-scaling (RS)
RS = 2   # pos_mode bit: params[2:5] = (theta, s1, s2), Sigma = (RS)(RS)^T (Eq. 2-3)


def test_rs_covariance_worked_examples(gio):
    # RS raw (theta = 0, s1 = 0.5, s2 = 1.5) -> Sigma = [[1,0],[0,4]]
    pr = gio.project(one((0, 0), (0.0, 0.5, 1.5), (1, 1, 1)), 64, 64, pos_mode=NORM | RS)
    assert np.array_equal(pr["sigma"][0], [1.0, 0.0, 4.0])
    # a quarter turn swaps the axes (Eq. 3 R(theta))
    th = np.float32(np.pi / 2)
    pr = gio.project(one((0, 0), (th, 0.5, 1.5), (1, 1, 1)), 64, 64, pos_mode=NORM | RS)
    assert np.allclose(pr["sigma"][0], [4.0, 0.0, 1.0], atol=1e-6)
    # eigen-structure: det = (s1 s2)^2, trace = s1^2 + s2^2 for any theta
    rng = np.random.default_rng(4)
    for _ in range(50):
        t, a, b = rng.uniform(-4, 4), rng.uniform(0.1, 3), rng.uniform(0.1, 3)
        p = one((0, 0), (t, a - 0.5, b - 0.5), (1, 1, 1))
        S = gio.project(p, 64, 64, pos_mode=NORM | RS)["sigma"][0]
        a32, b32 = float(np.float32(a - 0.5)) + 0.5, float(np.float32(b - 0.5)) + 0.5
        assert abs(S[0] * S[2] - S[1] ** 2 - (a32 * b32) ** 2) < 1e-9 * (a32 * b32) ** 2
        assert abs(S[0] + S[2] - a32 ** 2 - b32 ** 2) < 1e-12 * (a32 ** 2 + b32 ** 2)


def test_rs_box_and_equivalence_with_cholesky(gio):
    # theta = 0, s = (3.5, 0.5) -> Sigma = diag(16, 1): half extents (12, 3)
    pr = gio.project(one((0, 0), (0.0, 3.5, 0.5), (1, 1, 1)), 101, 101, pos_mode=NORM | RS)
    assert list(pr["box"][0]) == [38, 62, 47, 53]
    # the same Sigma through the Cholesky parameterisation renders the same
    # image (both factorisations express the same Sigma)
    rng = np.random.default_rng(8)
    for _ in range(20):
        t, a, b = rng.uniform(-3, 3), rng.uniform(0.6, 2.5), rng.uniform(0.6, 2.5)
        prs = one((0.05, -0.03), (t, a - 0.5, b - 0.5), (0.7, -0.2, 0.4))
        S = gio.project(prs, 48, 40, pos_mode=NORM | RS)["sigma"][0]
        l1 = np.sqrt(S[0]); l2 = S[1] / l1; l3 = np.sqrt(S[2] - l2 * l2)
        pch = one((0.05, -0.03), (l1 - 0.5, l2, l3 - 0.5), (0.7, -0.2, 0.4))
        a_img = gio.render(prs, 48, 40, pos_mode=NORM | RS, mode=gio.DENSE)
        b_img = gio.render(pch, 48, 40, pos_mode=NORM, mode=gio.DENSE)
        assert np.abs(a_img - b_img).max() < 2e-6


def test_rs_backward_worked_examples(gio):
    # theta = 0 and G diagonal -> dtheta = 0;
    # G = [[1,0],[0,0]], theta = 0, s = (1,1) -> ds1 = 2, ds2 = 0
    d = gio.rs_backward([0.7, 0.0, -1.3], 0.0, 1.2, 0.8)
    assert abs(d[0]) < 1e-15
    assert list(gio.rs_backward([1.0, 0.0, 0.0], 0.0, 1.0, 1.0)) == [0.0, 2.0, 0.0]
    # FD of <G, Sigma(theta, s1, s2)> (Frobenius, symmetric G)
    G = np.array([0.4, -0.9, 0.25]); x = np.array([0.7, 1.3, 0.6])

    def f(t, a, b):
        c, s = np.cos(t), np.sin(t)
        R = np.array([[c, -s], [s, c]])
        Sg = R @ np.diag([a * a, b * b]) @ R.T
        return G[0] * Sg[0, 0] + 2 * G[1] * Sg[0, 1] + G[2] * Sg[1, 1]
    h = 1e-6
    fd = [(f(*(x + h * e)) - f(*(x - h * e))) / (2 * h) for e in np.eye(3)]
    assert np.allclose(gio.rs_backward(G, *x), fd, rtol=1e-8)


@pytest.mark.parametrize("seed", range(3))
def test_rs_backward_matches_finite_differences(gio, seed):
    rng = np.random.default_rng(300 + seed)
    n, W, H = 3, 12, 10
    p = synth.init_params(seed, n)
    p[:, 2] = rng.uniform(-3, 3, size=n).astype(np.float32)          # theta
    p[:, 3:5] = rng.uniform(0.3, 1.5, size=(n, 2)).astype(np.float32)  # s1, s2
    p[:, 5:8] = rng.uniform(-1, 1, size=(n, 3)).astype(np.float32)
    target = rng.uniform(0, 1, size=(3, H, W)).astype(np.float32)
    img = gio.render(p, W, H, pos_mode=RS, mode=gio.DENSE)
    _, g = gio.mse(img, target)
    an = gio.backward(p, g, W, H, pos_mode=RS, mode=gio.DENSE)
    fd = _fd_grads(gio, p, target, gio.DENSE, pos_mode=RS, h=1e-4)
    err = np.abs(an - fd) / np.maximum(np.abs(fd), 1e-6)
    assert err.max() < 1e-5, err.max()
