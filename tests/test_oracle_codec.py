"""Pins for the oracle's NEXT-2 encoder (``-m "not gpu"``): IEEE binary16
rounding against numpy's independent implementation, the worked Eq. 8
examples of SPEC, the Eq. 9 greedy RVQ against per-stage brute
force, and the encode -> pack -> decode round trip through the (separately
pinned) decoder.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import numpy as np

import synth


def test_float_to_half_matches_numpy(gio):
    # IEEE 754 binary16, round to nearest even, against numpy's
    # conversion: normals, subnormals, exact ties, overflow, signed zero
    rng = np.random.default_rng(1)
    xs = np.concatenate([
        rng.uniform(-1, 1, 20000), rng.normal(0, 1e-5, 5000), rng.normal(0, 3e4, 2000),
        np.ldexp(rng.integers(1, 2048, 2000).astype(np.float64) + 0.5, -24 - 10),   # ties
        (1.0 + (np.arange(1, 1024) + 0.5) / 1024.0),                                 # ties
        [0.0, -0.0, 65504.0, 65519.0, 65520.0, 1e9, -1e9, 2.0 ** -24, 2.0 ** -25, 2.0 ** -26,
         3 * 2.0 ** -26, 6.1e-5],
    ]).astype(np.float32)
    with np.errstate(over="ignore"):
        ref = xs.astype(np.float16).view(np.uint16).astype(np.int64)
    got = np.array([gio.float_to_half(x) for x in xs], np.int64)
    assert np.array_equal(got, ref)


def _enc(gio, p, gamma=(0.1, 0.1, 0.1), beta=(-3.2, -3.2, -3.2), books=None, bits=6, stages=2,
         codebook=8, pos_mode=1):
    if books is None:
        books = np.zeros((stages, codebook, 3), np.float32)
    return gio.vq_encode(p, np.float32(gamma), np.float32(beta), np.float32(books), bits, stages,
                         codebook, pos_mode)


def test_quantise_worked_examples(gio):
    # S:318-320 (Eq. 8): b = 6, gamma 0.1, beta -3.2: l = 1.234 -> 44,
    # dequant 1.2; l = beta -> 0; far above -> 63 (clamp); far below -> 0
    p = np.array([[0, 0, 1.234, -3.2, 50.0, 0, 0, 0],
                  [0, 0, -99.0, 1.234, -3.2, 0, 0, 0]], np.float32)
    e = _enc(gio, p)
    assert e["codes"].tolist() == [[44, 0, 63], [0, 44, 0]]
    assert np.allclose(e["eff"][0, 2:5], [1.2, -3.2, 63 * 0.1 - 3.2], atol=1e-6)
    # exact ties round half to even (reading R30, as torch.round): x = 44.5
    # -> 44, 45.5 -> 46 (gamma 0.5, beta 0)
    t = np.zeros((1, 8), np.float32)
    t[0, 2:5] = [22.25, 22.75, 0.25]
    e = _enc(gio, t, gamma=(0.5, 0.5, 0.5), beta=(0.0, 0.0, 0.0))
    assert e["codes"].tolist() == [[44, 46, 0]]
    # in range: |dequant - l| <= gamma / 2 (SPEC invariant)
    rng = np.random.default_rng(2)
    q = np.zeros((4000, 8), np.float32)
    q[:, 2:5] = rng.uniform(-3.2, 6.3 - 3.2, (4000, 3))
    e = _enc(gio, q)
    assert np.all(np.abs(e["eff"][:, 2:5] - q[:, 2:5]) <= 0.05 + 1e-6)
    assert e["codes"].max() <= 63


def test_position_is_fp16_of_tanh(gio):
    # positions are stored as binary16 of the post-tanh u (R19)
    rng = np.random.default_rng(3)
    p = np.zeros((500, 8), np.float32)
    p[:, :2] = rng.normal(0, 1.5, (500, 2))
    e = _enc(gio, p, pos_mode=0)
    u = np.tanh(p[:, :2].astype(np.float64)).astype(np.float32)
    assert np.array_equal(e["pos16"].astype(np.uint16), u.astype(np.float16).view(np.uint16))
    assert np.array_equal(e["eff"][:, :2], u.astype(np.float16).astype(np.float32))


def test_rvq_examples_and_brute_force(gio):
    # c' equal to C1[3] with C2[0] = 0 -> indices (3, 0), exact
    books = np.zeros((2, 8, 3), np.float32)
    books[0] = np.arange(24, dtype=np.float32).reshape(8, 3) / 10
    books[1, 1:] = 0.5
    p = np.zeros((1, 8), np.float32)
    p[0, 5:] = books[0, 3]
    e = _enc(gio, p, books=books)
    assert e["idx"].tolist() == [[3, 0]] and np.array_equal(e["eff"][0, 5:], books[0, 3])
    # M = 1, B = 2, {0, 1}: (0.9, 0.9, 0.9) -> 1
    b1 = np.array([[[0, 0, 0], [1, 1, 1]]], np.float32)
    p[0, 5:] = 0.9
    e = _enc(gio, p, books=b1, stages=1, codebook=2)
    assert e["idx"].tolist() == [[1]] and np.array_equal(e["eff"][0, 5:], [1, 1, 1])
    # random: each stage's index is the brute-force (fp64) nearest codeword to
    # the stage residual, whose energy never exceeds that of any other choice
    rng = np.random.default_rng(4)
    books = rng.normal(0, 0.5, (2, 8, 3)).astype(np.float32)
    p = np.zeros((3000, 8), np.float32)
    p[:, 5:] = rng.normal(0, 0.6, (3000, 3))
    e = _enc(gio, p, books=books)
    c = p[:, 5:].astype(np.float64)
    chat = np.zeros_like(c)
    for m in range(2):
        r = c - chat
        d = ((books[m][None, :, :].astype(np.float64) - r[:, None, :]) ** 2).sum(-1)
        srt = np.sort(d, axis=1)
        clear = srt[:, 1] - srt[:, 0] > 1e-5          # no near-ties in fp32
        assert np.array_equal(e["idx"][clear, m], d.argmin(1)[clear])
        chat = chat + books[m][e["idx"][:, m]]
    assert np.allclose(e["eff"][:, 5:], chat, atol=1e-6)


def test_encode_pack_decode_round_trip(gio):
    # the packed records (S:404 layout, synth packer pinned separately) decode
    # to exactly the encoder's effective parameters
    rng = np.random.default_rng(6)
    n = 777
    p = synth.fitted_params(6, n)
    gamma = np.float32([0.05, 0.04, 0.05])
    beta = np.float32([-1.0, -1.2, -1.0])
    books = rng.normal(0, 0.3, (2, 8, 3)).astype(np.float32)
    e = gio.vq_encode(p, gamma, beta, books)
    data = synth.pack_records(e["pos16"].astype(np.uint16), e["codes"], e["idx"], 6, 8)
    dec = gio.vq_decode(data, n, gamma, beta, books)
    assert np.array_equal(dec.view(np.uint32), e["eff"].view(np.uint32))


def test_kmeans_pins(gio):
    # P:307 K-means init (5 Lloyd iterations).
    # N = B distinct points, initialised on them -> each its own centroid
    rng = np.random.default_rng(7)
    pts = rng.normal(0, 1, (8, 3)).astype(np.float32)
    cent, asg, d = gio.kmeans(pts, pts[::-1], iters=5)
    assert np.array_equal(np.sort(asg), np.arange(8)) and d == 0.0
    assert np.array_equal(cent[asg], pts)
    # two well-separated blobs, B = 2: centroids = blob means (closed form)
    a = rng.normal(0, 0.05, (500, 3)) + [1, 0, 0]
    b = rng.normal(0, 0.05, (300, 3)) + [-1, 0.5, 0]
    pts = np.concatenate([a, b]).astype(np.float32)
    cent, asg, _ = gio.kmeans(pts, np.float32([[0.5, 0, 0], [-0.5, 0, 0]]), iters=5)
    assert np.allclose(cent[0], pts[:500].astype(np.float64).mean(0), atol=1e-6)
    assert np.allclose(cent[1], pts[500:].astype(np.float64).mean(0), atol=1e-6)
    assert asg[:500].max() == 0 and asg[500:].min() == 1
    # Lloyd monotonicity: the distortion never increases (fp64, numpy)
    pts = rng.normal(0, 0.4, (3000, 3)).astype(np.float32)
    cent = pts[:8].copy()
    prev = np.inf
    for _ in range(6):
        cent, asg, d = gio.kmeans(pts, cent, iters=1)
        ref = ((pts.astype(np.float64) - cent.astype(np.float64)[asg]) ** 2).sum()
        assert d <= prev + 1e-9
        prev = ref            # distortion w.r.t. the updated centroids bounds the next one
    # an empty cluster keeps its centroid (reading R31)
    cent, asg, _ = gio.kmeans(pts, np.concatenate([pts[:7], [[50, 50, 50]]]).astype(np.float32), 1)
    assert np.array_equal(cent[7], [50, 50, 50]) and 7 not in asg


def _qat_state(n, rng, stages=2, codebook=8):
    books = rng.normal(0, 0.3, (stages, codebook, 3)).astype(np.float32)
    return dict(m=np.zeros((n, 8), np.float32), v=np.zeros((n, 8), np.float32),
                gamma=np.float32([0.05, 0.04, 0.05]), beta=np.float32([-1.0, -1.2, -1.0]),
                qm=np.zeros(6, np.float32), qv=np.zeros(6, np.float32), books=books,
                ema_n=np.ones((stages, codebook), np.float32), ema_s=books.copy())


def test_qat_straight_through_gradients_fd(gio):
    # Reading R32 (LSQ+ straight-through estimator): the oracle's gradients
    # w.r.t. raw positions, l, gamma and beta equal central finite
    # differences of L_rec through the quantiser with its rounding offsets
    # frozen at the base point (dense render: no box discontinuities)
    rng = np.random.default_rng(11)
    W = H = 24
    n = 40
    p = synth.fitted_params(11, n)
    p[:, 2:5] = rng.uniform(-1.2, 2.0, (n, 3)).astype(np.float32)   # some clamp on both sides
    t = synth.image(11, W, H)
    st = _qat_state(n, rng)
    out = gio.qat_step(p, t, st, 1, 1e-4, mode=gio.DENSE)
    enc = out["enc"]
    gamma, beta = st["gamma"].astype(np.float64), st["beta"].astype(np.float64)
    qmax = 63.0
    x0 = ((p[:, 2:5] - st["beta"]) / st["gamma"]).astype(np.float32).astype(np.float64)
    inside = (x0 >= 0) & (x0 <= qmax)
    delta = enc["codes"] - x0                         # frozen rounding offsets
    u0 = np.tanh(p[:, :2].astype(np.float64))
    du = enc["eff"][:, :2] - u0                        # frozen fp16 offsets

    def loss(raw_xy, l, g, b):
        e = np.array(enc["eff"], np.float64)
        e[:, :2] = np.tanh(raw_xy) + du
        x = (l - b) / g
        e[:, 2:5] = np.where(inside, g * (x + delta) + b, g * enc["codes"] + b)
        img = gio.render(e.astype(np.float64).astype(np.float32), W, H, pos_mode=gio.POS_NORMALIZED,
                         mode=gio.DENSE)
        return float(((img - t) ** 2).mean())

    raw = p[:, :2].astype(np.float64)
    l = p[:, 2:5].astype(np.float64)
    # Richardson-extrapolated central differences (params reach the render in
    # fp32, which bounds how small h can be); 1e-2 still separates every
    # plausible slip (sign, code vs code - x, inside/outside swapped: O(1))
    def rich(f, h):
        d1 = (f(h) - f(-h)) / (2 * h)
        d2 = (f(h / 2) - f(-h / 2)) / h
        return (4 * d2 - d1) / 3

    for j in range(3):
        e = np.zeros(3); e[j] = 1.0
        fd_g = rich(lambda s: loss(raw, l, gamma + s * e, beta), 4e-4)
        fd_b = rich(lambda s: loss(raw, l, gamma, beta + s * e), 4e-4)
        assert abs(fd_g - out["dgamma"][j]) <= 1e-2 * abs(fd_g) + 1e-7, (j, fd_g, out["dgamma"][j])
        assert abs(fd_b - out["dbeta"][j]) <= 1e-2 * abs(fd_b) + 1e-7, (j, fd_b, out["dbeta"][j])
    h = 1e-4
    for (i, j) in [(0, 0), (3, 1), (7, 2), (11, 0)]:
        d = np.zeros_like(l); d[i, j] = h
        fd = (loss(raw, l + d, gamma, beta) - loss(raw, l - d, gamma, beta)) / (2 * h)
        assert abs(fd - out["grads"][i, 2 + j]) <= 2e-3 * abs(fd) + 1e-7
        d = np.zeros_like(raw); d[i, j % 2] = h
        fd = (loss(raw + d, l, gamma, beta) - loss(raw - d, l, gamma, beta)) / (2 * h)
        assert abs(fd - out["grads"][i, j % 2]) <= 2e-3 * abs(fd) + 1e-7


def test_qat_ema_and_commitment_pins(gio):
    # SPEC ema_update and Eq. 10 commitment loss
    rng = np.random.default_rng(12)
    W = H = 16
    n = 64
    p = synth.init_params(12, n)
    t = synth.image(12, W, H)
    st = _qat_state(n, rng)
    # exact codewords (stage-2 codeword 0 = 0): L_c = 0 and the books only
    # move by the EMA of themselves
    st["books"][1, 0] = 0.0
    st["ema_s"] = st["books"].copy()
    pick = rng.integers(0, 8, n)
    p[:, 5:8] = st["books"][0][pick]
    out = gio.qat_step(p, t, st, 1, 1e-4, mode=gio.DENSE)
    assert out["l_c"] == 0.0
    assert np.array_equal(out["enc"]["idx"][:, 0], pick)
    # decay 0: each used codeword becomes the mean of its residuals, unused
    # codewords are unchanged (stationary in one step)
    p2 = synth.init_params(13, n)
    out = gio.qat_step(p2, t, st, 1, 1e-4, decay=0.0, mode=gio.DENSE)
    idx = out["enc"]["idx"][:, 0]
    for kk in range(8):
        sel = idx == kk
        if sel.any():
            assert np.allclose(out["state"]["books"][0, kk], p2[sel, 5:8].astype(np.float64).mean(0),
                               atol=1e-6)
        else:
            assert np.array_equal(out["state"]["books"][0, kk], st["books"][0, kk])
    # N = 1, B = 1, M = 1: c' = (1, 0, 0), C = 0 -> L_c = 1
    one = np.zeros((1, 8), np.float32); one[0, 5] = 1.0
    s1 = _qat_state(1, rng, stages=1, codebook=1)
    s1["books"][:] = 0.0
    s1["ema_s"] = s1["books"].copy()
    out = gio.qat_step(one, t, s1, 1, 1e-4, stages=1, codebook=1, mode=gio.DENSE)
    assert out["l_c"] == 1.0
