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
