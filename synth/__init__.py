"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module holds NONE of the method's arithmetic (no projection, binning,
rendering, gradients, optimiser or decode).  It only draws inputs, so that the
GPU path (``paper_2403_08551_b200``) and the CPU oracle (``oracle``) read
identical fp32 bits.  Recipes:

* ``image``: "Kodak-shaped" natural-image proxy -- per-channel 1/f (pink)
  noise mixed by a fixed channel-correlation matrix, plus 40 random filled
  disks / convex polygons (sharp edges), affine-mapped to [0.02, 0.98].
  Planar fp32 ``[3][H][W]``.
* ``init_params``: the paper's initialisation (App. C):
  position logits mu = atanh(rand*2-1), Cholesky factors and weighted colours
  "initialized using a uniform distribution" -- U[0,1) (reading R5).
  AoS fp32 ``[N][8]`` = {mux, muy, l1, l2, l3, c'r, c'g, c'b}.
* ``fitted_params``: proxy for a post-fit cloud (no trained weights exist
  here): same positions, Gaussians ~3x larger, small signed colours.
* ``payload``: random codec records (fp16 positions, b-bit Cholesky codes,
  M RVQ indices) packed MSB-first per SPEC.md:404, plus random gamma/beta and
  codebooks.  Packing is the bitstream *format*, not the decode arithmetic.
"""
from __future__ import annotations

import numpy as np

PARAMS_PER_GAUSSIAN = 8  # PAPER.md:232 "a total of 8 parameters"


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.PCG64(int(seed)))


def image(seed: int, width: int, height: int) -> np.ndarray:
    """Planar fp32 [3][H][W] natural-image proxy in [0.02, 0.98]."""
    rng = _rng(10_000 + seed)
    h, w = int(height), int(width)
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.rfftfreq(w)[None, :]
    f = np.sqrt(fx * fx + fy * fy)
    f[0, 0] = 1.0
    amp = 1.0 / f
    amp[0, 0] = 0.0
    chans = []
    for _ in range(3):
        phase = rng.uniform(0.0, 2.0 * np.pi, size=amp.shape)
        spec = amp * np.exp(1j * phase)
        field = np.fft.irfft2(spec, s=(h, w))
        field = (field - field.mean()) / (field.std() + 1e-12)
        chans.append(field)
    noise = np.stack(chans, 0)
    mix = np.array([[1.0, 0.6, 0.4], [0.6, 1.0, 0.6], [0.4, 0.6, 1.0]])
    img = np.einsum("ij,jhw->ihw", mix, noise) * 0.12 + 0.5
    yy, xx = np.mgrid[0:h, 0:w]
    yy = yy + 0.5
    xx = xx + 0.5
    for s in range(40):
        col = rng.uniform(0.0, 1.0, size=3)
        cx, cy = rng.uniform(0, w), rng.uniform(0, h)
        rad = rng.uniform(0.02, 0.15) * min(w, h)
        if s % 2 == 0:
            mask = (xx - cx) ** 2 + (yy - cy) ** 2 <= rad * rad
        else:
            k = int(rng.integers(3, 7))
            ang = np.sort(rng.uniform(0, 2 * np.pi, size=k))
            px, py = cx + rad * np.cos(ang), cy + rad * np.sin(ang)
            mask = np.ones((h, w), bool)
            for i in range(k):
                x0, y0 = px[i], py[i]
                x1, y1 = px[(i + 1) % k], py[(i + 1) % k]
                mask &= (x1 - x0) * (yy - y0) - (y1 - y0) * (xx - x0) >= 0
        img[:, mask] = col[:, None] * 0.85 + img[:, mask] * 0.15
    lo, hi = img.min(), img.max()
    img = 0.02 + 0.96 * (img - lo) / max(hi - lo, 1e-12)
    return np.clip(img, 0.02, 0.98).astype(np.float32)


def init_params(seed: int, n: int) -> np.ndarray:
    """Paper init (App. C; reading R5). fp64 draws -> fp32."""
    rng = _rng(20_000 + seed)
    n = int(n)
    u = rng.uniform(0.0, 1.0, size=(n, 2))
    # keep atanh finite: rand*2-1 in [-1+2^-24, 1-2^-24] (a 0-probability
    # edge of the paper's recipe; reading R5)
    t = np.clip(u * 2.0 - 1.0, -1.0 + 2.0**-24, 1.0 - 2.0**-24)
    mu = np.arctanh(t)
    chol = rng.uniform(0.0, 1.0, size=(n, 3))
    col = rng.uniform(0.0, 1.0, size=(n, 3))
    p = np.concatenate([mu, chol, col], axis=1)
    return np.ascontiguousarray(p.astype(np.float32))


def fitted_params(seed: int, n: int) -> np.ndarray:
    """Post-fit proxy: same position law, Gaussians ~3x larger (l_eff in
    [1.5,4.5) on the diagonal, |l2| < 1.5), signed colours U[-0.1, 0.2)."""
    rng = _rng(30_000 + seed)
    n = int(n)
    u = rng.uniform(0.0, 1.0, size=(n, 2))
    t = np.clip(u * 2.0 - 1.0, -1.0 + 2.0**-24, 1.0 - 2.0**-24)
    mu = np.arctanh(t)
    l1 = 3.0 * rng.uniform(0.0, 1.0, size=n) + 1.0      # l1 + 0.5 in [1.5, 4.5)
    l2 = 3.0 * rng.uniform(-0.5, 0.5, size=n)
    l3 = 3.0 * rng.uniform(0.0, 1.0, size=n) + 1.0
    col = rng.uniform(-0.1, 0.2, size=(n, 3))
    p = np.concatenate([mu, np.stack([l1, l2, l3], 1), col], axis=1)
    return np.ascontiguousarray(p.astype(np.float32))


def clustered_params(seed: int, n: int, width: int, height: int, clusters: int = 8,
                     frac: float = 0.5, radius_px: float = 6.0) -> np.ndarray:
    """A clustered cloud (dense features, as fitted images concentrate
    Gaussians on edges and detail): the paper's init, except that a fraction
    `frac` of the Gaussians is moved into `clusters` discs of `radius_px`
    pixels.  Positions are drawn in normalised image coordinates and stored
    as logits, u = tanh(mu_raw) (App. C)."""
    rng = _rng(50_000 + seed)
    p = init_params(seed, n).astype(np.float64)
    m = int(round(frac * n))
    cx = rng.uniform(0.1, 0.9, size=clusters) * width
    cy = rng.uniform(0.1, 0.9, size=clusters) * height
    k = rng.integers(0, clusters, size=m)
    r = radius_px * np.sqrt(rng.uniform(0.0, 1.0, size=m))
    a = rng.uniform(0.0, 2.0 * np.pi, size=m)
    x = np.clip(cx[k] + r * np.cos(a), 0.0, width)
    y = np.clip(cy[k] + r * np.sin(a), 0.0, height)
    u = np.stack([2.0 * x / width - 1.0, 2.0 * y / height - 1.0], 1)
    u = np.clip(u, -1.0 + 2.0**-24, 1.0 - 2.0**-24)
    p[:m, 0:2] = np.arctanh(u)
    return np.ascontiguousarray(p.astype(np.float32))


def target_images(seed: int, batch: int, width: int, height: int) -> np.ndarray:
    return np.stack([image(seed + b, width, height) for b in range(int(batch))], 0)


def batch_params(seed: int, batch: int, n: int, fitted: bool = False) -> np.ndarray:
    gen = fitted_params if fitted else init_params
    return np.stack([gen(seed + b, n) for b in range(int(batch))], 0)


def record_bits(bits: int, stages: int, codebook: int) -> int:
    """Bits per record: 32 + 3b + M*ceil(log2 B)."""
    return 32 + 3 * int(bits) + int(stages) * index_bits(codebook)


def index_bits(codebook: int) -> int:
    return max(1, int(np.ceil(np.log2(int(codebook)))))


def pack_records(pos16: np.ndarray, codes: np.ndarray, idx: np.ndarray,
                 bits: int, codebook: int) -> np.ndarray:
    """MSB-first concatenation of per-record fields: 2 x fp16
    position bit patterns, 3 x b-bit codes, M x ceil(log2 B)-bit indices;
    byte-padded with zeros at the end."""
    n = pos16.shape[0]
    ib = index_bits(codebook)
    fields = [(pos16[:, 0].astype(np.uint64), 16), (pos16[:, 1].astype(np.uint64), 16)]
    fields += [(codes[:, i].astype(np.uint64), int(bits)) for i in range(3)]
    fields += [(idx[:, m].astype(np.uint64), ib) for m in range(idx.shape[1])]
    cols = []
    for val, width in fields:
        sh = np.arange(width - 1, -1, -1, dtype=np.uint64)
        cols.append(((val[:, None] >> sh[None, :]) & np.uint64(1)).astype(np.uint8))
    bitmat = np.concatenate(cols, axis=1).reshape(-1) if n else np.zeros(0, np.uint8)
    return np.packbits(bitmat)  # numpy packbits is MSB-first, zero-padded


def payload(seed: int, n: int, bits: int = 6, stages: int = 2, codebook: int = 8):
    """Random codec input: (payload bytes, gamma[3], beta[3], codebooks[M][B][3]).

    Positions are post-tanh coordinates in (-1, 1) rounded to IEEE binary16
    (RNE, reading R19); codes uniform in [0, 2^b); indices uniform in [0, B).
    """
    rng = _rng(40_000 + seed)
    n = int(n)
    u = rng.uniform(-1.0, 1.0, size=(n, 2)).astype(np.float16)
    pos16 = u.view(np.uint16)
    codes = rng.integers(0, 2 ** int(bits), size=(n, 3), dtype=np.int64)
    idx = rng.integers(0, int(codebook), size=(n, int(stages)), dtype=np.int64)
    gamma = rng.uniform(0.01, 0.1, size=3).astype(np.float32)
    beta = rng.uniform(-0.5, 0.5, size=3).astype(np.float32)
    books = rng.uniform(-0.3, 0.6, size=(int(stages), int(codebook), 3)).astype(np.float32)
    data = pack_records(pos16, codes, idx, bits, codebook)
    return data, gamma, beta, books
