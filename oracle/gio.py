"""ctypes/numpy front end of the fp64 oracle ``libgio.so`` (TEST INFRASTRUCTURE).

Every function takes fp32 parameters ``[N][8]`` = {mux, muy, l1, l2, l3,
c'r, c'g, c'b} for ONE image and returns fp64 results.  Passages followed are
cited in ``gio.cpp``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gio.cpp")
_LIB = os.path.join(_HERE, "libgio.so")

POS_LOGIT = 0
POS_NORMALIZED = 1
COV_RS = 2          # OR-ed into pos_mode: params[2:5] = (theta, s1, s2) (Eq. 2-3, NEXT-3)
ALL_PAIRS, TILED, DENSE = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, fp64, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC",
                               "-shared", "-std=c++17", _SRC, "-o", _LIB])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp, fp, ip, up = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                          C.POINTER(C.c_int32), C.POINTER(C.c_uint32))
        L.gio_kmeans.restype = C.c_double
        L.gio_kmeans.argtypes = [fp, C.c_int, C.c_int, fp, C.c_int, up]
        L.gio_float_to_half.restype = C.c_uint32
        L.gio_float_to_half.argtypes = [C.c_float]
        L.gio_vq_encode.argtypes = [fp, C.c_int, C.c_int, fp, fp, fp, C.c_int, C.c_int, C.c_int,
                                    up, up, up, fp]
        L.gio_eval_sigma.restype = C.c_double
        L.gio_eval_sigma.argtypes = [dp, C.c_double, C.c_double]
        L.gio_inverse2.argtypes = [dp, dp]
        L.gio_chol_backward.argtypes = [dp, C.c_double, C.c_double, C.c_double, dp]
        L.gio_rs_backward.argtypes = [dp, C.c_double, C.c_double, C.c_double, dp]
        L.gio_project.argtypes = [fp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int,
                                  dp, dp, dp, ip, ip, up]
        L.gio_bin.restype = C.c_int64
        L.gio_bin.argtypes = [fp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int, C.c_int,
                              up, up, C.c_int64, up]
        L.gio_render.argtypes = [fp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int,
                                 C.c_int, dp]
        L.gio_mse.restype = C.c_double
        L.gio_mse.argtypes = [dp, fp, C.c_int, C.c_int, dp]
        L.gio_backward.argtypes = [fp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int,
                                   C.c_int, dp, dp]
        L.gio_lr_at.restype = C.c_double
        L.gio_lr_at.argtypes = [C.c_int, C.c_double, C.c_int]
        L.gio_adam.argtypes = [fp, fp, fp, fp, C.c_int64, C.c_int, C.c_float, C.c_float,
                               C.c_float, C.c_float, dp, dp, dp]
        L.gio_adan.argtypes = [fp, fp, fp, fp, fp, fp, C.c_int64, C.c_int, C.c_float, C.c_float,
                               C.c_float, C.c_float, C.c_float, C.c_float, dp, dp, dp, dp]
        L.gio_half_to_double.restype = C.c_double
        L.gio_half_to_double.argtypes = [C.c_uint32]
        L.gio_vq_decode.restype = C.c_int
        L.gio_vq_decode.argtypes = [C.POINTER(C.c_uint8), C.c_int64, C.c_int, C.c_int, C.c_int,
                                    C.c_int, fp, fp, fp, fp]
        L.gio_psnr.restype = C.c_double
        L.gio_psnr.argtypes = [dp, fp, C.c_int64]
        L.gio_num_threads.restype = C.c_int
        L.gio_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def num_threads() -> int:
    return lib().gio_num_threads()


def set_threads(t: int) -> None:
    lib().gio_set_threads(int(t))


def eval_sigma(sinv, dx, dy) -> float:
    s = np.ascontiguousarray(sinv, dtype=np.float64)
    return lib().gio_eval_sigma(_p(s, C.c_double), float(dx), float(dy))


def inverse2(S):
    s = np.ascontiguousarray(S, dtype=np.float64)
    out = np.zeros(3)
    lib().gio_inverse2(_p(s, C.c_double), _p(out, C.c_double))
    return out


def chol_backward(G, l1e, l2, l3e):
    g = np.ascontiguousarray(G, dtype=np.float64)
    out = np.zeros(3)
    lib().gio_chol_backward(_p(g, C.c_double), float(l1e), float(l2), float(l3e),
                            _p(out, C.c_double))
    return out


def rs_backward(G, th, s1e, s2e):
    g = np.ascontiguousarray(G, dtype=np.float64)
    out = np.zeros(3)
    lib().gio_rs_backward(_p(g, C.c_double), float(th), float(s1e), float(s2e), _p(out, C.c_double))
    return out


def project(params, W, H, k=3.0, tile=16, pos_mode=POS_LOGIT):
    """-> dict(mu[n,2], sigma[n,3], sinv[n,3], box[n,4], rect[n,4], touched[n])."""
    p = _f32(params)
    n = p.shape[0]
    mu = np.zeros((n, 2)); sig = np.zeros((n, 3)); sinv = np.zeros((n, 3))
    box = np.zeros((n, 4), np.int32); rect = np.zeros((n, 4), np.int32)
    touched = np.zeros(n, np.uint32)
    lib().gio_project(_p(p, C.c_float), n, int(W), int(H), float(k), int(tile), int(pos_mode),
                      _p(mu, C.c_double), _p(sig, C.c_double), _p(sinv, C.c_double),
                      _p(box, C.c_int32), _p(rect, C.c_int32), _p(touched, C.c_uint32))
    return dict(mu=mu, sigma=sig, sinv=sinv, box=box, rect=rect, touched=touched)


def n_tiles(W, H, tile=16) -> int:
    return ((int(W) + tile - 1) // tile) * ((int(H) + tile - 1) // tile)


def bin(params, W, H, k=3.0, tile=16, pos_mode=POS_LOGIT, method=1):
    """-> (key_tile[K] u32, key_gid[K] u32, tile_range[T+1] u32)."""
    p = _f32(params)
    n = p.shape[0]
    T = n_tiles(W, H, tile)
    rng = np.zeros(T + 1, np.uint32)
    L = lib()
    K = L.gio_bin(_p(p, C.c_float), n, int(W), int(H), float(k), int(tile), int(pos_mode),
                  int(method), None, None, 0, _p(rng, C.c_uint32))
    kt = np.zeros(max(K, 1), np.uint32); kg = np.zeros(max(K, 1), np.uint32)
    L.gio_bin(_p(p, C.c_float), n, int(W), int(H), float(k), int(tile), int(pos_mode),
              int(method), _p(kt, C.c_uint32), _p(kg, C.c_uint32), K, _p(rng, C.c_uint32))
    return kt[:K], kg[:K], rng


def render(params, W, H, k=3.0, tile=16, pos_mode=POS_LOGIT, mode=ALL_PAIRS):
    """Eq. 7 render -> fp64 planar [3][H][W]."""
    p = _f32(params)
    img = np.zeros((3, int(H), int(W)))
    lib().gio_render(_p(p, C.c_float), p.shape[0], int(W), int(H), float(k), int(tile),
                     int(pos_mode), int(mode), _p(img, C.c_double))
    return img


def mse(image, target):
    """-> (loss, dL/dC) for the L2 loss of P:298 (mean over 3HW)."""
    im = np.ascontiguousarray(image, dtype=np.float64)
    t = _f32(target)
    g = np.zeros_like(im)
    H, W = im.shape[1], im.shape[2]
    loss = lib().gio_mse(_p(im, C.c_double), _p(t, C.c_float), W, H, _p(g, C.c_double))
    return loss, g


def backward(params, dL_dC, W, H, k=3.0, tile=16, pos_mode=POS_LOGIT, mode=ALL_PAIRS):
    """Appendix A backward -> fp64 grads [N][8] (mode ALL_PAIRS/TILED = boxed, DENSE)."""
    p = _f32(params)
    g = np.ascontiguousarray(dL_dC, dtype=np.float64)
    out = np.zeros((p.shape[0], 8))
    lib().gio_backward(_p(p, C.c_float), p.shape[0], int(W), int(H), float(k), int(tile),
                       int(pos_mode), 2 if mode == DENSE else 0, _p(g, C.c_double),
                       _p(out, C.c_double))
    return out


def loss_and_grads(params, target, k=3.0, tile=16, pos_mode=POS_LOGIT, mode=TILED):
    t = _f32(target)
    H, W = t.shape[1], t.shape[2]
    img = render(params, W, H, k, tile, pos_mode, mode)
    loss, g = mse(img, t)
    return img, loss, backward(params, g, W, H, k, tile, pos_mode, mode)


def lr_at(step, lr0=1e-3, half_every=20000) -> float:
    return lib().gio_lr_at(int(step), float(lr0), int(half_every))


def adam(p, g, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """One fp64 Adam step from fp32 state -> (p, m, v) fp64."""
    p, g, m, v = _f32(p), _f32(g), _f32(m), _f32(v)
    po, mo, vo = np.zeros(p.shape), np.zeros(p.shape), np.zeros(p.shape)
    lib().gio_adam(_p(p, C.c_float), _p(g, C.c_float), _p(m, C.c_float), _p(v, C.c_float),
                   p.size, int(step), float(lr), float(beta1), float(beta2), float(eps),
                   _p(po, C.c_double), _p(mo, C.c_double), _p(vo, C.c_double))
    return po, mo, vo


def adan(p, g, m, v, n, gprev, step, lr, beta1=0.98, beta2=0.92, beta3=0.99, eps=1e-8, wd=0.0):
    """One fp64 Adan step from fp32 state -> (p, m, v, n) fp64 (g_prev' = g)."""
    p, g, m, v, n, gp = (_f32(x) for x in (p, g, m, v, n, gprev))
    outs = [np.zeros(p.shape) for _ in range(4)]
    lib().gio_adan(_p(p, C.c_float), _p(g, C.c_float), _p(m, C.c_float), _p(v, C.c_float),
                   _p(n, C.c_float), _p(gp, C.c_float), p.size, int(step), float(lr),
                   float(beta1), float(beta2), float(beta3), float(eps), float(wd),
                   *[_p(o, C.c_double) for o in outs])
    return tuple(outs)


def half_to_double(bits: int) -> float:
    return lib().gio_half_to_double(int(bits))


def vq_decode(payload, n, gamma, beta, books, bits=6, stages=2, codebook=8):
    """Attribute decode -> fp32 params [n][8] (positions normalised, pos_mode 1)."""
    data = np.ascontiguousarray(payload, dtype=np.uint8)
    g, b, cb = _f32(gamma), _f32(beta), _f32(books)
    out = np.zeros((int(n), 8), np.float32)
    rc = lib().gio_vq_decode(_p(data, C.c_uint8), data.size, int(n), int(bits), int(stages),
                             int(codebook), _p(g, C.c_float), _p(b, C.c_float),
                             _p(cb, C.c_float), _p(out, C.c_float))
    if rc != 0:
        raise ValueError("payload too short")
    return out


def psnr(x, y) -> float:
    a = np.ascontiguousarray(x, dtype=np.float64)
    b = _f32(y)
    return lib().gio_psnr(_p(a, C.c_double), _p(b, C.c_float), a.size)


def float_to_half(x) -> int:
    return int(lib().gio_float_to_half(float(np.float32(x))))


def vq_encode(params, gamma, beta, books, bits=6, stages=2, codebook=8, pos_mode=POS_LOGIT):
    """Attribute quantisation (NEXT-2): -> dict(pos16 [n][2], codes [n][3],
    idx [n][M] (uint32), eff [n][8] fp32 = what vq_decode returns)."""
    p = _f32(params).reshape(-1, 8)
    n = p.shape[0]
    g, b, cb = _f32(gamma), _f32(beta), _f32(books)
    pos16 = np.zeros((n, 2), np.uint32)
    codes = np.zeros((n, 3), np.uint32)
    idx = np.zeros((n, int(stages)), np.uint32)
    eff = np.zeros((n, 8), np.float32)
    up = C.POINTER(C.c_uint32)
    lib().gio_vq_encode(_p(p, C.c_float), n, int(pos_mode), _p(g, C.c_float), _p(b, C.c_float),
                        _p(cb, C.c_float), int(bits), int(stages), int(codebook), _p(pos16, C.c_uint32),
                        _p(codes, C.c_uint32), _p(idx, C.c_uint32), _p(eff, C.c_float))
    return dict(pos16=pos16, codes=codes, idx=idx, eff=eff)


def kmeans(points, centroids, iters=5):
    """Lloyd iterations (NEXT-2 codebook init) -> (centroids fp32 [B][3],
    assignment uint32 [n], fp64 distortion of the last assignment)."""
    pts = _f32(points).reshape(-1, 3)
    cent = np.array(_f32(centroids).reshape(-1, 3), copy=True)
    asg = np.zeros(pts.shape[0], np.uint32)
    d = lib().gio_kmeans(_p(pts, C.c_float), pts.shape[0], cent.shape[0], _p(cent, C.c_float),
                         int(iters), _p(asg, C.c_uint32))
    return cent, asg, d



def qat_step(params, target, state, step, lr, lam=1.0, decay=0.99, bits=6, stages=2, codebook=8,
             mode=TILED, k=3.0, beta1=0.9, beta2=0.999, eps=1e-8):
    """One attribute quantisation-aware fine-tuning step (NEXT-2; P:249-276,
    P:301-307; SPEC quant module), composed from the oracle's pinned parts:

      1. forward on the quantised cloud p^ = Q(p)  (vq_encode: fp16 position,
         Eq. 8 codes, Eq. 9 greedy RVQ), L_rec = L2 of its render
      2. straight-through gradients (reading R32): position d/draw = d/du *
         (1 - tanh^2 raw); l: d/dl = d/dl^ inside the clamp range, 0 outside;
         gamma_i += d/dl^ * (code - x) inside, * code outside (LSQ+ without
         gradient scaling); beta_i += d/dl^ outside the range only; c' gets
         d/dc^ (Eq. 10's stop-gradient leaves the commitment term to the
         codebooks)
      3. Adam (R16 constants, constant lr) on p and on (gamma, beta)
      4. EMA codebooks (SPEC ema_update, reading R33): per stage m and
         codeword k with n_k assigned residuals r = c' - c^^{m-1} summing to
         s_k: N_k <- d N_k + (1 - d) n_k, S_k <- d S_k + (1 - d) s_k, and
         C^m[k] <- S_k / N_k when n_k > 0 (unchanged otherwise)
      5. L_c (Eq. 10) = 1/(N B) sum_m sum_n ||r_n^{m-1} - C^m[i_n^m]||^2 with
         the pre-update codebooks; L = L_rec + lam L_c

    state: dict(m, v [N][8]; gamma, beta [3]; qm, qv [6] (Adam state of
    gamma|beta); books [M][B][3]; ema_n [M][B]; ema_s [M][B][3]) -- fp32
    arrays, returned updated (fp32) with grads / eff / losses.
    """
    p = _f32(params).reshape(-1, 8)
    n = p.shape[0]
    gamma, beta = _f32(state["gamma"]), _f32(state["beta"])
    books = _f32(state["books"]).reshape(stages, codebook, 3)
    enc = vq_encode(p, gamma, beta, books, bits, stages, codebook, POS_LOGIT)
    eff = enc["eff"]
    t = _f32(target)
    H, W = t.shape[1], t.shape[2]
    img = render(eff, W, H, k, 16, POS_NORMALIZED, mode)
    l_rec, dimg = mse(img, t)
    ge = backward(eff, dimg, W, H, k, 16, POS_NORMALIZED, mode)          # d/dp^ (fp64)
    # 2. straight-through map
    g = np.array(ge, copy=True)
    th = np.tanh(p[:, :2].astype(np.float64))
    g[:, :2] = ge[:, :2] * (1.0 - th * th)
    qmax = float((1 << bits) - 1)
    x = ((p[:, 2:5] - beta[None, :]) / gamma[None, :]).astype(np.float32)   # fp32 as the encoder
    inside = (x >= 0) & (x <= qmax)
    code = enc["codes"].astype(np.float64)
    g[:, 2:5] = np.where(inside, ge[:, 2:5], 0.0)
    dgamma = (ge[:, 2:5] * np.where(inside, code - x.astype(np.float64), code)).sum(0)
    dbeta = (ge[:, 2:5] * np.where(inside, 0.0, 1.0)).sum(0)
    # 3. Adam
    po, mo, vo = adam(p, g.astype(np.float32), state["m"], state["v"], step, lr, beta1, beta2, eps)
    qg = np.concatenate([dgamma, dbeta]).astype(np.float32)
    qp = np.concatenate([gamma, beta])
    qpo, qmo, qvo = adam(qp, qg, state["qm"], state["qv"], step, lr, beta1, beta2, eps)
    # 4./5. residuals per stage with the pre-update books, EMA, commitment
    c = p[:, 5:8]
    chat = np.zeros((n, 3), np.float32)
    ema_n = np.array(_f32(state["ema_n"]).reshape(stages, codebook), np.float64)
    ema_s = np.array(_f32(state["ema_s"]).reshape(stages, codebook, 3), np.float64)
    new_books = np.array(books, copy=True)
    l_c = 0.0
    for m in range(stages):
        r = (c - chat).astype(np.float32)                                 # fp32 as the encoder
        ii = enc["idx"][:, m].astype(np.int64)
        cw = books[m][ii]
        l_c += ((r.astype(np.float64) - cw.astype(np.float64)) ** 2).sum()
        cnt = np.bincount(ii, minlength=codebook).astype(np.float64)
        sums = np.zeros((codebook, 3))
        np.add.at(sums, ii, r.astype(np.float64))
        ema_n[m] = decay * ema_n[m] + (1.0 - decay) * cnt
        ema_s[m] = decay * ema_s[m] + (1.0 - decay) * sums
        upd = cnt > 0
        new_books[m][upd] = (ema_s[m][upd] / ema_n[m][upd][:, None]).astype(np.float32)
        chat = (cw if m == 0 else (chat + cw)).astype(np.float32)
    l_c /= float(n * codebook)
    out = dict(state)
    out.update(m=mo.astype(np.float32), v=vo.astype(np.float32), gamma=qpo[:3].astype(np.float32),
               beta=qpo[3:].astype(np.float32), qm=qmo.astype(np.float32),
               qv=qvo.astype(np.float32), books=new_books, ema_n=ema_n.astype(np.float32),
               ema_s=ema_s.astype(np.float32))
    return dict(params=po.astype(np.float32), state=out, grads=g, grads_eff=ge, eff=eff,
                dgamma=dgamma, dbeta=dbeta, l_rec=l_rec, l_c=l_c, loss=l_rec + lam * l_c,
                enc=enc)
