"""Thin Python binding of libgi (include/gi.h): same names, argument
marshalling only.  Every step of the hot path runs in the CUDA kernels of
``libgi.so``; there is no CPU fallback -- if the library or a CUDA device is
missing, calls raise.

Tensors are torch tensors on the CUDA device (torch is used for device memory
and streams only).  ``stream=None`` means torch's current stream.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import build as _build

GI_OK, GI_EINVAL, GI_ECUDA, GI_ECAPACITY, GI_EFORMAT, GI_ENONFINITE = range(6)
GI_POS_LOGIT = 0
GI_POS_NORMALIZED = 1
GI_COV_RS = 2          # OR-ed flag: params[2:5] = (theta, s1, s2), Sigma = (RS)(RS)^T (NEXT-3)
GI_PROJ_BYTES = 48
TILE = 16

_STATUS = {0: "GI_OK", 1: "GI_EINVAL", 2: "GI_ECUDA", 3: "GI_ECAPACITY", 4: "GI_EFORMAT",
           5: "GI_ENONFINITE"}


class GiError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)} {detail}".strip())


class gi_frame(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tile", C.c_int32),
                ("batch", C.c_int32), ("k", C.c_float)]


class gi_codec_meta(C.Structure):
    _fields_ = [("n", C.c_int32), ("bits", C.c_int32), ("stages", C.c_int32),
                ("codebook", C.c_int32), ("gamma", C.c_float * 3), ("beta", C.c_float * 3),
                ("codebooks", C.c_void_p)]


class gi_qat_config(C.Structure):
    _fields_ = [("bits", C.c_int32), ("stages", C.c_int32), ("codebook", C.c_int32),
                ("lr", C.c_float), ("lam", C.c_float), ("decay", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float)]


def frame(width: int, height: int, batch: int = 1, k: float = 3.0, tile: int = TILE) -> gi_frame:
    return gi_frame(int(width), int(height), int(tile), int(batch), float(k))


# Every exported symbol of include/gi.h, with its ctypes signature.
_vp, _sz, _i32, _i64, _u32, _f32, _f64 = (C.c_void_p, C.c_size_t, C.c_int32, C.c_int64,
                                          C.c_uint32, C.c_float, C.c_double)
_FP = C.POINTER(gi_frame)
SIGNATURES = {
    "gi_status_string": (C.c_char_p, [C.c_int]),
    "gi_last_error": (C.c_char_p, []),
    "gi_abi_version": (_i32, []),
    "gi_num_tiles": (_i32, [_FP]),
    "gi_proj_bytes": (_sz, [_i32, _FP]),
    "gi_project": (C.c_int, [_vp, _i32, _FP, _u32, _vp, _vp, _vp]),
    "gi_bin_workspace_bytes": (_sz, [_i32, _i64, _FP]),
    "gi_bin": (C.c_int, [_vp, _vp, _i32, _FP, _i64, _vp, _sz, _vp, _vp, _vp, _vp, _vp]),
    "gi_render": (C.c_int, [_vp, _vp, _vp, _i32, _FP, _vp, _vp]),
    "gi_backward_workspace_bytes": (_sz, [_i32, _i64, _FP]),
    "gi_render_backward": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _FP, _u32, _vp, _vp, _i64,
                                     _vp, _sz, _vp, _vp, _vp, _vp]),
    "gi_adam_step": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _f32, _f32, _f32, _f32, _vp, _vp]),
    "gi_lr_at": (_f64, [_i32, _f64, _i32]),
    "gi_fit_workspace_bytes": (_sz, [_i32, _i64, _FP]),
    "gi_fit_n_keys": (_vp, [_vp, _i32, _i64, _FP]),
    "gi_fit_grads": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.POINTER(gi_frame), C.c_uint32, C.c_int32,
                               C.c_int32, C.c_int64, _vp, _sz, _vp, _vp]),
    "gi_peer_alloc": (C.c_int, [_sz, C.POINTER(_vp), _vp]),
    "gi_peer_free": (C.c_int, [_vp]),
    "gi_peer_open": (C.c_int, [_vp, C.POINTER(_vp)]),
    "gi_peer_close": (C.c_int, [_vp]),
    "gi_peer_adam_step": (C.c_int, [_vp, _vp, _vp, C.POINTER(_vp), C.c_int32, _i64, C.c_int32,
                                    _f32, _f32, _f32, _f32, C.c_int32, _vp, _vp, _vp]),
    "gi_fit_step": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _FP, _u32, _i64, _vp, _sz, _vp,
                              _f32, _i32, _f32, _f32, _f32, _vp, _vp, _vp, _vp]),
    "gi_launch_count": (_i64, []),
    "gi_adan_step": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _f32, _f32, _f32,
                               _f32, _f32, _vp, _vp]),
    "gi_fit_step_adan": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _FP, _u32, _i64, _vp,
                                   _sz, _vp, _f32, _i32, _f32, _f32, _f32, _f32, _f32, _vp, _vp,
                                   _vp]),
    "gi_fit_step_adan_chained": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _FP, _u32, _i64, _vp,
                                   _sz, _vp, _f32, _i32, _f32, _f32, _f32, _f32, _f32, _vp, _vp,
                                   _vp]),
    "gi_fit_prime": (C.c_int, [_vp, _i32, _FP, _u32, _i64, _vp, _sz, _vp]),
    "gi_fit_reset": (C.c_int, [_i32, _FP, _i64, _vp, _sz, _vp]),
    "gi_fit_seg_stats": (_vp, [_vp, _i32, _i64, _FP]),
    "gi_fit_bin_view": (C.c_int, [_vp, _i32, _i64, _FP, C.POINTER(_vp), C.POINTER(C.c_uint32),
                                  C.POINTER(_vp), C.POINTER(C.c_uint32)]),
    "gi_fit_step_chained": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _FP, _u32, _i64, _vp, _sz, _vp,
                                      _f32, _i32, _f32, _f32, _f32, _vp, _vp, _vp, _vp]),
    "gi_render_frame": (C.c_int, [_vp, _i32, _FP, _u32, _i64, _vp, _sz, _vp, _vp]),
    "gi_vq_decode": (C.c_int, [_vp, _sz, C.POINTER(gi_codec_meta), _vp, _vp]),
    "gi_decode_render_frame": (C.c_int, [_vp, _sz, C.POINTER(gi_codec_meta), _FP, _i64, _vp, _sz,
                                         _vp, _vp, _vp]),
    "gi_vq_encode": (C.c_int, [_vp, C.c_uint32, C.POINTER(gi_codec_meta), _vp, _sz, _vp, _vp]),
    "gi_kmeans_workspace_bytes": (_sz, [C.c_int32]),
    "gi_qat_workspace_bytes": (_sz, [C.c_int32, C.c_int64, C.POINTER(gi_frame),
                                     C.POINTER(gi_qat_config)]),
    "gi_qat_step": (C.c_int, [_vp] * 11 + [_vp, C.c_int32, C.POINTER(gi_frame),
                                           C.POINTER(gi_qat_config), C.c_int64, _vp, _sz, _vp, _vp,
                                           _vp, _vp]),
    "gi_kmeans_step": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _sz, _vp]),
    "gi_psnr_workspace_bytes": (_sz, [_FP]),
    "gi_psnr": (C.c_int, [_vp, _vp, _FP, _vp, _vp, _vp]),
    "gi_target_from_rgb8": (C.c_int, [_vp, _FP, _vp, _vp, _vp, _vp]),
    "gi_target_upload_rgb8": (C.c_int, [_vp, _vp, _FP, _vp, _vp, _vp]),
    "gi_check": (C.c_int, [_vp, _i64, _vp, _vp]),
}

_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_stale: bool = False):
    """Load libgi.so (raises if it is missing; the product has no fallback)."""
    global _lib
    if _lib is None:
        if build_if_stale:
            _build.build()
        path = os.environ.get("GI_LIB", _build.LIB)   # GI_LIB: an A/B variant build
        if not os.path.exists(path):
            raise RuntimeError(f"libgi.so not built at {path}: run __graft_entry__.build()")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not t.is_cuda:
        raise ValueError("libgi takes device tensors")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream) -> int | None:
    if stream is None:
        # torch's current stream on the current device (the capture stream
        # inside torch.cuda.graph); the raw getter skips building a Stream object
        if _raw_stream is not None:
            return _raw_stream(torch.cuda.current_device())
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ok(status: int, where: str):
    if status != GI_OK:
        detail = load().gi_last_error()
        raise GiError(status, where, detail.decode() if detail else "")


# ------------------------------------------------------------------ queries
def gi_abi_version() -> int:
    return load().gi_abi_version()


def gi_num_tiles(f: gi_frame) -> int:
    return load().gi_num_tiles(C.byref(f))


def gi_proj_bytes(n: int, f: gi_frame) -> int:
    return load().gi_proj_bytes(int(n), C.byref(f))


def gi_bin_workspace_bytes(n: int, key_capacity: int, f: gi_frame) -> int:
    return load().gi_bin_workspace_bytes(int(n), int(key_capacity), C.byref(f))


def gi_backward_workspace_bytes(n: int, key_capacity: int, f: gi_frame) -> int:
    return load().gi_backward_workspace_bytes(int(n), int(key_capacity), C.byref(f))


def gi_fit_workspace_bytes(n: int, key_capacity: int, f: gi_frame) -> int:
    return load().gi_fit_workspace_bytes(int(n), int(key_capacity), C.byref(f))


def gi_psnr_workspace_bytes(f: gi_frame) -> int:
    return load().gi_psnr_workspace_bytes(C.byref(f))


def gi_lr_at(step: int, lr0: float = 1e-3, half_every: int = 20000) -> float:
    return load().gi_lr_at(int(step), float(lr0), int(half_every))


def gi_fit_n_keys(fit_ws, n: int, key_capacity: int, f: gi_frame) -> int:
    return load().gi_fit_n_keys(_ptr(fit_ws), int(n), int(key_capacity), C.byref(f))


# ------------------------------------------------------------- hot path
def gi_project(params, n, f, flags, proj, tiles_touched, stream=None):
    _ok(load().gi_project(_ptr(params), int(n), C.byref(f), int(flags), _ptr(proj),
                          _ptr(tiles_touched), _stream(stream)), "gi_project")


def gi_bin(proj, tiles_touched, n, f, key_capacity, ws, key_tile, key_gid, tile_range, n_keys,
           stream=None):
    _ok(load().gi_bin(_ptr(proj), _ptr(tiles_touched), int(n), C.byref(f), int(key_capacity),
                      _ptr(ws), ws.numel() * ws.element_size(), _ptr(key_tile), _ptr(key_gid),
                      _ptr(tile_range), _ptr(n_keys), _stream(stream)), "gi_bin")


def gi_render(proj, key_gid, tile_range, n, f, image, stream=None):
    _ok(load().gi_render(_ptr(proj), _ptr(key_gid), _ptr(tile_range), int(n), C.byref(f),
                         _ptr(image), _stream(stream)), "gi_render")


def gi_render_backward(params, proj, key_gid, tile_range, n, f, flags, dL_dimage, target,
                       key_capacity, ws, grads, loss=None, image_out=None, stream=None):
    _ok(load().gi_render_backward(_ptr(params), _ptr(proj), _ptr(key_gid), _ptr(tile_range),
                                  int(n), C.byref(f), int(flags),
                                  _ptr(dL_dimage), _ptr(target), int(key_capacity), _ptr(ws),
                                  ws.numel() * ws.element_size(), _ptr(grads), _ptr(loss),
                                  _ptr(image_out), _stream(stream)), "gi_render_backward")


def gi_adam_step(params, grads, m, v, count, step, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                 nonfinite_flag=None, stream=None):
    _ok(load().gi_adam_step(_ptr(params), _ptr(grads), _ptr(m), _ptr(v), int(count), int(step),
                            float(lr), float(beta1), float(beta2), float(eps),
                            _ptr(nonfinite_flag), _stream(stream)), "gi_adam_step")


def _fit_step(fn, params, grads, m, v, target, n, f, flags, key_capacity, fit_ws, step_counter,
              lr0, half_every, beta1, beta2, eps, loss, status_flags, stage_events, stream, name):
    ev = None
    if stage_events is not None:
        handles = [e if isinstance(e, int) else e.cuda_event for e in stage_events]
        assert len(handles) == 6 and all(handles), "6 initialised events"
        ev = (C.c_void_p * 6)(*handles)
    _ok(fn(_ptr(params), _ptr(grads), _ptr(m), _ptr(v), _ptr(target), int(n), C.byref(f),
           int(flags), int(key_capacity), _ptr(fit_ws), fit_ws.numel() * fit_ws.element_size(),
           _ptr(step_counter), float(lr0), int(half_every), float(beta1), float(beta2), float(eps),
           _ptr(loss), _ptr(status_flags), ev, _stream(stream)), name)


class FitStepCall:
    """A prepared gi_fit_step_chained / gi_fit_step call (Adam) for a loop of
    steps on fixed buffers: the argument list is marshalled once; each call
    substitutes the target, the loss destination and the stream (the host cost
    per step is then one ctypes call -- it bounds a streaming fit's e2e rate)."""

    def __init__(self, chained, params, grads, m, v, n, f, flags, key_capacity, fit_ws,
                 step_counter, lr0, half_every, beta1, beta2, eps, status_flags):
        lib = load()
        self.fn = lib.gi_fit_step_chained if chained else lib.gi_fit_step
        self.name = "gi_fit_step_chained" if chained else "gi_fit_step"
        self.f = f
        self.argv = [_ptr(params), _ptr(grads), _ptr(m), _ptr(v), None, int(n), C.byref(f),
                     int(flags), int(key_capacity), _ptr(fit_ws),
                     fit_ws.numel() * fit_ws.element_size(), _ptr(step_counter), float(lr0),
                     int(half_every), float(beta1), float(beta2), float(eps), None,
                     _ptr(status_flags), None, None]

    def __call__(self, target: int, loss: int, stream: int):
        a = self.argv
        a[4] = target
        a[17] = loss
        a[20] = stream
        rc = self.fn(*a)
        if rc != GI_OK:
            _ok(rc, self.name)


def gi_fit_step(params, grads, m, v, target, n, f, flags, key_capacity, fit_ws, step_counter,
                lr0=1e-3, half_every=20000, beta1=0.9, beta2=0.999, eps=1e-8, loss=None,
                status_flags=None, stage_events=None, stream=None):
    """stage_events: None or 6 recorded torch.cuda.Event(external=True) / raw handles."""
    _fit_step(load().gi_fit_step, params, grads, m, v, target, n, f, flags, key_capacity, fit_ws,
              step_counter, lr0, half_every, beta1, beta2, eps, loss, status_flags, stage_events,
              stream, "gi_fit_step")


def gi_fit_step_chained(params, grads, m, v, target, n, f, flags, key_capacity, fit_ws,
                        step_counter, lr0=1e-3, half_every=20000, beta1=0.9, beta2=0.999, eps=1e-8,
                        loss=None, status_flags=None, stage_events=None, stream=None):
    _fit_step(load().gi_fit_step_chained, params, grads, m, v, target, n, f, flags, key_capacity,
              fit_ws, step_counter, lr0, half_every, beta1, beta2, eps, loss, status_flags,
              stage_events, stream, "gi_fit_step_chained")


def gi_adan_step(params, grads, m, v, n, grad_prev, count, step, lr, beta1=0.98, beta2=0.92,
                 beta3=0.99, eps=1e-8, weight_decay=0.0, nonfinite_flag=None, stream=None):
    _ok(load().gi_adan_step(_ptr(params), _ptr(grads), _ptr(m), _ptr(v), _ptr(n), _ptr(grad_prev),
                            int(count), int(step), float(lr), float(beta1), float(beta2),
                            float(beta3), float(eps), float(weight_decay), _ptr(nonfinite_flag),
                            _stream(stream)), "gi_adan_step")


def gi_fit_step_adan(params, grads, m, v, n, grad_prev, target, n_gauss, f, flags, key_capacity,
                     fit_ws, step_counter, lr0=1e-3, half_every=20000, beta1=0.98, beta2=0.92,
                     beta3=0.99, eps=1e-8, weight_decay=0.0, loss=None, status_flags=None,
                     stream=None):
    _ok(load().gi_fit_step_adan(_ptr(params), _ptr(grads), _ptr(m), _ptr(v), _ptr(n),
                                _ptr(grad_prev), _ptr(target), int(n_gauss), C.byref(f), int(flags),
                                int(key_capacity), _ptr(fit_ws),
                                fit_ws.numel() * fit_ws.element_size(), _ptr(step_counter),
                                float(lr0), int(half_every), float(beta1), float(beta2),
                                float(beta3), float(eps), float(weight_decay), _ptr(loss),
                                _ptr(status_flags), _stream(stream)), "gi_fit_step_adan")


def gi_fit_step_adan_chained(params, grads, m, v, n, grad_prev, target, n_gauss, f, flags,
                             key_capacity, fit_ws, step_counter, lr0=1e-3, half_every=20000,
                             beta1=0.98, beta2=0.92, beta3=0.99, eps=1e-8, weight_decay=0.0,
                             loss=None, status_flags=None, stream=None):
    _ok(load().gi_fit_step_adan_chained(_ptr(params), _ptr(grads), _ptr(m), _ptr(v), _ptr(n),
                                        _ptr(grad_prev), _ptr(target), int(n_gauss), C.byref(f),
                                        int(flags), int(key_capacity), _ptr(fit_ws),
                                        fit_ws.numel() * fit_ws.element_size(), _ptr(step_counter),
                                        float(lr0), int(half_every), float(beta1), float(beta2),
                                        float(beta3), float(eps), float(weight_decay), _ptr(loss),
                                        _ptr(status_flags), _stream(stream)),
        "gi_fit_step_adan_chained")


def gi_fit_prime(params, n, f, flags, key_capacity, fit_ws, stream=None):
    _ok(load().gi_fit_prime(_ptr(params), int(n), C.byref(f), int(flags), int(key_capacity),
                            _ptr(fit_ws), fit_ws.numel() * fit_ws.element_size(), _stream(stream)),
        "gi_fit_prime")


def gi_fit_reset(n, f, key_capacity, fit_ws, stream=None):
    _ok(load().gi_fit_reset(int(n), C.byref(f), int(key_capacity), _ptr(fit_ws),
                            fit_ws.numel() * fit_ws.element_size(), _stream(stream)),
        "gi_fit_reset")


def gi_fit_seg_stats(fit_ws, n, key_capacity, f) -> int:
    """Device address of the u32[2] segment statistics inside fit_ws."""
    return load().gi_fit_seg_stats(_ptr(fit_ws), int(n), int(key_capacity), C.byref(f)) or 0


def gi_fit_bin_view(fit_ws, n, key_capacity, f):
    """Device addresses of the direct-binning state inside fit_ws:
    (tile_count address, count stride in u32, slab address, slab capacity)."""
    tc, sl = _vp(), _vp()
    stride, scap = C.c_uint32(), C.c_uint32()
    _ok(load().gi_fit_bin_view(_ptr(fit_ws), int(n), int(key_capacity), C.byref(f), C.byref(tc),
                               C.byref(stride), C.byref(sl), C.byref(scap)), "gi_fit_bin_view")
    return int(tc.value or 0), int(stride.value), int(sl.value or 0), int(scap.value)


def gi_render_frame(params, n, f, flags, key_capacity, frame_ws, image, stream=None):
    _ok(load().gi_render_frame(_ptr(params), int(n), C.byref(f), int(flags), int(key_capacity),
                               _ptr(frame_ws), frame_ws.numel() * frame_ws.element_size(),
                               _ptr(image), _stream(stream)), "gi_render_frame")


def gi_launch_count() -> int:
    return load().gi_launch_count()


def gi_vq_encode(params, meta: gi_codec_meta, payload=None, eff=None, flags=0, stream=None):
    """NEXT-2 encoder: quantise params [n][8] into packed records (payload,
    uint8 device tensor) and/or the dequantised parameters eff [n][8]."""
    _ok(load().gi_vq_encode(_ptr(params), int(flags), C.byref(meta), _ptr(payload),
                            0 if payload is None else payload.numel() * payload.element_size(), _ptr(eff), _stream(stream)),
        "gi_vq_encode")


def gi_kmeans_workspace_bytes(B) -> int:
    return int(load().gi_kmeans_workspace_bytes(int(B)))


def gi_kmeans_step(points, centroids, assign, ws, stream=None):
    """One Lloyd iteration on device tensors points [n][3], centroids [B][3]."""
    n, B = points.shape[0], centroids.shape[0]
    _ok(load().gi_kmeans_step(_ptr(points), int(n), int(B), _ptr(centroids), _ptr(assign),
                              _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)), "gi_kmeans_step")


def qat_config(bits=6, stages=2, codebook=8, lr=1e-4, lam=1.0, decay=0.99, beta1=0.9,
               beta2=0.999, eps=1e-8) -> gi_qat_config:
    return gi_qat_config(int(bits), int(stages), int(codebook), float(lr), float(lam),
                         float(decay), float(beta1), float(beta2), float(eps))


def gi_qat_workspace_bytes(n, key_capacity, f: gi_frame, cfg: gi_qat_config) -> int:
    return int(load().gi_qat_workspace_bytes(int(n), int(key_capacity), C.byref(f), C.byref(cfg)))


def gi_qat_step(params, m, v, eff, grads, qparams, qm, qv, books, ema_n, ema_s, target, n,
                f: gi_frame, cfg: gi_qat_config, key_capacity, ws, step_counter, losses,
                status_flags=None, stream=None):
    _ok(load().gi_qat_step(*(_ptr(t) for t in (params, m, v, eff, grads, qparams, qm, qv, books,
                                                ema_n, ema_s, target)), int(n), C.byref(f),
                           C.byref(cfg), int(key_capacity), _ptr(ws), ws.numel() * ws.element_size(),
                           _ptr(step_counter), _ptr(losses), _ptr(status_flags), _stream(stream)),
        "gi_qat_step")


def gi_fit_grads(params, grads, target, n, f: gi_frame, flags, tile_row0, tile_rows, key_capacity,
                 fit_ws, loss, stream=None):
    """NEXT-4: gradient half of a fit step over a tile-row window (see gi.h)."""
    _ok(load().gi_fit_grads(_ptr(params), _ptr(grads), _ptr(target), int(n), C.byref(f),
                            int(flags), int(tile_row0), int(tile_rows), int(key_capacity),
                            _ptr(fit_ws), fit_ws.numel() * fit_ws.element_size(), _ptr(loss),
                            _stream(stream)), "gi_fit_grads")


# --- NEXT-4 peer exchange (see gi.h) ---------------------------------------
def gi_peer_alloc(nbytes: int):
    """cudaMalloc'd, zero-filled exchange buffer: (device pointer, 64-byte IPC handle)."""
    ptr = C.c_void_p()
    h = C.create_string_buffer(64)
    _ok(load().gi_peer_alloc(int(nbytes), C.byref(ptr), h), "gi_peer_alloc")
    return int(ptr.value), bytes(h.raw)


def gi_peer_free(ptr: int):
    _ok(load().gi_peer_free(ptr), "gi_peer_free")


def gi_peer_open(handle: bytes) -> int:
    ptr = C.c_void_p()
    _ok(load().gi_peer_open(C.create_string_buffer(bytes(handle), 64), C.byref(ptr)),
        "gi_peer_open")
    return int(ptr.value)


def gi_peer_close(ptr: int):
    _ok(load().gi_peer_close(ptr), "gi_peer_close")


def gi_peer_adam_step(params, m, v, grad_ptrs, count, step, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                      n_loss=0, loss_out=None, nonfinite_flag=None, stream=None):
    """Sum the G exchange buffers (rank order) and apply Adam (NEXT-4)."""
    arr = (_vp * len(grad_ptrs))(*[_ptr(g) for g in grad_ptrs])
    _ok(load().gi_peer_adam_step(_ptr(params), _ptr(m), _ptr(v), arr, len(grad_ptrs), int(count),
                                 int(step), float(lr), float(beta1), float(beta2), float(eps),
                                 int(n_loss), _ptr(loss_out), _ptr(nonfinite_flag),
                                 _stream(stream)), "gi_peer_adam_step")


def gi_vq_decode(payload, meta: gi_codec_meta, params, stream=None):
    _ok(load().gi_vq_decode(_ptr(payload), payload.numel() * payload.element_size(), C.byref(meta), _ptr(params),
                            _stream(stream)), "gi_vq_decode")


def gi_decode_render_frame(payload, meta: gi_codec_meta, f: gi_frame, key_capacity, frame_ws,
                           image, params=None, stream=None):
    """configs[4] in two kernels: decode fused into the projection, then render."""
    _ok(load().gi_decode_render_frame(_ptr(payload), payload.numel() * payload.element_size(),
                                      C.byref(meta), C.byref(f), int(key_capacity), _ptr(frame_ws),
                                      frame_ws.numel() * frame_ws.element_size(), _ptr(params),
                                      _ptr(image), _stream(stream)), "gi_decode_render_frame")


def _event(e):
    if e is None:
        return None
    return e if isinstance(e, int) else e.cuda_event


def gi_target_from_rgb8(rgb, f, target, wait_event=None, done_event=None, stream=None):
    """rgb: device u8 [B][H][W][3]; target: device fp32 [B][3][H][W] <- rgb / 255.
    Events: created torch.cuda.Event (recorded once) or raw handles."""
    _ok(load().gi_target_from_rgb8(_ptr(rgb), C.byref(f), _ptr(target), _event(wait_event),
                                   _event(done_event), _stream(stream)), "gi_target_from_rgb8")


def gi_target_upload_rgb8(host_rgb, dev_rgb, f, wait_event=None, ready_event=None, stream=None):
    """host_rgb: (pinned) host u8 [B][H][W][3] tensor or address -> dev_rgb (device)."""
    if isinstance(host_rgb, torch.Tensor):
        if host_rgb.is_cuda or not host_rgb.is_contiguous():
            raise ValueError("host_rgb: a contiguous host tensor")
        host_rgb = host_rgb.data_ptr()
    _ok(load().gi_target_upload_rgb8(host_rgb, _ptr(dev_rgb), C.byref(f), _event(wait_event),
                                     _event(ready_event), _stream(stream)),
        "gi_target_upload_rgb8")


def gi_psnr(image, target, f, psnr, ws, stream=None):
    _ok(load().gi_psnr(_ptr(image), _ptr(target), C.byref(f), _ptr(psnr), _ptr(ws),
                       _stream(stream)), "gi_psnr")


def gi_check(n_keys=None, key_capacity=0, status_flags=None, stream=None) -> int:
    """Sync and translate device status words -> GI_OK / GI_ECAPACITY / GI_ENONFINITE."""
    return load().gi_check(_ptr(n_keys), int(key_capacity), _ptr(status_flags), _stream(stream))


def codec_meta(n, gamma, beta, codebooks, bits=6, stages=2, codebook=8) -> gi_codec_meta:
    m = gi_codec_meta()
    m.n, m.bits, m.stages, m.codebook = int(n), int(bits), int(stages), int(codebook)
    for i in range(3):
        m.gamma[i] = float(gamma[i])
        m.beta[i] = float(beta[i])
    m.codebooks = _ptr(codebooks)
    m._keep = codebooks        # the struct holds a raw pointer: keep the tensor alive
    return m
