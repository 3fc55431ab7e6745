"""Host-side checks that need no GPU: libgi.so loads, exports every symbol
include/gi.h declares, and its host-only entry points validate arguments."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gi_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2403_08551_b200 import build, gi
    build.build()
    return gi.load()


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2403_08551_b200 import gi
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in gi.SIGNATURES, f"binding lacks {s}"
        assert hasattr(gi, s) or s in ("gi_status_string", "gi_last_error"), s


def test_host_queries_and_validation(lib):
    from paper_2403_08551_b200 import gi
    assert gi.gi_abi_version() == 1
    f = gi.frame(768, 512)
    assert gi.gi_num_tiles(f) == 48 * 32
    assert gi.gi_proj_bytes(70000, f) == 70000 * 48
    assert gi.gi_bin_workspace_bytes(70000, 1 << 20, f) >= 2 * 4 * 1536   # counts + cursors
    assert gi.gi_backward_workspace_bytes(70000, 1 << 20, f) >= 32 * (1 << 20)
    assert gi.gi_lr_at(1) == 1e-3 and gi.gi_lr_at(20001) == 5e-4 and gi.gi_lr_at(40001) == 2.5e-4
    bad = gi.frame(768, 512, tile=8)
    assert gi.gi_num_tiles(bad) == -1
    # invalid arguments are rejected before any launch (no device needed)
    rc = lib.gi_project(None, -1, C.byref(f), 0, None, None, None)
    assert rc == gi.GI_EINVAL
    assert b"n must be" in lib.gi_last_error()
    rc = lib.gi_project(None, 10, C.byref(bad), 0, None, None, None)
    assert rc == gi.GI_EINVAL
    rc = lib.gi_adam_step(None, None, None, None, 8, 0, 1e-3, 0.9, 0.999, 1e-8, None, None)
    assert rc == gi.GI_EINVAL          # step is 1-based
    meta = gi.gi_codec_meta()
    meta.n, meta.bits, meta.stages, meta.codebook = 10, 20, 2, 8
    assert lib.gi_vq_decode(None, 0, C.byref(meta), None, None) == gi.GI_EFORMAT
    meta.bits = 6
    assert lib.gi_vq_decode(None, 69, C.byref(meta), None, None) == gi.GI_EFORMAT  # needs 70 B
    # fused decode + render: codec checks, one image per payload, buffers
    f1, f2b = gi.frame(768, 512), gi.frame(768, 512, batch=2)
    meta.bits = 20
    assert lib.gi_decode_render_frame(None, 0, C.byref(meta), C.byref(f1), 1 << 16, None, 0, None,
                                      None, None) == gi.GI_EFORMAT
    meta.bits = 6
    assert lib.gi_decode_render_frame(None, 69, C.byref(meta), C.byref(f1), 1 << 16, None, 0, None,
                                      None, None) == gi.GI_EFORMAT
    assert lib.gi_decode_render_frame(None, 70, C.byref(meta), C.byref(f2b), 1 << 16, None, 0, None,
                                      None, None) == gi.GI_EINVAL
    assert lib.gi_decode_render_frame(None, 70, C.byref(meta), C.byref(f1), 1 << 16, None, 0, None,
                                      None, None) == gi.GI_EINVAL        # no workspace
    assert lib.gi_status_string(3) == b"GI_ECAPACITY"
    # NEXT-2 / NEXT-4 entry points validate before any launch
    meta.bits = 20
    assert lib.gi_vq_encode(None, 0, C.byref(meta), None, 0, None, None) == gi.GI_EFORMAT
    meta.bits = 6
    fake = C.c_void_p(256)                  # never dereferenced: validation comes first
    assert lib.gi_vq_encode(fake, 0, C.byref(meta), fake, 69, None, None) == gi.GI_EFORMAT
    assert lib.gi_vq_encode(None, 2, C.byref(meta), None, 0, None, None) == gi.GI_EINVAL  # RS flag
    assert gi.gi_kmeans_workspace_bytes(1) == 0 and gi.gi_kmeans_workspace_bytes(8) == 8 * 32
    assert lib.gi_kmeans_step(None, 10, 1, None, None, None, 0, None) == gi.GI_EINVAL
    cfg = gi.qat_config(bits=20)
    assert gi.gi_qat_workspace_bytes(100, 1 << 16, f, cfg) == 0
    cfg = gi.qat_config()
    assert gi.gi_qat_workspace_bytes(100, 1 << 16, f, cfg) > gi.gi_fit_workspace_bytes(100, 1 << 16, f)
    f2 = gi.frame(768, 512, batch=2)
    rc = lib.gi_qat_step(*([None] * 12), 10, C.byref(f2), C.byref(cfg), 1 << 16, None, 0, None,
                         None, None, None)
    assert rc == gi.GI_EINVAL and b"batch 1" in lib.gi_last_error()
    rc = lib.gi_fit_grads(None, None, None, 10, C.byref(f), 0, 30, 5, 1 << 16, None, 0, None, None)
    assert rc == gi.GI_EINVAL and b"tile window" in lib.gi_last_error()
    rc = lib.gi_fit_grads(None, None, None, 10, C.byref(f), 0, -1, 0, 1 << 16, None, 0, None, None)
    assert rc == gi.GI_EINVAL and b"tile window" in lib.gi_last_error()
    # 8-bit targets: NULL buffers with a non-empty frame, a bad frame
    assert lib.gi_target_from_rgb8(None, C.byref(f), None, None, None, None) == gi.GI_EINVAL
    assert lib.gi_target_from_rgb8(None, C.byref(bad), None, None, None, None) == gi.GI_EINVAL
    assert lib.gi_target_upload_rgb8(None, None, C.byref(f), None, None, None) == gi.GI_EINVAL


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2403_08551_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), fn
                assert not re.search(r"^\s*#\s*include.*(oracle|gio)", txt, re.M), fn
                assert "libgio" not in txt and "gio." not in txt, fn
