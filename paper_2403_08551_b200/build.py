"""Build libgi.so in-tree for sm_100a (explicit nvcc; no JIT cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgi.so")
SOURCES = ["api.cu", "project.cu", "scan.cu", "bin.cu", "render.cu", "backward.cu", "adam.cu",
           "adan.cu", "decode.cu", "psnr.cu", "qat.cu", "peer.cu"]
HEADERS = ["gi_internal.cuh", "raster_common.cuh", "project_core.cuh", "codec_core.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "gi.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        extra = os.environ.get("GI_NVCC_EXTRA", "").split()   # experiments (-D...)
        cmd = [NVCC] + FLAGS + extra + ["-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd, cwd=CSRC)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
