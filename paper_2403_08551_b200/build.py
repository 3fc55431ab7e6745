"""Build libgi.so in-tree for sm_100a (explicit nvcc; no JIT cache).

Each translation unit is compiled to an object in parallel (one nvcc per
source), then linked into the shared library."""
from __future__ import annotations

import os
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgi.so")
SOURCES = ["api.cu", "project.cu", "scan.cu", "bin.cu", "render.cu", "backward.cu", "adam.cu",
           "adan.cu", "decode.cu", "psnr.cu", "qat.cu", "peer.cu", "fused.cu", "image.cu"]
HEADERS = ["gi_internal.cuh", "raster_common.cuh", "project_core.cuh", "codec_core.cuh",
           "chunks.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "gi.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Compile libgi.so (or, for A/B experiments, a variant at `out` with
    GI_NVCC_EXTRA flags; load it with GI_LIB=<path>)."""
    lib = os.path.abspath(out) if out else LIB
    if not (force or out or _stale()):
        return lib
    extra = os.environ.get("GI_NVCC_EXTRA", "").split()   # experiments (-D...)
    with tempfile.TemporaryDirectory(prefix="libgi_") as tmp:
        objs = [os.path.join(tmp, s.replace(".cu", ".o")) for s in SOURCES]
        cmds = [[NVCC] + FLAGS + extra + ["-c", os.path.join(CSRC, s), "-o", o]
                for s, o in zip(SOURCES, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c))

        def run(c):
            return subprocess.run(c, cwd=CSRC, capture_output=True, text=True)

        with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
            results = list(ex.map(run, cmds))
        for c, r in zip(cmds, results):
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(c)}\n{r.stderr}")
            if verbose and r.stderr.strip():
                print(r.stderr)
        link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs
        if verbose:
            print(" ".join(link))
        subprocess.check_call(link, cwd=CSRC)
    return lib


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose=True, out=sys.argv[1] if len(sys.argv) > 1 else None))
