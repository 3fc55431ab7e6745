"""B200-native (sm_100a) GaussianImage hot path (arXiv 2403.08551).

``gi``        -- thin ctypes binding of libgi.so (include/gi.h), same names.
``pipeline``  -- device buffers, render / fit-step sequences, CUDA graphs.
``dist``      -- image-batch data parallelism over torch.distributed.
"""
from . import gi  # noqa: F401

__all__ = ["gi"]
