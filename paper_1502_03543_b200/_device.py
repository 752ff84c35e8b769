"""Device plumbing: CUDA memory and streams come from PyTorch (allocation,
H2D/D2H copies, the current stream); all arithmetic of the path runs in the
sm_100a kernels of libpdas_b200.so.  No CPU fallback: without a CUDA device
every compute entry point raises NativeLibraryError."""

from __future__ import annotations

import numpy as np

from ._lib import NativeLibraryError, load

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_gpu():
    t = torch()
    if not t.cuda.is_available():
        raise NativeLibraryError(
            "a CUDA (sm_100a) device is required: paper_1502_03543_b200 has no CPU fallback")
    load()
    return t


def device():
    t = require_gpu()
    return t.device("cuda", t.cuda.current_device())


def stream() -> int:
    """cudaStream_t of torch's current stream, as an int for ctypes."""
    return require_gpu().cuda.current_stream().cuda_stream


def synchronize() -> None:
    require_gpu().cuda.current_stream().synchronize()


def empty(n: int, dtype=None):
    t = require_gpu()
    return t.empty(max(int(n), 0), dtype=dtype or t.float64, device=device())


def zeros(n: int, dtype=None):
    t = require_gpu()
    return t.zeros(max(int(n), 0), dtype=dtype or t.float64, device=device())


def upload(a, pin: bool = False):
    """numpy -> flat device fp64 tensor.  2-D arrays are flattened in column
    (Fortran) order: element (i,j) at j*rows+i (reference linalg.py:1-7)."""
    t = require_gpu()
    arr = np.asarray(a, dtype=np.float64)
    flat = arr.ravel(order="F") if arr.ndim == 2 else np.ascontiguousarray(arr).ravel()
    host = t.from_numpy(np.ascontiguousarray(flat))
    if pin:
        host = host.pin_memory()
    return host.to(device(), non_blocking=pin)


def download(x) -> np.ndarray:
    return x.detach().cpu().numpy().copy()


def ptr(x) -> int:
    return 0 if x is None else int(x.data_ptr())
