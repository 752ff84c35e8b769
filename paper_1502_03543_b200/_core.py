"""The kernel table: drop-in for the reference's `adascale._core.kernels`.

Reference: adascale/_core.py:10-16 selects `_kernels` (compiled) or
`_pykernels` (numpy) at import time and exports it as `kernels`; every caller
(linalg.py, normal.py, parallel.py) goes through that table.  Here the table
has a single implementation, the sm_100a CUDA library, with the same function
names, argument meaning, in-place semantics and sentinel returns
(SURVEY.md §8b).  numpy arrays in, numpy arrays out -- each call stages its
operands through device memory.  (The solver itself never uses this table: it
keeps everything device-resident, see engine.py.)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as dv
from ._lib import call

COMPILED = True
DENOM_EPS_REL = 1e-12  # _kernels.pyx:21-23


def _fmat(a, name="matrix"):
    a = np.asarray(a)
    if a.dtype != np.float64 or a.ndim != 2 or not a.flags.f_contiguous:
        # the reference's typed memoryviews (double[::1, :]) reject these
        raise ValueError(f"{name}: expected an F-contiguous float64 matrix")
    return a


def _vec(v, name="vector"):
    v = np.asarray(v)
    if v.dtype != np.float64 or v.ndim != 1:
        raise ValueError(f"{name}: expected a float64 vector")
    return v


class _CudaKernels:
    """Function table with the reference's signatures (_kernels.pyx)."""

    COMPILED = True
    DENOM_EPS_REL = DENOM_EPS_REL

    @staticmethod
    def dot_tree(u, v) -> float:  # _kernels.pyx:55-71
        u = _vec(u, "u")
        v = _vec(v, "v")
        n = u.shape[0]
        du, dvv, out = dv.upload(u), dv.upload(v), dv.empty(1)
        call("pdas_dot_tree", dv.ptr(du), 1, dv.ptr(dvv), 1, n, dv.ptr(out), dv.stream())
        return float(dv.download(out)[0])

    @staticmethod
    def mat_vec(a, x) -> np.ndarray:  # _kernels.pyx:74-88
        a = _fmat(a, "a")
        x = _vec(x, "x")
        m, n = a.shape
        da, dx, out = dv.upload(a), dv.upload(x), dv.empty(m)
        call("pdas_mat_vec", dv.ptr(da), m, n, dv.ptr(dx), dv.ptr(out), dv.stream())
        return dv.download(out)

    @staticmethod
    def mat_t_vec(a, y) -> np.ndarray:  # _kernels.pyx:91-105
        a = _fmat(a, "a")
        y = _vec(y, "y")
        m, n = a.shape
        da, dy, out = dv.upload(a), dv.upload(y), dv.empty(n)
        call("pdas_mat_t_vec", dv.ptr(da), m, n, dv.ptr(dy), dv.ptr(out), dv.stream())
        return dv.download(out)

    @staticmethod
    def gram(a) -> np.ndarray:  # _kernels.pyx:108-123
        a = _fmat(a, "a")
        m, n = a.shape
        da, g = dv.upload(a), dv.empty(m * m)
        call("pdas_gram", dv.ptr(da), m, n, dv.ptr(g), dv.stream())
        return dv.download(g).reshape((m, m), order="F")

    @staticmethod
    def scaled_gram(a, d) -> np.ndarray:  # _kernels.pyx:126-141
        a = _fmat(a, "a")
        d = _vec(d, "d")
        m, n = a.shape
        da, dd, g = dv.upload(a), dv.upload(d), dv.empty(m * m)
        call("pdas_scaled_gram", dv.ptr(da), m, n, dv.ptr(dd), dv.ptr(g), dv.stream())
        return dv.download(g).reshape((m, m), order="F")

    @staticmethod
    def cholesky_factor(g, eps_rel):  # _kernels.pyx:144-171
        g = _fmat(g, "g")
        nn = g.shape[0]
        t = dv.require_gpu()
        dg, low = dv.upload(g), dv.empty(nn * nn)
        fail = dv.empty(1, dtype=t.int64)
        call("pdas_cholesky_factor", dv.ptr(dg), nn, float(eps_rel), dv.ptr(low), dv.ptr(fail),
             dv.stream())
        return dv.download(low).reshape((nn, nn), order="F"), int(dv.download(fail)[0])

    @staticmethod
    def cholesky_solve_many(low, b) -> np.ndarray:  # _kernels.pyx:174-193
        low = _fmat(low, "low")
        b = np.asfortranarray(np.asarray(b, dtype=np.float64))
        m, k = b.shape
        dl, x = dv.upload(low), dv.upload(b)
        call("pdas_cholesky_solve_many", dv.ptr(dl), m, dv.ptr(x), k, dv.stream())
        return dv.download(x).reshape((m, k), order="F")

    @staticmethod
    def build_v(a, l0, dl, v) -> None:  # _kernels.pyx:196-202
        a = _fmat(a, "a")
        m = a.shape[0]
        da, out = dv.upload(a), dv.empty(m)
        call("pdas_build_v", dv.ptr(da), m, int(l0), float(dl), dv.ptr(out), dv.stream())
        v[:] = dv.download(out)

    @staticmethod
    def sweep_phase1(cols, v, inner, k0, k1) -> None:  # _kernels.pyx:205-218
        cols = _fmat(cols, "cols")
        m = cols.shape[0]
        dc, dvv, di = dv.upload(cols), dv.upload(v), dv.upload(inner)
        call("pdas_sweep_phase1", dv.ptr(dc), m, dv.ptr(dvv), dv.ptr(di), int(k0), int(k1),
             dv.stream())
        inner[:] = dv.download(di)

    @staticmethod
    def sweep_phase2(cols, l0, inner, denom, k0, k1) -> None:  # _kernels.pyx:221-231
        cols = _fmat(cols, "cols")
        m = cols.shape[0]
        dc, di = dv.upload(cols), dv.upload(inner)
        call("pdas_sweep_phase2", dv.ptr(dc), m, int(l0), dv.ptr(di), float(denom), int(k0),
             int(k1), dv.stream())
        cols[...] = dv.download(dc).reshape(cols.shape, order="F")

    @staticmethod
    def solve_sweeps(cols, a, d, inner, v, workers) -> int:  # _kernels.pyx:270-291
        cols = _fmat(cols, "cols")
        a = _fmat(a, "a")
        m, n = a.shape
        if cols.shape != (m, n + 1):
            raise ValueError("cols must be m x (n+1)")
        t = dv.require_gpu()
        dc, da, dd = dv.upload(cols), dv.upload(a), dv.upload(d)
        fail = dv.zeros(1, dtype=t.int32)
        call("pdas_solve_sweeps", dv.ptr(dc), dv.ptr(da), dv.ptr(dd), None, None, m, n,
             int(workers), dv.ptr(fail), dv.stream())
        cols[...] = dv.download(dc).reshape(cols.shape, order="F")
        return int(dv.download(fail)[0])


kernels = _CudaKernels()


def active_core() -> str:
    """Name of the kernel core (reference _core.py:19-21): always the CUDA one."""
    return "cuda-sm_100a"


def device_info():
    """(sm_count, (major, minor)) of the current device."""
    dv.require_gpu()
    sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    call("pdas_device_info", ctypes.addressof(sm), ctypes.addressof(ma), ctypes.addressof(mi))
    return sm.value, (ma.value, mi.value)
