"""ctypes binding of the C-ABI in include/pdas_b200.h (libpdas_b200.so).

This mirrors how the reference binds its compiled core (adascale/_core.py:
import-time selection of `_kernels`), except that there is exactly ONE core:
the sm_100a CUDA library.  There is no CPU fallback -- a missing library or
a missing GPU raises immediately and loudly.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDAS_B200_LIB", os.path.join(HERE, "libpdas_b200.so"))

PDAS_OK = 0
PDAS_ERR_ARG = -1
PDAS_ERR_CUDA = -2
PDAS_ERR_UNSUPPORTED = -3
PDAS_ERR_NOMEM = -4

_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_VP = ctypes.c_void_p
_D = ctypes.c_double


class PdasIterState(ctypes.Structure):
    """Mirror of `PdasIterState` in include/pdas_b200.h."""

    _fields_ = [
        ("chol_fail", ctypes.c_int64),
        ("blocking", ctypes.c_int64),
        ("cascade_fail", ctypes.c_int32),
        ("interior_flags", ctypes.c_uint32),
        ("nonfinite", ctypes.c_int32),
        ("stepped", ctypes.c_int32),
        ("fallback", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("gap", ctypes.c_double),
        ("pobj", ctypes.c_double),
        ("dobj", ctypes.c_double),
        ("r_primal", ctypes.c_double),
        ("r_dual", ctypes.c_double),
        ("r_comp", ctypes.c_double),
        ("min_ratio", ctypes.c_double),
    ]


STATE_BYTES = ctypes.sizeof(PdasIterState)
OFF_CHOL_FAIL = PdasIterState.chol_fail.offset
OFF_CASCADE_FAIL = PdasIterState.cascade_fail.offset

# name -> (restype, argtypes): every symbol include/pdas_b200.h declares.
SIGNATURES = {
    "pdas_abi_version": (ctypes.c_int, []),
    "pdas_last_error": (ctypes.c_char_p, []),
    "pdas_device_info": (ctypes.c_int, [_VP, _VP, _VP]),
    "pdas_cascade_max_m": (ctypes.c_int64, []),
    "pdas_dot_tree": (ctypes.c_int, [_VP, _I64, _VP, _I64, _I64, _VP, _VP]),
    "pdas_mat_vec": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP, _VP]),
    "pdas_mat_t_vec": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP, _VP]),
    "pdas_gram": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP]),
    "pdas_scaled_gram": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP, _VP]),
    "pdas_cholesky_factor": (ctypes.c_int, [_VP, _I64, _D, _VP, _VP, _VP]),
    "pdas_cholesky_solve_many": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP]),
    "pdas_build_v": (ctypes.c_int, [_VP, _I64, _I64, _D, _VP, _VP]),
    "pdas_sweep_phase1": (ctypes.c_int, [_VP, _I64, _VP, _VP, _I64, _I64, _VP]),
    "pdas_sweep_phase2": (ctypes.c_int, [_VP, _I64, _I64, _VP, _D, _I64, _I64, _VP]),
    "pdas_solve_sweeps": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _I64, _I64, ctypes.c_int, _VP, _VP]),
    "pdas_cascade_ws_bytes": (ctypes.c_int64, [_I64, _I64]),
    "pdas_solve_sweeps_ws": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _VP, ctypes.c_int32, _VP, _VP]),
    "pdas_solve_sweeps_ws_x0": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _I64, _VP, ctypes.c_int32,
                                               _VP, _VP]),
    "pdas_cascade_tile_width": (ctypes.c_int, [_I64]),
    "pdas_cascade_block_pivots": (ctypes.c_int, []),
    "pdas_cascade_solve_block": (ctypes.c_int, []),
    "pdas_cascade_one_cta": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64]),
    "pdas_cascade_solve_blocks": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int64]),
    "pdas_cascade_panel": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _I64, _I64, _VP,
                                          ctypes.c_int32, _VP, _VP]),
    "pdas_cascade_update": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _I64, _VP, _I64,
                                           _VP, _VP, _VP]),
    "pdas_cascade_panel_peers": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _I64, _I64, _VP,
                                                ctypes.c_int32, _VP, ctypes.c_int32, _VP, _VP, _VP,
                                                _VP]),
    "pdas_cascade_panel_chained": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _I64, _VP,
                                                  ctypes.c_int32, _VP, ctypes.c_int32, _VP]),
    "pdas_cascade_update_tagged": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _I64, _VP, _I64,
                                                  _VP, _VP, ctypes.c_int32, _VP]),
    "pdas_cascade_reset_tags": (ctypes.c_int, [_VP, _I64, _VP]),
    "pdas_cascade_peer_wait": (ctypes.c_int, [_VP, _I64, _I64, _I64, _I64, ctypes.c_int32, _VP]),
    "pdas_cholesky_solve_one": (ctypes.c_int, [_VP, _I64, _VP, _VP]),
    "pdas_iter_reset": (ctypes.c_int, [_VP, _VP]),
    "pdas_iter_scaling": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "pdas_iter_directions": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _D, _VP, _VP]),
    "pdas_ratio_test": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _D, _VP, _VP]),
    "pdas_iter_update": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _VP, _VP]),
    "pdas_iter_objectives": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _I64, _I64, _VP, _VP]),
    "pdas_probe_fp64": (ctypes.c_int, [_VP, _I64, _VP, _VP]),
    "pdas_selftest_div": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "pdas_debug_cascade_profile": (ctypes.c_int64, [_VP, _I64]),
}

_LIB = None


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing or a CUDA call failed (no CPU fallback)."""


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpdas_b200.so and declare every exported signature."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} is missing: build it with `make -C paper_1502_03543_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pdas_abi_version() != 1:
        raise NativeLibraryError("libpdas_b200.so ABI version mismatch")
    _LIB = lib
    return lib


def last_error() -> str:
    return (load().pdas_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != PDAS_OK:
        raise NativeLibraryError(f"{what} failed ({rc}): {last_error()}")


def call(name: str, *args) -> None:
    """Call an entry point and raise on a non-OK status."""
    check(getattr(load(), name)(*args), name)
