"""The C-ABI boundary: libpdas_b200.so loads (no GPU needed) and exports every
symbol include/pdas_b200.h declares, with the ctypes signatures in _lib.py
covering exactly that set; the header's struct layout matches ctypes."""

import ctypes
import os
import re

from conftest import REPO

HEADER = os.path.join(REPO, "include", "pdas_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdas_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_kernel_table():
    syms = declared_symbols()
    for name in ("dot_tree", "mat_vec", "mat_t_vec", "gram", "scaled_gram", "cholesky_factor",
                 "cholesky_solve_many", "build_v", "sweep_phase1", "sweep_phase2",
                 "solve_sweeps"):
        assert f"pdas_{name}" in syms


def test_library_loads_and_exports_every_symbol():
    from paper_1502_03543_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert syms, "no symbols parsed from the header"
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == syms
    assert lib.pdas_abi_version() == 1
    assert lib.pdas_cascade_max_m() >= 2000


def test_state_struct_layout():
    from paper_1502_03543_b200 import _lib

    assert ctypes.sizeof(_lib.PdasIterState) == 2 * 8 + 6 * 4 + 8 * 8
    assert _lib.OFF_CHOL_FAIL == 0 and _lib.OFF_CASCADE_FAIL == 16


def test_library_is_sm100a():
    """The shared object carries sm_100a SASS (cuobjdump when available)."""
    import shutil
    import subprocess

    so = os.path.join(REPO, "paper_1502_03543_b200", "libpdas_b200.so")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    out = subprocess.run([tool, "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_cascade_schedule_queries():
    """Host-only queries of the 1-GPU cascade's schedule (no GPU needed): the
    one-CTA cascade for m <= 64 when [Y|x] + A fit, else pivot blocks of 256
    then 512 (cascade.cu run_cascade_impl)."""
    from paper_1502_03543_b200 import _lib

    lib = _lib.load()
    assert lib.pdas_cascade_one_cta(50, 200) == 1       # c1
    assert lib.pdas_cascade_one_cta(64, 400) == 0       # [Y|x] + A > 200 KB
    assert lib.pdas_cascade_one_cta(65, 100) == 0
    assert lib.pdas_cascade_solve_block() == 256
    assert lib.pdas_cascade_solve_blocks(50, 200) == 0  # one kernel
    for n, nb in ((100, 1), (256, 1), (257, 2), (768, 2), (769, 3), (20000, 40),
                  (100000, 196)):
        assert lib.pdas_cascade_solve_blocks(2000, n) == nb, n
