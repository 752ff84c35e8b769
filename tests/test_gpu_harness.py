"""The reference's `check` / `bench` harnesses (cli.py:144-217) on the GPU path,
against the values the UNMODIFIED reference printed for the same seeds
(tests/golden/check.npz): the seeded systems, both solutions and the backend
gap bit for bit; the Z-residual (cuBLAS products here, numpy BLAS there) to
rounding, both far below the 1e-9 tolerance.  Plus the instance cache."""

import numpy as np
import pytest

from conftest import bits_equal, load_golden

pytestmark = pytest.mark.gpu


def _cases(g):
    return sorted({k.rsplit("/", 1)[0] for k in g.files})


def test_check_matches_reference_per_seed(gpu):
    from paper_1502_03543_b200 import harness as H

    g = load_golden("check.npz")
    for case in _cases(g):
        tag, seed = case.split("/")
        m, n = (None, None) if tag == "auto" else (20, 60)
        mm, nn, z, gap, wd, ww = H.check_system(int(seed), m, n)
        assert [mm, nn] == list(g[case + "/mn"]), case
        assert bits_equal(wd, g[case + "/w_direct"]) and bits_equal(ww, g[case + "/w_woodbury"])
        assert gap == float(g[case + "/gap"]), case
        zr = float(g[case + "/z"])
        assert z < 1e-9 and zr < 1e-9
        assert z <= max(100 * zr, 1e-13) and zr <= max(100 * z, 1e-13), (case, z, zr)


def test_check_command_exit_codes(gpu, capsys):
    from paper_1502_03543_b200.__main__ import main

    assert main(["check", "--seeds", "1..20"]) == 0
    assert "max Z-residual" in capsys.readouterr().out
    assert main(["check", "--seeds", "1..3", "--equiv-tol", "1e-300"]) in (0, 5)
    assert main(["check", "--seeds", "3..1"]) == 2
    assert main(["check", "--seeds", "1", "--m", "3", "--n", "2"]) == 2


def test_bench_rows(gpu):
    from paper_1502_03543_b200 import harness as H

    rows = H.run_bench([(10, 30)], seed=1, max_iter=3, out=lambda *_: None)
    assert rows[0] == "m,n,backend,workers,iterations,ms_per_iter"
    assert [r.split(",")[:5] for r in rows[1:]] == [["10", "30", "direct", "1", "3"],
                                                     ["10", "30", "woodbury", "1", "3"]]


def test_instance_cache_roundtrip(gpu, tmp_path):
    from paper_1502_03543_b200 import harness as H

    P = gpu
    lp0, s0 = P.gen_random_feasible(40, 120, 7)
    lp1, s1 = H.cached_instance(40, 120, 7, str(tmp_path))
    lp2, s2 = H.cached_instance(40, 120, 7, str(tmp_path))  # from disk
    for lp, st in ((lp1, s1), (lp2, s2)):
        assert bits_equal(lp.A.data, lp0.A.data) and bits_equal(lp.b, lp0.b)
        assert bits_equal(lp.c, lp0.c) and bits_equal(st.x, s0.x) and bits_equal(st.s, s0.s)
    path = tmp_path / "lp_m40_n120_s7.npz"
    path.write_bytes(b"corrupt")
    lp3, _ = H.cached_instance(40, 120, 7, str(tmp_path))  # regenerated
    assert bits_equal(lp3.A.data, lp0.A.data)
