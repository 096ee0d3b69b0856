"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its pure host logic (argument errors, level count,
tuner pruning) agrees with the oracle -- no GPU compute is called here."""
import ctypes
import random
import re
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import build
    build.build()
    from paper_1102_5328_b200 import tileqr
    return tileqr


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tileqr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tileqr_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol(tq):
    lib = ctypes.CDLL(tq.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(tq.EXPORTED)


def test_version_and_t_size(tq):
    assert "sm_100a" in tq.version()
    assert tq.t_size(256, 256, 64, 16) == 4 * 4 * 16 * 64
    assert tq.t_size(250, 190, 64, 8) == 4 * 3 * 8 * 64
    with pytest.raises(tq.TileQRError, match="returned -4"):
        tq.t_size(10, 10, 64, 7)  # IB must divide NB
    with pytest.raises(tq.TileQRError, match="returned -3"):
        tq.t_size(10, 10, 513, 1)


def test_factor_argument_errors_need_no_gpu(tq):
    lib = ctypes.CDLL(tq.LIB_PATH)
    f = lib.tileqr_factor
    f.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                  ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    assert f(-1, 4, 8, 4, 2, 1, 8, None, None) == -1
    assert f(4, -1, 8, 4, 2, 1, 8, None, None) == -2
    assert f(4, 4, None, 4, 2, 1, 8, None, None) == -3
    assert f(4, 4, 8, 3, 2, 1, 8, None, None) == -4
    assert f(4, 4, 8, 4, 0, 1, 8, None, None) == -5
    assert f(4, 4, 8, 4, 4, 3, 8, None, None) == -6
    assert f(4, 4, 8, 4, 4, 2, None, None, None) == -7
    assert "illegal argument 7" in tq.last_error()


def test_num_levels_matches_oracle_dp(tq):
    from oracle.tuner import dag_levels
    for mt, nt in [(1, 1), (2, 2), (4, 4), (5, 5), (16, 16), (6, 3), (3, 6), (7, 2), (2, 7)]:
        assert tq.num_levels(mt, nt) == max(dag_levels(mt, nt).values()) + 1
    assert tq.num_levels(79, 79) == 235 and tq.num_levels(250, 250) == 748


def test_preselect_matches_oracle(tq):
    from oracle import tuner
    rnd = random.Random(7)
    for trial in range(200):
        nbs = rnd.sample(range(2, 520, 2), rnd.randint(1, 20))
        samples = []
        for nb in nbs:
            for ib in rnd.sample(range(1, 65), rnd.randint(1, 4)):
                samples.append((nb, ib, float(rnd.randint(0, 60))))
        for h in (0, 1, 2):
            cap = rnd.choice([1, 2, 8])
            got = tq.preselect(samples, h, cap)
            exp = tuner.preselect(samples, h, cap)
            assert got == exp, (trial, h, cap)
            tie = rnd.choice([0.005, 0.05, 0.3])
            assert tq.preselect(samples, h, cap, tie) == tuner.preselect(samples, h, cap, tie), (trial, h, tie)


def test_payg_prune_matches_oracle(tq):
    from oracle import tuner
    rnd = random.Random(8)
    for _ in range(200):
        res = [(nb, 1, float(rnd.randint(0, 10))) for nb in rnd.sample(range(8, 512, 8), rnd.randint(1, 9))]
        assert tq.payg_prune(res) == tuner.payg_prune(res)


def test_lookup_matches_oracle_nearest_point(tq, tmp_path, monkeypatch):
    """tileqr_lookup (the library's decision-table interpolation, PAPER.md:631-635,
    826-832) against oracle.tuner.lookup on a (N, ngpus) grid, square queries;
    a rectangular query uses the square order of equal flop count (R19)."""
    import json
    from oracle import tuner
    rnd = random.Random(5)
    ns, gs = [500, 1000, 2000, 4000, 6000, 8000, 10000], [1, 2, 4, 8]
    pairs = [(64, 16), (96, 32), (128, 16), (160, 32), (192, 24), (256, 32)]
    table = {(n, g): rnd.choice(pairs) for n in ns for g in gs}
    path = tmp_path / "table.json"
    json.dump({"format_version": 1, "entries": [{"n": n, "ngpus": g, "nb": v[0], "ib": v[1]}
                                                for (n, g), v in table.items()]}, open(path, "w"))
    monkeypatch.setenv("TILEQR_TUNED_TABLE", str(path))
    for _ in range(300):
        n, g = rnd.randint(1, 12000), rnd.randint(1, 9)
        assert tq.lookup(n, n, g) == (*tuner.lookup(table, n, g), True), (n, g)
    for n in ns:  # on-grid points and exact midpoints (ties -> larger)
        assert tq.lookup(n, n, 1)[:2] == table[(n, 1)]
    assert tq.lookup(750, 750, 3)[:2] == table[(1000, 4)]
    # 40000 x 1000: (3/4 * (2*M*N^2 - 2N^3/3))^(1/3) = 3904 -> grid order 4000
    assert tq.lookup(40000, 1000, 1)[:2] == table[(4000, 1)]
    assert tq.t_size(300, 300, 0, 0) == tq.t_size(300, 300, *tq.lookup(300, 300)[:2])
    monkeypatch.setenv("TILEQR_TUNED_TABLE", str(tmp_path / "missing.json"))
    assert tq.lookup(1000, 1000) == (128, 16, False)


def test_installed_table_is_readable(tq):
    nb, ib, found = tq.lookup(10000, 10000)
    assert found and nb % ib == 0
