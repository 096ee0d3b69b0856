"""Pins of the oracle's tuning rules and DAG schedule.

Expected values: SPEC.md worked examples (S:255-287, S:355, S:374-376,
S:442), O(n^3) brute-force hull membership written here, a hand-derived DAG
for 2x2 tiles, and the paper's own Istanbul tables reproducing
Table 2's 97.1 % / 7 of 16.
"""
import itertools
import os
import random
from fractions import Fraction

import pytest

from oracle import tuner

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_orthogonal_prune_spec_example():
    out = tuner.orthogonal_prune([(64, 16, 5.0), (64, 32, 6.0), (128, 32, 7.0)])
    assert out == [(64, 32, 6.0), (128, 32, 7.0)]


def test_orthogonal_prune_tie_to_larger_ib():
    assert tuner.orthogonal_prune([(64, 8, 5.0), (64, 32, 5.0), (64, 16, 5.0)]) == [(64, 32, 5.0)]


def test_orthogonal_prune_brute_force():
    rnd = random.Random(1)
    for _ in range(50):
        s = [(rnd.choice([64, 96, 128]), rnd.randint(1, 64), float(rnd.randint(0, 20))) for _ in range(30)]
        out = tuner.orthogonal_prune(s)
        for nb, ib, g in out:
            grp = [x for x in s if x[0] == nb]
            assert g == max(x[2] for x in grp)
            assert ib == max(x[1] for x in grp if x[2] == g)


def test_orthogonal_prune_tie_width():  # DESIGN.md R18 (Step-1 rates of a B200 run, NB=128)
    s = [(128, 8, 28394.0), (128, 16, 28379.0), (128, 32, 27771.0)]
    assert tuner.orthogonal_prune(s) == [(128, 8, 28394.0)]             # exact rule: the argmax
    assert tuner.orthogonal_prune(s, 0.005) == [(128, 16, 28379.0)]     # 0.05 % apart: tied, larger IB
    assert tuner.orthogonal_prune(s, 0.05) == [(128, 32, 27771.0)]      # 2.2 % apart: tied at 5 %


def test_orthogonal_prune_tie_width_brute_force():
    rnd = random.Random(2)
    for _ in range(50):
        tie = rnd.choice([0.0, 0.01, 0.1, 0.5])
        s = [(rnd.choice([64, 96, 128]), rnd.randint(1, 64), float(rnd.randint(1, 20))) for _ in range(30)]
        for nb, ib, g in tuner.orthogonal_prune(s, tie):
            grp = [x for x in s if x[0] == nb]
            top = max(x[2] for x in grp)
            tied = [x for x in grp if x[2] >= top * (1 - tie)]
            assert ib == max(x[1] for x in tied)
            assert g == max(x[2] for x in tied if x[1] == ib)


def P(x, y):
    return (x, 0, y)


def test_hull_spec_examples():
    h = tuner.upper_hull([P(1, 1), P(2, 3), P(3, 3.5), P(4, 5)])
    assert [(p[0], p[2]) for p in h] == [(1, 1), (2, 3), (4, 5)]
    assert len(tuner.upper_hull([P(1, 1), P(2, 5)])) == 2
    h = tuner.upper_hull([P(1, 1), P(2, 2), P(3, 3)])
    assert [(p[0], p[2]) for p in h] == [(1, 1), (3, 3)]


def _brute_hull(pts):
    """x is a strict upper-hull vertex iff no chord between two other points
    (one left, one right) lies on or above it; endpoints always in."""
    xs = sorted(pts)
    out = []
    for i, p in enumerate(xs):
        if i in (0, len(xs) - 1):
            out.append(p)
            continue
        dominated = False
        for a, b in itertools.product(xs[:i], xs[i + 1:]):
            t = Fraction(p[0] - a[0], b[0] - a[0])
            if Fraction(a[2]) + t * (Fraction(b[2]) - Fraction(a[2])) >= Fraction(p[2]):
                dominated = True
                break
        if not dominated:
            out.append(p)
    return out


def test_hull_brute_force_and_invariants():
    rnd = random.Random(2)
    for _ in range(300):
        n = rnd.randint(1, 25)
        xs = rnd.sample(range(2, 600, 2), n)
        pts = [(x, 1, float(rnd.randint(0, 40))) for x in xs]
        h = tuner.upper_hull(pts)
        assert h == _brute_hull(pts)
        s = tuner.incoming_slopes(h)
        assert all(s[i] > s[i + 1] for i in range(1, len(s) - 1))


def _hull(xs, ys):
    return [(x, 1, y) for x, y in zip(xs, ys)]


def test_heuristic1_examples():  # S:275-277, with reading R13 (first slope from the origin)
    h = _hull([1, 2, 3], [0.0, 0.9, 1.0])
    assert [p[0] for p in tuner.heuristic1(h)] == [1, 2, 3]  # |hull| <= cap: all selected
    assert [p[0] for p in tuner.heuristic1(h, 2)] == [2, 3]  # first point: slope 0 from origin
    xs = list(range(10, 130, 10))
    ys = [0.0]
    for i in range(1, 12):
        ys.append(ys[-1] + (12 - i))  # concave increasing: slopes decrease
    h = _hull(xs, ys)
    assert [p[0] for p in tuner.heuristic1(h, 8)] == xs[1:9]
    assert [p[0] for p in tuner.heuristic1(h, 1)] == [20]


def test_heuristic2_examples():
    xs = [40, 80, 120, 160, 200, 240]
    ys = [0, 10, 18, 24, 28, 30]
    h = _hull(xs, ys)
    assert [p[0] for p in tuner.heuristic2(h, 2)] == [80, 160]
    assert [p[0] for p in tuner.heuristic2(h, 8)] == xs  # first point (y=0) alone in its segment
    h = _hull([10, 11, 12, 100], [0, 5, 8, 9])
    assert [p[0] for p in tuner.heuristic2(h, 1)] == [11]


def test_first_hull_point_selectable_from_origin():
    """Reading R13: the smallest NB carries the slope of the segment from the
    origin, so a steep start (the usual small-N optimum) is pre-selected."""
    h = _hull([64, 128, 224, 256], [20.0, 24.0, 22.7, 21.8])[:2]
    assert [p[0] for p in tuner.heuristic2(h, 8)] == [64, 128]
    assert [p[0] for p in tuner.heuristic1(h, 1)] == [64]


def test_heuristic_caps_and_subsets():
    rnd = random.Random(3)
    for _ in range(100):
        xs = sorted(rnd.sample(range(2, 512, 2), rnd.randint(2, 40)))
        pts = [(x, 1, float(rnd.randint(0, 100))) for x in xs]
        hull = tuner.upper_hull(pts)
        h1, h2 = tuner.heuristic1(hull), tuner.heuristic2(hull)
        assert len(h1) <= 8 and len(h2) <= 8
        assert set(h1) <= set(hull) and set(h2) <= set(hull)


def test_payg_prune_spec_examples():
    out = tuner.payg_prune([(96, 1, 10.0), (168, 1, 12.0), (300, 1, 9.0)])
    assert [p[0] for p in out] == [168, 300]
    assert len(tuner.payg_prune([(96, 1, 5.0), (168, 1, 5.0)])) == 2


def test_lookup_paper_example():
    ns = [500, 1000, 2000, 4000, 6000, 8000, 10000]
    cs = tuner.plan_cores(48)
    table = {(n, c): (n, c) for n in ns for c in cs}
    assert tuner.lookup(table, 1800, 5) == (2000, 4)
    assert tuner.lookup(table, 1500, 48) == (2000, 48)  # tie -> larger
    assert tuner.plan_cores(48) == [1, 2, 4, 8, 16, 32, 48]
    assert tuner.plan_cores(16) == [1, 2, 4, 8, 16] and tuner.plan_cores(1) == [1]


def test_dag_levels_2x2_by_hand():
    lv = tuner.dag_levels(2, 2)
    assert lv == {("G", 0): 0, ("L", 0, 1): 1, ("T", 0, 1): 1, ("S", 0, 1, 1): 2, ("G", 1): 3}


@pytest.mark.parametrize("mt,nt", [(1, 1), (4, 4), (5, 5), (8, 8), (6, 3), (3, 6), (7, 2)])
def test_dag_levels_closed_form(mt, nt):
    # Closed form the CUDA launcher uses: G=3k, L=3k+1,
    # T=2k+m, S=2k+m+1; the DP above is the definition it must agree with.
    lv = tuner.dag_levels(mt, nt)
    for task, v in lv.items():
        kind, k = task[0], task[1]
        exp = {"G": 3 * k, "L": 3 * k + 1}.get(kind)
        if kind == "T":
            exp = 2 * k + task[2]
        if kind == "S":
            exp = 2 * k + task[2] + 1
        assert v == exp, task


def _read_table(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if line and not line.startswith("#") and not line.startswith("n,"):
            rows.append([float(x) for x in line.split(",")])
    return rows


def test_istanbul_h2_pspayg_reproduces_table2():
    """Table 2: Istanbul H2+PSPAYG averages 97.1 % of ES and finds
    the optimum in 7 of 16 cases; recomputed from the appendix tables."""
    es = {(int(r[0]), int(r[1])): r[2] for r in _read_table("istanbul_es.csv")}
    h2 = {(int(r[0]), int(r[1])): r[2] for r in _read_table("istanbul_h2_pspayg.csv")}
    assert set(es) == set(h2) and len(es) == 16
    ratios = [100.0 * h2[k] / es[k] for k in es]
    assert round(sum(ratios) / 16, 1) == 97.1
    assert sum(1 for k in es if h2[k] == es[k]) == 7
