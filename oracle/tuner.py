"""Oracle of the paper's tuning rules and of the tile-DAG schedule (plain Python).

*** TEST INFRASTRUCTURE ONLY *** (see oracle/__init__.py).

Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
Readings of unclear points are DESIGN.md R13/R14.
"""
from __future__ import annotations

from fractions import Fraction


def orthogonal_prune(samples, tie_rel: float = 0.0):
    """Property 1: per NB keep the IB with the highest rate.

    samples: iterable of (nb, ib, gflops).  Ties -> larger IB; with
    tie_rel > 0 every IB whose rate is >= (1 - tie_rel) * the NB's best rate
    counts as tied (R18: rates closer than the timing's
    repeatability are not distinguishable).  Returns [(nb, ib, gflops)] sorted
    by nb, gflops being the kept IB's own rate.
    """
    rates = {}
    for nb, ib, g in samples:
        rates.setdefault(nb, []).append((ib, g))
    if not rates:
        raise ValueError("empty dataset")
    out = []
    for nb in sorted(rates):
        gmax = max(g for _, g in rates[nb])
        ib, g = max((ib, g) for ib, g in rates[nb] if g >= gmax * (1.0 - tie_rel))
        out.append((nb, ib, g))
    return out


def _cross(o, a, b):
    return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])


def upper_hull(points):
    """Property 2 / Heuristic 0: upper convex hull of (nb, gflops).

    points: [(nb, ib, gflops)] with distinct nb.  Returns the hull vertices in
    increasing nb with strictly decreasing segment slopes (collinear interior
    points dropped); both endpoints are always kept.
    Monotone chain, exact arithmetic via Fraction.
    """
    pts = sorted(points)
    hull = []
    for p in pts:
        q = (Fraction(p[0]), Fraction(p[2]))
        while len(hull) >= 2:
            o = (Fraction(hull[-2][0]), Fraction(hull[-2][2]))
            a = (Fraction(hull[-1][0]), Fraction(hull[-1][2]))
            if _cross(o, a, q) >= 0:  # a on or below chord o->q: not a strict upper vertex
                hull.pop()
            else:
                break
        hull.append(p)
    return hull


def incoming_slopes(hull):
    """Incoming steepness of every hull point: the slope of the hull
    segment ending at it; the first point's segment starts at the origin (0, 0)
    (R13: a tile of order 0 runs at 0 Gflop/s)."""
    out = [Fraction(hull[0][2]) / Fraction(hull[0][0])]
    return out + [Fraction(hull[i][2] - hull[i - 1][2]) / Fraction(hull[i][0] - hull[i - 1][0])
                  for i in range(1, len(hull))]


def heuristic1(hull, cap: int = 8):
    """Heuristic 1: the points after the `cap` steepest hull segments
    (the first point's segment starts at the origin, R13).
    Ties on slope -> smaller nb."""
    s = incoming_slopes(hull)
    order = sorted(range(len(hull)), key=lambda i: (-s[i], hull[i][0]))
    pick = sorted(order[:cap])
    return [hull[i] for i in pick]


def heuristic2(hull, cap: int = 8):
    """Heuristic 2: split [min nb, max nb] into `cap` equal
    half-open intervals (last closed) and keep, in each, the hull point with
    the largest incoming slope (the first point's slope from the origin,
    DESIGN.md R13)."""
    if len(hull) == 1:
        return list(hull)
    s = incoming_slopes(hull)
    x0, x1 = Fraction(hull[0][0]), Fraction(hull[-1][0])
    width = (x1 - x0) / cap
    best = {}
    for i in range(len(hull)):
        x = Fraction(hull[i][0])
        seg = cap - 1 if x == x1 else int((x - x0) // width)
        cur = best.get(seg)
        if cur is None or s[i] > s[cur]:
            best[seg] = i
    return [hull[i] for i in sorted(best.values())]


def preselect(samples, heuristic: int = 2, cap: int = 8, tie_rel: float = 0.0):
    """Step 1 pre-selection: Property 1 -> hull -> H0/H1/H2."""
    hull = upper_hull(orthogonal_prune(samples, tie_rel))
    if heuristic == 0:
        return hull
    if heuristic == 1:
        return heuristic1(hull, cap)
    if heuristic == 2:
        return heuristic2(hull, cap)
    raise ValueError("heuristic must be 0, 1 or 2")


def payg_prune(results):
    """Property 3 / PSPAYG: drop (nb2, ib2) when some nb1 > nb2 is
    strictly faster at this N.  results: [(nb, ib, gflops)].  Order-independent."""
    keep = []
    for nb2, ib2, g2 in results:
        if not any(nb1 > nb2 and g1 > g2 for nb1, _, g1 in results):
            keep.append((nb2, ib2, g2))
    return keep


def nearest(values, x):
    """Per-axis nearest grid value, ties toward the larger value."""
    return min(values, key=lambda v: (abs(v - x), -v))


def lookup(table, n: int, ncores: int):
    """Nearest-point interpolation: table {(n, c): (nb, ib)}."""
    ns = sorted({k[0] for k in table})
    cs = sorted({k[1] for k in table})
    return table[(nearest(ns, n), nearest(cs, ncores))]


def plan_cores(max_cores: int):
    """Powers of two plus the maximum."""
    out, c = [], 1
    while c <= max_cores:
        out.append(c)
        c *= 2
    if out[-1] != max_cores:
        out.append(max_cores)
    return out


def dag_levels(mt: int, nt: int):
    """ASAP level of every task of the flat-tree tile QR DAG, by an explicit
    dependency DP (nodes are tile tasks, edges data dependencies).

    Tasks: ('G',k), ('L',k,n), ('T',k,m), ('S',k,m,n).  Each task depends on
    the last task that wrote each tile it reads or writes.
    Returns dict task -> level (0-based)."""
    last_write = {}  # tile (i, j) -> level of last writer
    # the diagonal tile is split: its strict lower (V_kk, read by L) and its
    # upper triangle (R_kk, written by T); L(k,n) must only wait for G(k).
    level = {}

    def dep(*tiles):
        return max([last_write.get(t, -1) for t in tiles], default=-1) + 1

    for k in range(min(mt, nt)):
        g = dep((k, k), (k, k, "U"), (k, k, "L"))
        level[("G", k)] = g
        last_write[(k, k, "U")] = g
        last_write[(k, k, "L")] = g
        for n in range(k + 1, nt):
            lv = max(dep((k, n)), last_write[(k, k, "L")] + 1)
            level[("L", k, n)] = lv
            last_write[(k, n)] = lv
        for m in range(k + 1, mt):
            t = dep((k, k, "U"), (m, k))
            level[("T", k, m)] = t
            last_write[(k, k, "U")] = t
            last_write[(m, k)] = t
            for n in range(k + 1, nt):
                s = max(dep((k, n), (m, n)), t + 1)
                level[("S", k, m, n)] = s
                last_write[(k, n)] = s
                last_write[(m, n)] = s
    return level
