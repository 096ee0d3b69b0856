"""The tree variant's dataflow work list (tileqr_tree_plan_items: the task
graph tree.cu derives by last-writer tracking, in the claim order of its
schedule simulation) executed on the CPU with the oracle's tile kernels.

One worker walks the list in claim order; every dependency must already be
complete when an item is reached (the order is topological), every item
touches only what its task names, and the result must be BITWISE the
oracle's tree tile QR (oracle_tileqr_factor_tree, pinned in
test_oracle_tree.py): every tile sees the same kernels on the same inputs.
Panel tasks are whole tiles here (sub_cols = NB: the oracle kernels have no
inner-panel ranges); update slabs apply to their column ranges.
"""
import numpy as np
import pytest

import oracle
import synth_inputs as si

GEQRT, TSQRT, LARFB, SSRFB, TTQRT, TTMQR = 0, 1, 2, 3, 8, 9
COLS = {32: 32, 64: 32, 96: 64, 128: 64}  # update columns per item (dag_item.h dag_cols)


def run_plan(tq, m, n, nb, ib, bs, workers):
    mt, nt = m // nb, n // nb
    a = si.uniform(m, n, 70 + bs)
    tile = {(i, j): np.asfortranarray(a[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]) for i in range(mt) for j in range(nt)}
    t1, t2 = {}, {}
    rows = tq.tree_plan_items(m, n, nb, ib, bs, workers, nb)
    parts = {}
    for r in rows:
        parts[r[6]] = parts.get(r[6], 0) + 1
    count, done = {}, set()
    cols = COLS[nb]
    for kind, ta, tb, k, c, s, task, deps in rows:
        for d in deps:
            assert d in done, ("claimed before its input", kind, ta, tb, k, c, d)
        if kind == GEQRT:
            tile[(ta, k)], t1[(ta, k)] = oracle.geqrt(tile[(ta, k)], ib)
        elif kind == TSQRT:
            r_, v2, tt = oracle.tsqrt(tile[(ta, k)], tile[(tb, k)], ib)
            tile[(ta, k)] = np.asfortranarray(np.triu(r_) + np.tril(tile[(ta, k)], -1))
            tile[(tb, k)], t1[(tb, k)] = v2, tt
        elif kind == TTQRT:
            r_, v2, tt = oracle.ttqrt(tile[(ta, k)], tile[(tb, k)], ib)
            tile[(ta, k)], tile[(tb, k)], t2[(tb, k)] = r_, v2, tt
        else:
            j0, j1 = s * cols, min(nb, (s + 1) * cols)
            if kind == LARFB:
                cur = tile[(ta, c)].copy()
                cur[:, j0:j1] = oracle.larfb(tile[(ta, k)], t1[(ta, k)], cur[:, j0:j1], "T")
                tile[(ta, c)] = np.asfortranarray(cur)
            else:
                fn = oracle.ssrfb if kind == SSRFB else oracle.ttmqrt
                tt = t1[(tb, k)] if kind == SSRFB else t2[(tb, k)]
                c1, c2 = tile[(ta, c)].copy(), tile[(tb, c)].copy()
                c1[:, j0:j1], c2[:, j0:j1] = fn(tile[(tb, k)], tt, c1[:, j0:j1], c2[:, j0:j1], "T")
                tile[(ta, c)], tile[(tb, c)] = np.asfortranarray(c1), np.asfortranarray(c2)
        count[task] = count.get(task, 0) + 1
        if count[task] == parts[task]:
            done.add(task)
    f = np.zeros((m, n))
    for (i, j), v in tile.items():
        f[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb] = v
    return a, f, t1, t2


@pytest.mark.parametrize("m,n,nb,ib,bs,workers", [
    (512, 128, 64, 16, 1, 4),     # binary tree over 8 tile rows
    (640, 192, 64, 32, 2, 8),     # domains of 2
    (384, 384, 32, 8, 3, 16),     # square, 12 x 12 tiles
    (768, 256, 128, 16, 2, 3),
    (256, 512, 64, 16, 1, 4),     # wide
])
def test_tree_plan_executes_to_the_oracle_tree_qr(m, n, nb, ib, bs, workers):
    from paper_1102_5328_b200 import tileqr as tq
    a, f, t1, t2 = run_plan(tq, m, n, nb, ib, bs, workers)
    fo, to, _ = oracle.tileqr_factor_tree(a, nb, ib, bs)
    assert np.array_equal(f, fo)
    mt = m // nb
    half = to.size // 2
    for (i, k), t in t1.items():
        off = (i + k * mt) * ib * nb
        assert np.array_equal(t, to[off:off + ib * nb].reshape((ib, nb), order="F")), (i, k)
    for (i, k), t in t2.items():
        off = half + (i + k * mt) * ib * nb
        assert np.array_equal(t, to[off:off + ib * nb].reshape((ib, nb), order="F")), (i, k)


def test_tree_plan_counts():
    """Task counts of the derived graph: GEQRT per domain head, TSQRT per
    non-head row, one TTQRT per merge (heads - 1), and their updates."""
    from paper_1102_5328_b200 import tileqr as tq
    for m, n, nb, bs in [(1024, 256, 64, 3), (512, 512, 64, 1), (640, 320, 64, 100)]:
        mt, nt = m // nb, n // nb
        rows = tq.tree_plan_items(m, n, nb, 16, bs, 4, nb)
        kinds = {}
        for r in rows:
            if r[5] == 0:  # one row per task (slab / sub-task 0)
                kinds[r[0]] = kinds.get(r[0], 0) + 1
        heads = [len(oracle.tree_heads(mt, k, bs)) for k in range(min(mt, nt))]
        assert kinds.get(GEQRT, 0) == sum(heads)
        assert kinds.get(TSQRT, 0) == sum(mt - k - h for k, h in enumerate(heads))
        assert kinds.get(TTQRT, 0) == sum(h - 1 for h in heads)
        assert kinds.get(LARFB, 0) == sum(h * (nt - k - 1) for k, h in enumerate(heads))
        assert kinds.get(TTMQR, 0) == sum((h - 1) * (nt - k - 1) for k, h in enumerate(heads))
