"""GPU parity of the batched tile kernels (through the C ABI) against the oracle.

Each case runs a batch of independent seeded tiles through one
tileqr_*_batched call and compares every tile with the oracle's kernel on the
same inputs.  Tolerance: normwise relative 100*NB*eps.
Covers the DMMA path (NB % 32 == 0, <= 256) including odd / tiny IB, IB = NB,
partial ncols, both trans, and the SIMT path (other NB).
"""
import numpy as np
import pytest
import torch

import oracle
import synth_inputs as si
from _tq import EPS, nrel

pytestmark = pytest.mark.gpu

BATCH = 5
CASES = [(32, 8), (64, 16), (64, 1), (64, 64), (96, 12), (96, 3), (128, 32), (128, 128),
         (160, 10), (160, 40), (192, 48), (192, 64), (224, 7), (224, 56), (256, 32), (256, 256),
         (48, 6), (100, 25), (20, 5), (2, 1)]


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import tileqr
    return tileqr


def tol(nb):
    return 100 * nb * EPS


def dev_tiles(mats):
    """list of m x n numpy matrices -> (device storage, pointer tensor)."""
    bufs = [torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float64).T)).cuda() for m in mats]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    return bufs, ptrs


def host(buf):
    return buf.cpu().numpy().T


def seeds(nb, ib, k):
    return [si.uniform(nb, nb, 1000 + 17 * nb + ib, offset=(k * BATCH + i) * nb * nb) for i in range(BATCH)]


@pytest.mark.parametrize("nb,ib", CASES)
def test_geqrt_batched(tq, nb, ib):
    a = seeds(nb, ib, 0)
    ab, ap = dev_tiles(a)
    tb, tp = dev_tiles([np.zeros((ib, nb))] * BATCH)
    tq.geqrt_batched(nb, ib, ap, tp)
    torch.cuda.synchronize()
    for i in range(BATCH):
        ao, to = oracle.geqrt(a[i], ib)
        assert nrel(host(ab[i]), ao) < tol(nb), i
        assert nrel(host(tb[i]), to) < tol(nb), i


@pytest.mark.parametrize("nb,ib", CASES)
def test_tsqrt_batched(tq, nb, ib):
    r = [np.triu(x) + np.tril(np.full((nb, nb), 7.0), -1) for x in seeds(nb, ib, 1)]  # strict lower = V_kk stand-in
    b = seeds(nb, ib, 2)
    rb, rp = dev_tiles(r)
    bb, bp = dev_tiles(b)
    tb, tp = dev_tiles([np.zeros((ib, nb))] * BATCH)
    tq.tsqrt_batched(nb, ib, rp, bp, tp)
    torch.cuda.synchronize()
    for i in range(BATCH):
        ro, vo, to = oracle.tsqrt(r[i], b[i], ib)
        rg = host(rb[i])
        assert np.array_equal(np.tril(rg, -1), np.tril(r[i], -1)), "TSQRT wrote the strict lower part of R"
        assert nrel(np.triu(rg), np.triu(ro)) < tol(nb), i
        assert nrel(host(bb[i]), vo) < tol(nb), i
        assert nrel(host(tb[i]), to) < tol(nb), i


@pytest.mark.parametrize("nb,ib", CASES)
@pytest.mark.parametrize("trans", ["T", "N"])
def test_larfb_batched(tq, nb, ib, trans):
    vs, ts = [], []
    for x in seeds(nb, ib, 3):
        v, t = oracle.geqrt(x, ib)
        vs.append(v)
        ts.append(t)
    c = seeds(nb, ib, 4)
    ncols = nb if nb < 64 else nb - 5  # ragged column slab
    c = [x[:, :ncols] for x in c]
    vb, vp = dev_tiles(vs)
    tb, tp = dev_tiles(ts)
    cb, cp = dev_tiles([np.hstack([x, np.full((nb, nb - ncols), 3.0)]) for x in c])
    tq.larfb_batched(trans, nb, ib, vp, tp, cp, ncols)
    torch.cuda.synchronize()
    for i in range(BATCH):
        co = oracle.larfb(vs[i], ts[i], c[i], trans)
        g = host(cb[i])
        assert nrel(g[:, :ncols], co) < tol(nb), i
        assert np.all(g[:, ncols:] == 3.0), "columns beyond ncols were touched"


@pytest.mark.parametrize("nb,ib", CASES)
@pytest.mark.parametrize("trans", ["T", "N"])
def test_ssrfb_batched(tq, nb, ib, trans):
    v2s, ts = [], []
    for i, (x, y) in enumerate(zip(seeds(nb, ib, 5), seeds(nb, ib, 6))):
        _, v2, t = oracle.tsqrt(np.triu(x), y, ib)
        v2s.append(v2)
        ts.append(t)
    c1, c2 = seeds(nb, ib, 7), seeds(nb, ib, 8)
    ncols = nb if nb < 64 else nb - 3
    vb, vp = dev_tiles(v2s)
    tb, tp = dev_tiles(ts)
    c1b, c1p = dev_tiles(c1)
    c2b, c2p = dev_tiles(c2)
    tq.ssrfb_batched(trans, nb, ib, vp, tp, c1p, c2p, ncols)
    torch.cuda.synchronize()
    for i in range(BATCH):
        o1, o2 = oracle.ssrfb(v2s[i], ts[i], c1[i][:, :ncols], c2[i][:, :ncols], trans)
        g1, g2 = host(c1b[i]), host(c2b[i])
        assert nrel(g1[:, :ncols], o1) < tol(nb), i
        assert nrel(g2[:, :ncols], o2) < tol(nb), i
        assert np.array_equal(g1[:, ncols:], c1[i][:, ncols:])
        assert np.array_equal(g2[:, ncols:], c2[i][:, ncols:])


def test_ssrfb_zero_reflectors_is_identity(tq):
    nb, ib = 128, 32
    c1, c2 = seeds(nb, ib, 9), seeds(nb, ib, 10)
    vb, vp = dev_tiles([np.zeros((nb, nb))] * BATCH)
    tb, tp = dev_tiles([np.zeros((ib, nb))] * BATCH)
    c1b, c1p = dev_tiles(c1)
    c2b, c2p = dev_tiles(c2)
    tq.ssrfb_batched("T", nb, ib, vp, tp, c1p, c2p, nb)
    torch.cuda.synchronize()
    for i in range(BATCH):
        assert np.array_equal(host(c1b[i]), c1[i]) and np.array_equal(host(c2b[i]), c2[i])


def test_ssrfb_uses_dmma_path(tq):
    assert tq.ssrfb_impl(128, 32) == "dmma"
    assert tq.ssrfb_impl(100, 25) == "simt"


def test_rng_matches_synth_inputs(tq):
    m, n = 301, 77
    buf = torch.empty((n, 310), dtype=torch.float64, device="cuda")
    tq.rng_uniform(buf, m, n, seed=4, offset=123, lda=310)
    got = buf.cpu().numpy().T[:m, :]
    assert np.array_equal(got, si.uniform(m, n, 4, offset=123))  # bit-exact


PACKED = [(nb, ib) for nb in (32, 64, 96, 128, 160, 192, 224, 256) for ib in (8, 16, 24, 32) if nb % ib == 0]
# wide panels (IB > 32, one group per panel; one ring stage where two do not fit)
PACKED += [(64, 64), (96, 48), (128, 64), (160, 40), (192, 48), (192, 64), (224, 56), (256, 64)]


@pytest.mark.parametrize("nb,ib", PACKED)
@pytest.mark.parametrize("larfb", [False, True])
def test_packed_update_batched(tq, nb, ib, larfb):
    """The factorization's update kernel (packed reflector tiles, TMA-staged,
    barrier-free DMMA; update_v2.cuh) through tileqr_pack_batched +
    tileqr_update_packed_batched, against the oracle's SSRFB / LARFB (Q^T)."""
    assert tq.packed_size(nb, ib) > 0
    vs, ts = [], []
    for x, y in zip(seeds(nb, ib, 11), seeds(nb, ib, 12)):
        if larfb:
            v, t = oracle.geqrt(x, ib)
        else:
            _, v, t = oracle.tsqrt(np.triu(x), y, ib)
        vs.append(v)
        ts.append(t)
    c1, c2 = seeds(nb, ib, 13), seeds(nb, ib, 14)
    vb, vp = dev_tiles(vs)
    tb, tp = dev_tiles(ts)
    c1b, c1p = dev_tiles(c1)
    c2b, c2p = dev_tiles(c2)
    pk = torch.zeros(BATCH * tq.packed_size(nb, ib), dtype=torch.float64, device="cuda")
    pp = torch.arange(BATCH, dtype=torch.int64, device="cuda") * tq.packed_size(nb, ib) * 8 + pk.data_ptr()
    tq.pack_batched(larfb, nb, ib, vp, tp, pp)
    tq.update_packed_batched(larfb, nb, ib, pp, None if larfb else c1p, c2p)
    torch.cuda.synchronize()
    for i in range(BATCH):
        if larfb:
            o2 = oracle.larfb(vs[i], ts[i], c2[i], "T")
            assert nrel(host(c2b[i]), o2) < tol(nb), i
            assert np.array_equal(host(c1b[i]), c1[i])  # C1 untouched by the LARFB form
        else:
            o1, o2 = oracle.ssrfb(vs[i], ts[i], c1[i], c2[i], "T")
            assert nrel(host(c1b[i]), o1) < tol(nb), i
            assert nrel(host(c2b[i]), o2) < tol(nb), i


def test_packed_layout_is_a_permutation_of_v_and_t(tq):
    """The packed tile holds exactly the entries of V (unit lower trapezoid for
    the GEQRT form) and the upper triangles of the T_p blocks, nothing else."""
    nb, ib = 64, 16
    x = seeds(nb, ib, 15)[0]
    v, t = oracle.geqrt(x, ib)
    vb, vp = dev_tiles([v])
    tb, tp = dev_tiles([t])
    n = tq.packed_size(nb, ib)
    pk = torch.full((n,), 12345.0, dtype=torch.float64, device="cuda")
    pp = torch.tensor([pk.data_ptr()], dtype=torch.int64, device="cuda")
    tq.pack_batched(True, nb, ib, vp, tp, pp)
    torch.cuda.synchronize()
    got = np.sort(pk.cpu().numpy())
    vu = np.tril(v, -1) + np.eye(nb)                       # GEQRT reflectors, unit diagonal
    tt = [np.triu(t[:, p * ib:(p + 1) * ib]) for p in range(nb // ib)]
    want_nonzero = np.sort(np.concatenate([vu[vu != 0]] + [b[b != 0] for b in tt]))
    assert not np.any(got == 12345.0)                       # every slot written
    assert np.array_equal(got[got != 0], want_nonzero)


def test_packed_geometry_coverage(tq):
    """The packed update covers IB in {8, 16, 24, 32} and the wide panels whose
    two ring stages fit; the others report no packed form."""
    for nb, ib in PACKED:
        assert tq.packed_size(nb, ib) > 0, (nb, ib)
    for nb, ib in [(128, 128), (256, 128), (160, 80), (96, 12), (160, 10)]:
        assert tq.packed_size(nb, ib) == 0, (nb, ib)
