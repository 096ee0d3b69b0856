"""Pins of the oracle's tall-skinny / communication-avoiding variant (SURVEY
§8(f) f3): TTQRT / TTMQRT and the tree tile QR of
DESIGN.md R20, against things other than the oracle itself:
  * LAPACK computes the same kernels: dtpqrt / dtpmqrt with L = NB (the
    pentagonal B is then upper triangular);
  * the same tree QR composed from LAPACK kernels in the test (dgeqrt,
    dtpqrt(l=0), dtpqrt(l=NB), dgemqrt, dtpmqrt) -- an independent
    implementation of every step;
  * numpy.linalg.qr (sign-normalised R), R^T R = A^T A, residual and
    orthogonality of the Q the oracle applies;
  * the special case BS >= MT, which is the flat tree (bitwise the pinned
    oracle_tileqr_factor, T2 = 0).
"""
import numpy as np
import pytest
import scipy.linalg.lapack as lapack

import oracle
import synth_inputs as si
from _tq import EPS, nrel

TT_CASES = [(8, 1), (8, 4), (8, 8), (12, 3), (16, 4), (32, 8), (64, 16), (96, 24), (128, 32)]


def tol(nb):
    return 100 * nb * EPS


@pytest.mark.parametrize("nb,ib", TT_CASES)
def test_ttqrt_matches_lapack_dtpqrt_l_nb(nb, ib):
    r0 = np.triu(si.uniform(nb, nb, 700 + nb)) + np.tril(np.full((nb, nb), 9.0), -1)
    b0 = np.triu(si.uniform(nb, nb, 800 + ib)) + np.tril(np.full((nb, nb), 7.0), -1)
    r, v2, t = oracle.ttqrt(r0, b0, ib)
    rl, vl, tl, info = lapack.dtpqrt(nb, ib, np.triu(r0), np.triu(b0))
    assert info == 0
    assert nrel(np.triu(r), np.triu(rl)) < tol(nb)
    assert nrel(np.triu(v2), np.triu(vl)) < tol(nb)
    assert nrel(t, tl) < tol(nb)
    # strict lower parts (another kernel's V in the tile layout) never touched
    assert np.array_equal(np.tril(r, -1), np.tril(r0, -1))
    assert np.array_equal(np.tril(v2, -1), np.tril(b0, -1))


@pytest.mark.parametrize("nb,ib", TT_CASES)
@pytest.mark.parametrize("trans", ["T", "N"])
def test_ttmqrt_matches_lapack_dtpmqrt_l_nb(nb, ib, trans):
    r0 = np.triu(si.uniform(nb, nb, 900 + nb))
    b0 = np.triu(si.uniform(nb, nb, 901 + ib))
    _, v2, t = oracle.ttqrt(r0, b0, ib)
    v2 = np.triu(v2) + np.tril(np.full((nb, nb), 5.0), -1)   # junk below: must be ignored
    c1, c2 = si.uniform(nb, 11, 902), si.uniform(nb, 11, 903)
    o1, o2 = oracle.ttmqrt(v2, t, c1, c2, trans)
    l1, l2, info = lapack.dtpmqrt(nb, np.triu(v2), t, c1, c2, "L", trans)
    assert info == 0
    assert nrel(o1, l1) < tol(nb) and nrel(o2, l2) < tol(nb)


def test_ttqrt_closed_form_identity_on_identity():
    """[I; I] -> R = -sqrt(2) I, V2 = (sqrt(2) - 1) I, T = diag(1 + 1/sqrt(2)):
    the same closed form as TSQRT (the bottom is already triangular)."""
    nb = 8
    r, v2, t = oracle.ttqrt(np.eye(nb), np.eye(nb), 4)
    s2 = np.sqrt(2.0)
    np.testing.assert_allclose(np.triu(r), -s2 * np.eye(nb), atol=1e-15)
    np.testing.assert_allclose(np.triu(v2), (s2 - 1) * np.eye(nb), atol=1e-15)
    for p in range(2):
        np.testing.assert_allclose(t[:, 4 * p:4 * p + 4], (1 + 1 / s2) * np.eye(4), atol=1e-15)


def lapack_tree_qr(a, nb, ib, bs):
    """The tree tile QR of DESIGN.md R20 composed from LAPACK kernels (every
    dimension a multiple of nb): returns (R/V tiles, T, T2)."""
    m, n = a.shape
    mt, nt = m // nb, n // nb
    A = np.array(a, order="F")
    T = np.zeros((mt, nt, ib, nb))
    T2 = np.zeros((mt, nt, ib, nb))
    tile = lambda i, j: A[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]  # noqa: E731

    def put(i, j, v):
        A[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb] = v

    for k in range(min(mt, nt)):
        heads = oracle.tree_heads(mt, k, bs)
        for h in heads:
            end = min((h // bs + 1) * bs, mt)
            g, t, _ = lapack.dgeqrt(ib, tile(h, k))
            put(h, k, g)
            T[h, k] = t
            for j in range(k + 1, nt):
                c, _ = lapack.dgemqrt(np.tril(g, -1) + np.eye(nb), t, tile(h, j), "L", "T")
                put(h, j, c)
            for i in range(h + 1, end):
                r, v, t2, _ = lapack.dtpqrt(0, ib, np.triu(tile(h, k)), tile(i, k))
                put(h, k, np.triu(r) + np.tril(tile(h, k), -1))
                put(i, k, v)
                T[i, k] = t2
                for j in range(k + 1, nt):
                    c1, c2, _ = lapack.dtpmqrt(0, v, t2, tile(h, j), tile(i, j), "L", "T")
                    put(h, j, c1)
                    put(i, j, c2)
        s = 1
        while s < len(heads):
            for q in range(0, len(heads) - s, 2 * s):
                a_, b_ = heads[q], heads[q + s]
                r, v, t2, _ = lapack.dtpqrt(nb, ib, np.triu(tile(a_, k)), np.triu(tile(b_, k)))
                put(a_, k, np.triu(r) + np.tril(tile(a_, k), -1))
                put(b_, k, np.triu(v) + np.tril(tile(b_, k), -1))
                T2[b_, k] = t2
                for j in range(k + 1, nt):
                    c1, c2, _ = lapack.dtpmqrt(nb, np.triu(v), t2, tile(a_, j), tile(b_, j), "L", "T")
                    put(a_, j, c1)
                    put(b_, j, c2)
            s *= 2
    return A, T, T2


def split_t(t, m, n, nb, ib):
    mt, nt = m // nb, n // nb
    half = t.size // 2
    out = []
    for part in (t[:half], t[half:]):
        x = np.zeros((mt, nt, ib, nb))
        for k in range(nt):
            for i in range(mt):
                o = (i + k * mt) * ib * nb
                x[i, k] = part[o:o + ib * nb].reshape((ib, nb), order="F")
        out.append(x)
    return out


@pytest.mark.parametrize("m,n,nb,ib,bs", [(40, 16, 8, 4, 1), (40, 16, 8, 4, 2), (48, 24, 8, 2, 3),
                                          (64, 32, 16, 4, 1), (96, 32, 16, 8, 4), (56, 56, 8, 4, 2)])
def test_tree_qr_matches_lapack_composition(m, n, nb, ib, bs):
    a = si.uniform(m, n, 1000 + m + bs)
    f, t, info = oracle.tileqr_factor_tree(a, nb, ib, bs)
    assert info == 0
    fl, tl, t2l = lapack_tree_qr(a, nb, ib, bs)
    to, t2o = split_t(t, m, n, nb, ib)
    assert nrel(f, fl) < 1e-13
    assert nrel(to, tl) < 1e-13 and nrel(t2o, t2l) < 1e-13


@pytest.mark.parametrize("m,n,nb,ib,bs", [(250, 60, 16, 4, 1), (250, 60, 16, 8, 3), (300, 300, 32, 8, 2),
                                          (37, 5, 8, 2, 1), (520, 100, 64, 16, 2)])
def test_tree_qr_properties(m, n, nb, ib, bs):
    a = si.uniform(m, n, 2000 + m)
    f, t, _ = oracle.tileqr_factor_tree(a, nb, ib, bs)
    k = min(m, n)
    r = np.triu(f[:k, :])
    # sign-normalised R unique for full-rank A (numpy.linalg.qr)
    rq = np.linalg.qr(a, mode="r")
    sgn = lambda x: np.where(np.diag(x) < 0, -1.0, 1.0)[:, None] * x  # noqa: E731
    assert nrel(sgn(r), sgn(rq)) < 1e-12
    assert nrel(r.T @ r, a.T @ a) < 1e-13
    q = oracle.tileqr_apply_tree("N", f, t, nb, ib, bs, np.eye(m))
    assert np.linalg.norm(a - q[:, :k] @ r) / (np.linalg.norm(a) * max(m, n) * EPS) < 10
    assert np.linalg.norm(q.T @ q - np.eye(m)) / (m * EPS) < 10
    qta = oracle.tileqr_apply_tree("T", f, t, nb, ib, bs, a)
    assert nrel(qta[:k], r) < 1e-13 and np.linalg.norm(qta[k:]) < 1e-12


def test_tree_with_one_domain_is_the_flat_tree():
    a = si.uniform(200, 90, 31)
    for nb, ib in [(16, 4), (32, 8)]:
        f0, t0, _ = oracle.tileqr_factor(a, nb, ib)
        f1, t1, _ = oracle.tileqr_factor_tree(a, nb, ib, 1000)
        assert np.array_equal(f0, f1) and np.array_equal(t0, t1[:t0.size]) and not t1[t0.size:].any()


def test_tree_heads():
    assert oracle.tree_heads(10, 0, 3) == [0, 3, 6, 9]
    assert oracle.tree_heads(10, 4, 3) == [4, 6, 9]
    assert oracle.tree_heads(10, 3, 1) == list(range(3, 10))
    assert oracle.tree_heads(10, 2, 100) == [2]
