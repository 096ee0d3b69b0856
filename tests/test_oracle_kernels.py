"""Pins of the oracle's tile kernels against things other than itself.

Each test names what fixes the expected value: a closed form, a LAPACK
routine computing the same kernel (scipy: dgeqrt / dtpqrt(l=0) / dgemqrt /
dtpmqrt(l=0)), an explicitly formed product of Householder
matrices, or an algebraic identity (compact WY, Gram identity).
Tolerance for kernel agreement: 100*NB*eps normwise.
"""
import math

import numpy as np
import pytest
import scipy.linalg.lapack as lapack

import oracle
import synth_inputs as si
from _tq import EPS, nrel

CASES = [(8, 1), (8, 4), (8, 8), (12, 3), (15, 5), (14, 7), (64, 1), (64, 16), (64, 64),
         (96, 12), (160, 10), (128, 32)]


def tol(nb):
    return 100 * nb * EPS


# ---------------------------------------------------------------- reflector rule
def test_larfg_closed_form_3_4():
    beta, tau, v2 = oracle.larfg(3.0, [4.0])
    assert beta == -5.0 and tau == pytest.approx(1.6, abs=1e-15) and v2[0] == pytest.approx(0.5, abs=1e-15)


def test_larfg_zero_tail_is_identity():
    for alpha in (2.0, -3.0, 0.0):
        beta, tau, v2 = oracle.larfg(alpha, [0.0, 0.0, 0.0])
        assert tau == 0.0 and beta == alpha and not v2.any()


def test_larfg_negative_zero_alpha_takes_plus_sign():
    beta, tau, _ = oracle.larfg(-0.0, [1.0])
    assert beta == -1.0 and tau == 1.0


def test_larfg_reflects_to_beta_e1():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 33):
        x = rng.uniform(-1, 1, n + 1)
        beta, tau, v2 = oracle.larfg(x[0], x[1:])
        v = np.concatenate([[1.0], v2])
        hx = x - tau * v * (v @ x)
        assert abs(hx[0] - beta) < 1e-14 and np.abs(hx[1:]).max() < 1e-14
        assert abs(abs(beta) - np.linalg.norm(x)) < 1e-14


# ---------------------------------------------------------------- GEQRT
def test_geqrt_identity_tile():
    a, t = oracle.geqrt(np.eye(8), 2)
    assert np.array_equal(np.triu(a), np.eye(8)) and not np.tril(a, -1).any() and not t.any()


def test_geqrt_2x2_closed_form():  # SURVEY §8(c) pins: qr([[3,1],[4,2]])
    a, t = oracle.geqrt(np.array([[3.0, 1.0], [4.0, 2.0]]), 1)
    np.testing.assert_allclose(np.triu(a), [[-5.0, -2.2], [0.0, 0.4]], atol=1e-15)
    np.testing.assert_allclose(a[1, 0], 0.5, atol=1e-15)
    np.testing.assert_allclose(t, [[1.6, 0.0]], atol=1e-15)


@pytest.mark.parametrize("nb,ib", CASES)
def test_geqrt_matches_lapack_dgeqrt(nb, ib):
    a = si.uniform(nb, nb, 100 + nb + ib)
    ao, to = oracle.geqrt(a, ib)
    al, tl, info = lapack.dgeqrt(ib, a)
    assert info == 0
    assert nrel(ao, al) < tol(nb)
    assert nrel(to, tl) < tol(nb)
    for p in range(nb // ib):  # strictly-lower part of each IB x IB block is 0
        assert not np.tril(to[:, p * ib:(p + 1) * ib], -1).any()


def test_geqrt_r_independent_of_ib():
    a = si.uniform(48, 48, 3)
    r = [np.triu(oracle.geqrt(a, ib)[0]) for ib in (1, 4, 6, 48)]
    for x in r[1:]:
        assert nrel(x, r[0]) < 1e-13


def _householder_product(v_cols, taus, n):
    q = np.eye(n)
    for v, tau in zip(v_cols, taus):
        q = q @ (np.eye(n) - tau * np.outer(v, v))
    return q


def _geqrt_reflectors(a, t, ib):
    nb = a.shape[0]
    vs, taus = [], []
    for j in range(nb):
        v = np.zeros(nb)
        v[j] = 1.0
        v[j + 1:] = a[j + 1:, j]
        vs.append(v)
        taus.append(t[j % ib, j])
    return vs, taus


@pytest.mark.parametrize("nb,ib", [(16, 4), (12, 3), (20, 20)])
def test_geqrt_reconstructs_tile(nb, ib):
    a = si.uniform(nb, nb, 11)
    ao, to = oracle.geqrt(a, ib)
    vs, taus = _geqrt_reflectors(ao, to, ib)
    q = _householder_product(vs, taus, nb)
    assert nrel(q @ np.triu(ao), a) < tol(nb)
    assert np.linalg.norm(q.T @ q - np.eye(nb)) < tol(nb)


@pytest.mark.parametrize("nb,ib", [(16, 4), (12, 3), (24, 24)])
def test_geqrt_compact_wy_identities(nb, ib):
    ao, to = oracle.geqrt(si.uniform(nb, nb, 12), ib)
    vs, taus = _geqrt_reflectors(ao, to, ib)
    for p in range(nb // ib):
        tp = to[:, p * ib:(p + 1) * ib]
        vp = np.stack(vs[p * ib:(p + 1) * ib], axis=1)
        assert not np.tril(tp, -1).any()
        g = vp.T @ vp
        assert np.linalg.norm(tp @ g @ tp.T - tp - tp.T) < 1e-13 * max(1, np.linalg.norm(tp) ** 2)
        assert np.linalg.norm(tp.T @ g @ tp - tp - tp.T) < 1e-13 * max(1, np.linalg.norm(tp) ** 2)
        prod = _householder_product(vs[p * ib:(p + 1) * ib], taus[p * ib:(p + 1) * ib], nb)
        assert np.linalg.norm(prod - (np.eye(nb) - vp @ tp @ vp.T)) < 1e-13


# ---------------------------------------------------------------- TSQRT
def test_tsqrt_identity_pair_closed_form():  # S:75, SURVEY §A.3
    r, v2, t = oracle.tsqrt(np.eye(6), np.eye(6), 3)
    s2 = math.sqrt(2.0)
    np.testing.assert_allclose(np.triu(r), -s2 * np.eye(6), atol=1e-15)
    np.testing.assert_allclose(v2, (s2 - 1.0) * np.eye(6), atol=1e-15)
    np.testing.assert_allclose(t, np.hstack([(1 + 1 / s2) * np.eye(3)] * 2), atol=1e-15)


def test_tsqrt_zero_bottom_is_noop():
    r0 = np.triu(si.uniform(8, 8, 4))
    r, v2, t = oracle.tsqrt(r0, np.zeros((8, 8)), 4)
    assert np.array_equal(r, r0) and not v2.any() and not t.any()


def test_tsqrt_never_touches_strict_lower_of_r():
    r0 = si.uniform(16, 16, 5)  # full: the strict lower part stands for V_kk
    r, _, _ = oracle.tsqrt(r0, si.uniform(16, 16, 6), 4)
    assert np.array_equal(np.tril(r, -1), np.tril(r0, -1))


@pytest.mark.parametrize("nb,ib", CASES)
def test_tsqrt_matches_lapack_dtpqrt(nb, ib):
    r0 = np.triu(si.uniform(nb, nb, 200 + nb))
    b0 = si.uniform(nb, nb, 300 + ib)
    r, v2, t = oracle.tsqrt(r0, b0, ib)
    rl, vl, tl, info = lapack.dtpqrt(0, ib, r0, b0)
    assert info == 0
    assert nrel(np.triu(r), np.triu(rl)) < tol(nb)
    assert nrel(v2, vl) < tol(nb)
    assert nrel(t, tl) < tol(nb)


@pytest.mark.parametrize("nb,ib", [(16, 4), (15, 5), (32, 1)])
def test_tsqrt_gram_identity(nb, ib):  # R^T R = r^T r + b^T b
    r0 = np.triu(si.uniform(nb, nb, 7))
    b0 = si.uniform(nb, nb, 8)
    r, _, _ = oracle.tsqrt(r0, b0, ib)
    r = np.triu(r)
    g = r0.T @ r0 + b0.T @ b0
    assert nrel(r.T @ r, g) < 1e-14


def test_tsqrt_r_independent_of_ib():
    r0 = np.triu(si.uniform(24, 24, 9))
    b0 = si.uniform(24, 24, 10)
    rs = [np.triu(oracle.tsqrt(r0, b0, ib)[0]) for ib in (1, 2, 4, 8, 24)]
    for x in rs[1:]:
        assert nrel(x, rs[0]) < 1e-13


def _tsqrt_q(v2, t, ib):
    nb = v2.shape[0]
    vs, taus = [], []
    for j in range(nb):
        v = np.zeros(2 * nb)
        v[j] = 1.0
        v[nb:] = v2[:, j]
        vs.append(v)
        taus.append(t[j % ib, j])
    return _householder_product(vs, taus, 2 * nb)


@pytest.mark.parametrize("nb,ib", [(12, 4), (10, 5), (16, 16)])
def test_tsqrt_reconstructs_stack(nb, ib):
    r0 = np.triu(si.uniform(nb, nb, 13))
    b0 = si.uniform(nb, nb, 14)
    r, v2, t = oracle.tsqrt(r0, b0, ib)
    q = _tsqrt_q(v2, t, ib)
    stacked = np.vstack([np.triu(r), np.zeros((nb, nb))])
    assert nrel(q @ stacked, np.vstack([r0, b0])) < tol(nb)


# ---------------------------------------------------------------- LARFB
@pytest.mark.parametrize("nb,ib", CASES)
@pytest.mark.parametrize("trans", ["T", "N"])
def test_larfb_matches_lapack_dgemqrt(nb, ib, trans):
    v, t = oracle.geqrt(si.uniform(nb, nb, 400 + nb), ib)
    c = si.uniform(nb, nb + 3, 500 + ib)
    co = oracle.larfb(v, t, c, trans)
    cl, info = lapack.dgemqrt(v, t, c, "L", trans)
    assert info == 0 and nrel(co, cl) < tol(nb)


@pytest.mark.parametrize("nb,ib", [(12, 3), (16, 16)])
def test_larfb_equals_explicit_q(nb, ib):
    v, t = oracle.geqrt(si.uniform(nb, nb, 15), ib)
    q = _householder_product(*_geqrt_reflectors(v, t, ib), nb)
    c = si.uniform(nb, 5, 16)
    assert nrel(oracle.larfb(v, t, c, "T"), q.T @ c) < tol(nb)
    assert nrel(oracle.larfb(v, t, c, "N"), q @ c) < tol(nb)


def test_larfb_identity_reflector_and_round_trip():
    v, t = oracle.geqrt(np.eye(8), 4)
    c = si.uniform(8, 8, 17)
    assert np.array_equal(oracle.larfb(v, t, c, "T"), c)
    v, t = oracle.geqrt(si.uniform(8, 8, 18), 4)
    assert nrel(oracle.larfb(v, t, oracle.larfb(v, t, c, "T"), "N"), c) < 1e-14


def test_larfb_partial_columns():
    v, t = oracle.geqrt(si.uniform(16, 16, 19), 4)
    c = si.uniform(16, 3, 20)
    cl, _ = lapack.dgemqrt(v, t, c, "L", "T")
    assert nrel(oracle.larfb(v, t, c, "T"), cl) < tol(16)


# ---------------------------------------------------------------- SSRFB
@pytest.mark.parametrize("nb,ib", CASES)
@pytest.mark.parametrize("trans", ["T", "N"])
def test_ssrfb_matches_lapack_dtpmqrt(nb, ib, trans):
    _, v2, t = oracle.tsqrt(np.triu(si.uniform(nb, nb, 600 + nb)), si.uniform(nb, nb, 700 + ib), ib)
    c1 = si.uniform(nb, nb, 800)
    c2 = si.uniform(nb, nb, 801)
    o1, o2 = oracle.ssrfb(v2, t, c1, c2, trans)
    l1, l2, info = lapack.dtpmqrt(0, v2, t, c1, c2, "L", trans)
    assert info == 0
    assert nrel(o1, l1) < tol(nb) and nrel(o2, l2) < tol(nb)


@pytest.mark.parametrize("nb,ib", [(10, 5), (12, 12), (8, 1)])
def test_ssrfb_equals_explicit_q(nb, ib):
    _, v2, t = oracle.tsqrt(np.triu(si.uniform(nb, nb, 21)), si.uniform(nb, nb, 22), ib)
    q = _tsqrt_q(v2, t, ib)
    c1, c2 = si.uniform(nb, 7, 23), si.uniform(nb, 7, 24)
    o1, o2 = oracle.ssrfb(v2, t, c1, c2, "T")
    assert nrel(np.vstack([o1, o2]), q.T @ np.vstack([c1, c2])) < tol(nb)
    o1, o2 = oracle.ssrfb(v2, t, c1, c2, "N")
    assert nrel(np.vstack([o1, o2]), q @ np.vstack([c1, c2])) < tol(nb)


def test_ssrfb_zero_v_is_identity():
    c1, c2 = si.uniform(8, 8, 25), si.uniform(8, 8, 26)
    o1, o2 = oracle.ssrfb(np.zeros((8, 8)), np.zeros((4, 8)), c1, c2, "T")
    assert np.array_equal(o1, c1) and np.array_equal(o2, c2)
