"""Pins of the oracle's whole tile QR factorization and Q application.

Expected values come from: a textbook unblocked Householder QR written here,
the same flat-tree tile algorithm composed from LAPACK kernels (scipy),
numpy.linalg.qr, 50-digit Gram-Schmidt (decimal) on tiny matrices, the
identity R^T R = A^T A, residual/orthogonality bounds of BASELINE.json
north_star, and bitwise invariance across thread counts.
"""
import decimal

import numpy as np
import pytest
import scipy.linalg.lapack as lapack

import oracle
import synth_inputs as si
from _tq import EPS, nrel


def sign_norm(r):
    s = np.where(np.diag(r) < 0, -1.0, 1.0)
    return s[:, None] * r


def textbook_householder_r(a):
    """Unblocked Householder QR (Golub & Van Loan Alg. 5.2.1 with the LAPACK
    sign choice beta = -sign(alpha)*||x||), written independently here."""
    a = np.array(a, dtype=np.float64)
    m, n = a.shape
    for j in range(min(m, n)):
        x = a[j:, j].copy()
        normx = np.linalg.norm(x)
        if np.linalg.norm(x[1:]) == 0.0:
            continue
        beta = -normx if x[0] >= 0 else normx
        v = x.copy()
        v[0] -= beta
        v /= v[0]
        tau = (beta - x[0]) / beta
        a[j:, j:] -= tau * np.outer(v, v @ a[j:, j:])
    return np.triu(a[:min(m, n), :])


def scipy_tile_qr(a, nb, ib):
    """Flat-tree tile QR composed from LAPACK kernels (dgeqrt, dgemqrt,
    dtpqrt l=0, dtpmqrt l=0) -- the same algorithm with library kernels."""
    a = np.array(a, dtype=np.float64, order="F")
    nt = a.shape[0] // nb
    ts = {}

    def tile(i, j):
        return a[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb]

    for k in range(nt):
        akk, tkk, _ = lapack.dgeqrt(ib, tile(k, k))
        tile(k, k)[:] = akk
        ts[(k, k)] = tkk
        for n in range(k + 1, nt):
            c, _ = lapack.dgemqrt(akk, tkk, tile(k, n), "L", "T")
            tile(k, n)[:] = c
        for m in range(k + 1, nt):
            r, b, t, _ = lapack.dtpqrt(0, ib, np.triu(tile(k, k)), tile(m, k))
            tile(k, k)[:] = np.triu(r) + np.tril(tile(k, k), -1)
            tile(m, k)[:] = b
            ts[(m, k)] = t
            for n in range(k + 1, nt):
                c1, c2, _ = lapack.dtpmqrt(0, b, t, tile(k, n), tile(m, n), "L", "T")
                tile(k, n)[:] = c1
                tile(m, n)[:] = c2
    return a, ts


@pytest.mark.parametrize("n,nb,ib", [(256, 64, 16), (256, 64, 64), (192, 32, 1), (120, 24, 3), (64, 64, 8)])
def test_factor_matches_scipy_composed_tile_qr(n, nb, ib):
    a = si.uniform(n, n, 1)
    f, t, info = oracle.tileqr_factor(a, nb, ib)
    g, ts = scipy_tile_qr(a, nb, ib)
    assert info == 0
    assert nrel(f, g) < 1e-13  # R and every V tile
    for (m, k), tl in ts.items():
        assert nrel(oracle.t_tile(t, n, n, nb, ib, m, k), tl) < 1e-12


@pytest.mark.parametrize("m,n,nb,ib", [(256, 256, 64, 16), (250, 250, 64, 16), (300, 190, 64, 8),
                                       (150, 250, 64, 16), (97, 97, 32, 4), (64, 200, 32, 32)])
def test_factor_r_matches_numpy_qr_sign_normalised(m, n, nb, ib):
    a = si.uniform(m, n, 2)
    f, _, info = oracle.tileqr_factor(a, nb, ib)
    assert info == 0
    rn = np.linalg.qr(a, mode="r")
    assert nrel(oracle.sign_normalised_r(f), sign_norm(rn)) < 1e-13


def test_factor_nb_equals_n_ib1_is_textbook_householder():
    a = si.uniform(40, 40, 3)
    f, _, _ = oracle.tileqr_factor(a, 40, 1)
    assert nrel(np.triu(f), textbook_householder_r(a)) < 1e-14  # same signs, no normalisation


def test_factor_tiny_against_50_digit_gram_schmidt():
    decimal.getcontext().prec = 50
    D = decimal.Decimal
    for n in (2, 5, 8):
        a = si.uniform(n, n, 40 + n)
        cols = [[D(float(a[i, j])) for i in range(n)] for j in range(n)]
        q, r = [], [[D(0)] * n for _ in range(n)]
        for j in range(n):
            v = cols[j][:]
            for i in range(j):
                r[i][j] = sum(q[i][k] * cols[j][k] for k in range(n))
                v = [v[k] - r[i][j] * q[i][k] for k in range(n)]
            r[j][j] = sum(x * x for x in v).sqrt()
            q.append([x / r[j][j] for x in v])
        rgs = np.array([[float(x) for x in row] for row in r])
        f, _, _ = oracle.tileqr_factor(a, 2 if n % 2 == 0 else n, 1)
        assert nrel(oracle.sign_normalised_r(f), rgs) < 1e-14


def test_factor_2x2_closed_form():
    f, t, _ = oracle.tileqr_factor(np.array([[3.0, 1.0], [4.0, 2.0]]), 2, 1)
    np.testing.assert_allclose(np.triu(f), [[-5.0, -2.2], [0.0, 0.4]], atol=1e-15)
    f, t, _ = oracle.tileqr_factor(np.array([[3.0, 1.0], [4.0, 2.0]]), 1, 1)
    np.testing.assert_allclose(np.triu(f), [[-5.0, -2.2], [0.0, 0.4]], atol=1e-15)


@pytest.mark.parametrize("m,n,nb,ib", [(256, 256, 64, 16), (200, 130, 48, 12), (130, 200, 48, 6)])
def test_factor_gram_identity_and_tolerances(m, n, nb, ib):
    a = si.uniform(m, n, 5)
    f, t, _ = oracle.tileqr_factor(a, nb, ib)
    k = min(m, n)
    r = np.triu(f[:k, :])
    assert np.linalg.norm(r.T @ r - a.T @ a) / np.linalg.norm(a) ** 2 < 1e-15
    q = oracle.tileqr_apply("N", f, t, nb, ib, np.eye(m))
    qk = q[:, :k]
    # BASELINE.json north_star tolerances
    assert np.linalg.norm(a - qk @ r) / (np.linalg.norm(a) * max(m, n) * EPS) < 10
    assert np.linalg.norm(q.T @ q - np.eye(m)) / (m * EPS) < 10


def test_apply_round_trip_and_qt_a_is_r():
    m, n, nb, ib = 200, 160, 32, 8
    a = si.uniform(m, n, 6)
    f, t, _ = oracle.tileqr_factor(a, nb, ib)
    b = si.uniform(m, 9, 7)
    qb = oracle.tileqr_apply("N", f, t, nb, ib, b)
    assert nrel(oracle.tileqr_apply("T", f, t, nb, ib, qb), b) < 1e-14
    qta = oracle.tileqr_apply("T", f, t, nb, ib, a)
    assert nrel(qta[:n, :], np.triu(f[:n, :])) < 1e-14
    assert np.linalg.norm(qta[n:, :]) < 1e-13


def test_factor_bitwise_invariant_across_threads():
    a = si.uniform(320, 320, 8)
    outs = [oracle.tileqr_factor(a, 64, 16, nthreads=th) for th in (1, 2, 4, 8)]
    for f, t, _ in outs[1:]:
        assert np.array_equal(f, outs[0][0]) and np.array_equal(t, outs[0][1])


def test_factor_partial_kmax_rows_are_final():
    a = si.uniform(256, 256, 9)
    f, t, _ = oracle.tileqr_factor(a, 64, 16)
    fp, tp, _ = oracle.tileqr_factor(a, 64, 16, kmax=1)
    assert np.array_equal(fp[:64, :], f[:64, :])  # first block row of R
    assert np.array_equal(fp[:, :64], f[:, :64])  # panel 0: R_00, V_00, V2_m0
    assert np.array_equal(tp[: 4 * 16 * 64], t[: 4 * 16 * 64])  # T tiles (m, 0)


def test_padding_identity_and_zero_rows():
    # 250 -> 256 at NB=64: padded columns are e_j, so tau = 0 for them and the
    # thin factors equal those of the unpadded problem.
    a = si.uniform(250, 250, 10)
    f, t, _ = oracle.tileqr_factor(a, 64, 16)
    tkk = oracle.t_tile(t, 250, 250, 64, 16, 3, 3)
    assert not tkk[:, 250 - 192:].any()  # reflectors of padded columns: T columns 0


def test_nonfinite_input_sets_info():
    a = si.uniform(64, 64, 11)
    a[5, 7] = np.nan
    f, t, info = oracle.tileqr_factor(a, 32, 8)
    assert info == 1 and np.array_equal(np.isnan(f), np.isnan(a))
    a[5, 7] = np.inf
    assert oracle.tileqr_factor(a, 32, 8)[2] == 1


def test_quick_return_empty():
    f, t, info = oracle.tileqr_factor(np.zeros((0, 5)), 4, 2)
    assert info == 0 and f.shape == (0, 5)
