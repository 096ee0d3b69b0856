"""Round-2 parity cases of the CUDA path against the oracle (through the C ABI).

* configs[3] (10000^2) in FULL at the bench's own (NB, IB) -- read from the
  decision table with the oracle's nearest-point rule, not hard-coded --
  against the full oracle factorization (R, V, T normwise 1e-10; sign-
  normalised R 1e-10), plus the north_star Frobenius residual and
  orthogonality with Q formed on the GPU (an fp64 torch matmul is the
  checker only).
* every instantiation of the register-resident panel kernel (NB % 32 == 0,
  32 <= NB <= 256, IB in {8, 16, 24, 32} dividing NB: 26 pairs), batched
  GEQRT and TSQRT against oracle.geqrt / oracle.tsqrt, and the whole
  factorization (dataflow kernel, ragged) at every pair against the oracle.
* tileqr_apply_qt ('T' and 'N') against oracle.tileqr_apply element-wise on
  the same factor: square, ragged, tall, wide, NRHS not a multiple of NB.
* degenerate inputs: exactly-zero columns, an already upper-triangular
  matrix (every reflector tau = 0: R == A bit for bit, V = 0, T = 0), -0.0
  pivots (sgn(-0) = +1, R1).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth_inputs as si
from _tq import EPS, nrel
from oracle import tuner

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TABLE = os.path.join(ROOT, "paper_1102_5328_b200", "tuned_table.json")

PANEL_FAST = [(nb, ib) for nb in range(32, 257, 32) for ib in (8, 16, 24, 32) if nb % ib == 0]
assert len(PANEL_FAST) == 26


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import tileqr
    return tileqr


def host(buf):
    return buf.cpu().numpy().T


def dev_tiles(mats):
    bufs = [torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float64).T)).cuda() for m in mats]
    return bufs, torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")


def tuned_pair(n, ngpus=1):
    """The bench's (NB, IB): nearest point of the decision table (oracle rule)."""
    tab = json.load(open(TABLE))["entries"]
    table = {(e["n"], e["ngpus"]): (e["nb"], e["ib"]) for e in tab}
    return tuner.lookup(table, n, ngpus)


# ---------------------------------------------------------------------------
# configs[3] in full
# ---------------------------------------------------------------------------
@pytest.mark.slow
def test_config3_full_against_oracle(tq):
    n = 10000
    nb, ib = tuned_pair(n)
    a = si.uniform(n, n, 4)
    A = tq.to_colmajor(a)
    T, info = tq.factor(A, n, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)            # full oracle, all host cores
    f = A.cpu().numpy().T                                   # GPU factor (column-major storage)
    assert nrel(oracle.sign_normalised_r(f), oracle.sign_normalised_r(fo)) < 1e-10
    assert nrel(np.triu(f), np.triu(fo)) < 1e-10            # R
    assert nrel(np.tril(f, -1), np.tril(fo, -1)) < 1e-10    # V (V_kk strictly lower, V2 full tiles)
    assert nrel(T.cpu().numpy(), to) < 1e-10                # T
    del fo, to, f
    # north_star Frobenius tolerances, Q formed on the GPU (apply_q of I)
    Q = torch.eye(n, dtype=torch.float64, device="cuda")     # symmetric: its storage is column-major I
    tq.apply_qt("N", A, n, n, T, nb, ib, Q, n)
    torch.cuda.synchronize()
    Qm = Q.t()                                              # the matrix Q
    R = torch.triu(A.t())
    Ad = torch.from_numpy(a).cuda()
    res = float(torch.linalg.norm(Ad - Qm @ R) / (torch.linalg.norm(Ad) * n * EPS))
    del R, Ad
    Iq = Qm.t() @ Qm
    Iq.diagonal().sub_(1.0)
    orth = float(torch.linalg.norm(Iq) / (n * EPS))
    assert res < 10, res
    assert orth < 10, orth


# ---------------------------------------------------------------------------
# every panel_fast instantiation
# ---------------------------------------------------------------------------
def seeds(nb, ib, k, batch=3):
    return [si.uniform(nb, nb, 5000 + 17 * nb + ib, offset=(k * batch + i) * nb * nb) for i in range(batch)]


@pytest.mark.parametrize("nb,ib", PANEL_FAST)
def test_panel_fast_geqrt_tsqrt(tq, nb, ib):
    tol = 100 * nb * EPS
    a = seeds(nb, ib, 0)
    ab, ap = dev_tiles(a)
    tb, tp = dev_tiles([np.zeros((ib, nb))] * len(a))
    tq.geqrt_batched(nb, ib, ap, tp)
    r = [np.triu(x) + np.tril(np.full((nb, nb), 5.0), -1) for x in seeds(nb, ib, 1)]
    b = seeds(nb, ib, 2)
    rb, rp = dev_tiles(r)
    bb, bp = dev_tiles(b)
    t2b, t2p = dev_tiles([np.zeros((ib, nb))] * len(r))
    tq.tsqrt_batched(nb, ib, rp, bp, t2p)
    torch.cuda.synchronize()
    for i in range(len(a)):
        ao, to = oracle.geqrt(a[i], ib)
        assert nrel(host(ab[i]), ao) < tol and nrel(host(tb[i]), to) < tol, ("geqrt", i)
        ro, vo, t2o = oracle.tsqrt(r[i], b[i], ib)
        rg = host(rb[i])
        assert np.array_equal(np.tril(rg, -1), np.tril(r[i], -1)), "TSQRT wrote the strict lower part of R"
        assert nrel(np.triu(rg), np.triu(ro)) < tol, ("tsqrt R", i)
        assert nrel(host(bb[i]), vo) < tol and nrel(host(t2b[i]), t2o) < tol, ("tsqrt V/T", i)


@pytest.mark.parametrize("nb,ib", PANEL_FAST)
def test_factor_every_panel_fast_pair(tq, nb, ib):
    """The whole factorization (persistent dataflow kernel at these pairs) on a
    ragged 3 x 3-tile matrix against the oracle."""
    m, n = 3 * nb - 3, 3 * nb - 7
    a = si.uniform(m, n, 900 + nb + ib)
    A = tq.to_colmajor(a)
    T, info = tq.factor(A, m, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    assert tq.factor_schedule(nb, ib) == "dag"
    f = tq.from_colmajor(A)
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    assert nrel(oracle.sign_normalised_r(f), oracle.sign_normalised_r(fo)) < 1e-10
    assert nrel(f, fo) < 1e-10 and nrel(T.cpu().numpy(), to) < 1e-10


def test_factor_tuned_2048_pair(tq):
    """The decision table's own pick at N=2048 (configs[2]) against the oracle."""
    nb, ib = tuned_pair(2048)
    a = si.uniform(2048, 2048, 3)
    A = tq.to_colmajor(a)
    T, _ = tq.factor(A, 2048, 2048, nb, ib)
    torch.cuda.synchronize()
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    f = tq.from_colmajor(A)
    assert nrel(f, fo) < 1e-10 and nrel(T.cpu().numpy(), to) < 1e-10


@pytest.mark.parametrize("nb,ib", [(64, 32), (64, 16), (128, 16)])
def test_factor_1024_against_oracle(tq, nb, ib):
    a = si.uniform(1024, 1024, 77)
    A = tq.to_colmajor(a)
    T, _ = tq.factor(A, 1024, 1024, nb, ib)
    torch.cuda.synchronize()
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    assert nrel(tq.from_colmajor(A), fo) < 1e-10 and nrel(T.cpu().numpy(), to) < 1e-10


# The dataflow kernel's resident-CTA rules (session 4):
# widest step (MT-1)(NT-1) <= 1200 tile updates: one CTA per SM; <= 4000: two
# per SM with the second retiring in the tail (kModePlainRetire); above: the
# plain kernel.  One oracle comparison per regime and tile order, ragged sizes.
@pytest.mark.parametrize("n,nb,ib", [
    (2000, 64, 16),    # 31^2 = 961 tiles: one CTA per SM
    (2590, 64, 16),    # 40^2 = 1600: tail retirement
    (2590, 64, 32),
    (4650, 128, 16),   # 36^2 = 1296: tail retirement at NB = 128
    (4200, 64, 16),    # 65^2 = 4225: plain kernel
])
def test_factor_resident_cta_regimes_against_oracle(tq, n, nb, ib):
    a = si.uniform(n, n, 1000 + n)
    A = tq.to_colmajor(a)
    T, info = tq.factor(A, n, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    assert nrel(tq.from_colmajor(A), fo) < 1e-10 and nrel(T.cpu().numpy(), to) < 1e-10


# ---------------------------------------------------------------------------
# apply_qt against the oracle
# ---------------------------------------------------------------------------
APPLY = [
    (512, 512, 77, 128, 16),    # square, NRHS not a multiple of NB
    (450, 450, 130, 128, 32),   # ragged
    (700, 300, 45, 64, 16),     # tall
    (300, 700, 200, 96, 24),    # wide (K > M)
    (333, 333, 1, 64, 8),       # single right-hand side
    (260, 260, 70, 48, 6),      # level/staged path (NB % 32 != 0)
]


@pytest.mark.parametrize("m,k,nrhs,nb,ib", APPLY)
@pytest.mark.parametrize("trans", ["T", "N"])
def test_apply_qt_against_oracle(tq, m, k, nrhs, nb, ib, trans):
    a = si.uniform(m, k, 300 + m + nb)
    A = tq.to_colmajor(a)
    T, _ = tq.factor(A, m, k, nb, ib)
    b = si.uniform(m, nrhs, 400 + nrhs)
    B = tq.to_colmajor(b)
    tq.apply_qt(trans, A, m, k, T, nb, ib, B, nrhs)
    torch.cuda.synchronize()
    f, t = tq.from_colmajor(A), T.cpu().numpy()
    bo = oracle.tileqr_apply(trans, f, t, nb, ib, b)        # the same factor, applied by the oracle
    assert nrel(tq.from_colmajor(B), bo) < 100 * max(m, k) * EPS


# ---------------------------------------------------------------------------
# degenerate inputs
# ---------------------------------------------------------------------------
def test_zero_columns(tq):
    m, n, nb, ib = 400, 390, 128, 16
    a = si.uniform(m, n, 601)
    a[:, 5] = 0.0          # inside the first tile's first inner panel
    a[:, 130] = 0.0        # second tile column
    a[:, 256:384] = 0.0    # a whole tile column
    A = tq.to_colmajor(a)
    T, info = tq.factor(A, m, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    f = tq.from_colmajor(A)
    assert nrel(f, fo) < 1e-10 and nrel(T.cpu().numpy(), to) < 1e-10
    assert f[5, 5] == 0.0 and np.all(f[6:, 5] == 0.0)       # tau = 0: no reflection, v = 0


@pytest.mark.parametrize("nb,ib", [(64, 16), (128, 32), (96, 8)])
def test_upper_triangular_input_is_fixed_point(tq, nb, ib):
    """Every reflector of an upper-triangular A has x2 = 0, so tau = 0 and the
    factorization returns A itself: R == A exactly, V = 0, T = 0."""
    m = n = 3 * nb + 17
    a = np.triu(si.uniform(m, n, 602))
    A = tq.to_colmajor(a)
    T, _ = tq.factor(A, m, n, nb, ib)
    torch.cuda.synchronize()
    f = tq.from_colmajor(A)
    assert np.array_equal(f, a)
    assert not np.any(T.cpu().numpy())


def test_negative_zero_pivots(tq):
    """alpha = -0.0 with a nonzero tail: sgn(-0) = +1, beta = -||x2|| < 0;
    alpha = -0.0 with a zero tail: tau = 0 and beta = alpha (the sign kept)."""
    m, n, nb, ib = 256, 256, 64, 16
    a = si.uniform(m, n, 603)
    a[0, 0] = -0.0
    a[64, 64] = -0.0
    A = tq.to_colmajor(a)
    T, _ = tq.factor(A, m, n, nb, ib)
    torch.cuda.synchronize()
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    f = tq.from_colmajor(A)
    assert nrel(f, fo) < 1e-10 and nrel(T.cpu().numpy(), to) < 1e-10
    # one tile: R(0,0) is GEQRT's beta = -sgn(-0) ||x|| < 0 (later TSQRTs may flip it)
    c = si.uniform(64, 64, 605)
    c[0, 0] = -0.0
    C = tq.to_colmajor(c)
    tq.factor(C, 64, 64, 64, 16)
    torch.cuda.synchronize()
    fc, fco = tq.from_colmajor(C), oracle.tileqr_factor(c, 64, 16)[0]
    assert fc[0, 0] < 0 and fco[0, 0] < 0 and abs(fc[0, 0] + np.linalg.norm(c[:, 0])) < 1e-14 * abs(fc[0, 0])
    # zero tail under a -0.0 pivot
    b = np.triu(si.uniform(128, 128, 604))
    b[0, 0] = -0.0
    B = tq.to_colmajor(b)
    TB, _ = tq.factor(B, 128, 128, 64, 16)
    torch.cuda.synchronize()
    fb = tq.from_colmajor(B)
    assert fb[0, 0] == 0.0 and np.signbit(fb[0, 0])
    assert not np.any(TB.cpu().numpy())


@pytest.mark.parametrize("scale_exp", [-300, -100, 100, 300])
def test_scaled_inputs_within_the_supported_range(tq, scale_exp):
    """No safmin / safmax rescaling (R1, include/tileqr.h): inputs
    with |a| in [2^-450, 2^450] keep every sum of squares in the normal range.
    Scaling A by a power of two scales R exactly and leaves V, T unchanged."""
    m, n, nb, ib = 600, 500, 128, 16
    a = si.uniform(m, n, 650)
    s = 2.0 ** scale_exp
    A1, A2 = tq.to_colmajor(a), tq.to_colmajor(a * s)
    T1, _ = tq.factor(A1, m, n, nb, ib)
    T2, info = tq.factor(A2, m, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    f1, f2 = tq.from_colmajor(A1), tq.from_colmajor(A2)
    assert nrel(np.triu(f2) / s, np.triu(f1)) < 1e-13
    assert nrel(np.tril(f2, -1), np.tril(f1, -1)) < 1e-13
    assert nrel(T2.cpu().numpy(), T1.cpu().numpy()) < 1e-13


def test_concurrent_same_shape_calls_on_two_streams(tq):
    """Two factorizations of the same shape (one cached workspace) issued on
    two streams without synchronisation: the workspace's last-use event
    orders them, and both results are exact."""
    m = n = 1024
    nb, ib = 128, 16
    a, b = si.uniform(m, n, 660), si.uniform(m, n, 661)
    ref_a, ref_b = tq.to_colmajor(a), tq.to_colmajor(b)
    Ta, _ = tq.factor(ref_a, m, n, nb, ib)
    Tb, _ = tq.factor(ref_b, m, n, nb, ib)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        A, B = tq.to_colmajor(a), tq.to_colmajor(b)
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            T1, _ = tq.factor(A, m, n, nb, ib, stream=s1)
        with torch.cuda.stream(s2):
            T2, _ = tq.factor(B, m, n, nb, ib, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(A, ref_a) and torch.equal(T1, Ta)
        assert torch.equal(B, ref_b) and torch.equal(T2, Tb)


@pytest.mark.slow
def test_config4_size_on_one_gpu(tq):
    """BASELINE.json configs[4]'s matrix (40000^2, 12.8 GB) on ONE B200 -- the
    maximum size: the first block row of R and panel 0 (V, T) against the
    oracle (kmax=1, ~0.8 TFLOP on the host cores), residual and orthogonality
    on random vectors (properties that hold at any size)."""
    n = 40000
    nb, ib, _ = tq.lookup(n, n, 1)
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(A, n, n, seed=5)
    A0 = A.clone()
    T, info = tq.factor(A, n, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    # the oracle's first panel on the same matrix (column-major storage -> numpy matrix)
    a = A0.cpu().numpy().T
    fo, to, _ = oracle.tileqr_factor(a, nb, ib, kmax=1)
    f_row = A[:, :nb].cpu().numpy().T
    assert nrel(f_row, fo[:nb, :]) < 1e-10
    f_col = A[:nb, :].cpu().numpy().T
    assert nrel(f_col, fo[:, :nb]) < 1e-10
    mt = -(-n // nb)
    assert nrel(T[: mt * ib * nb].cpu().numpy(), to[: mt * ib * nb]) < 1e-10
    del a, fo, to, f_row, f_col
    x = torch.from_numpy(si.uniform(n, 4, 42)).cuda()
    Rx = torch.triu(A.t()) @ x
    QRx = Rx.t().contiguous()
    tq.apply_qt("N", A, n, n, T, nb, ib, QRx, 4)
    Ax = A0.t() @ x
    torch.cuda.synchronize()
    res = torch.linalg.norm(Ax - QRx.t()) / (torch.linalg.norm(A0) * torch.linalg.norm(x) * n * EPS)
    assert float(res) < 10
    y = tq.to_colmajor(si.uniform(n, 4, 43))
    y0 = y.clone()
    tq.apply_qt("N", A, n, n, T, nb, ib, y, 4)
    tq.apply_qt("T", A, n, n, T, nb, ib, y, 4)
    torch.cuda.synchronize()
    assert float(torch.linalg.norm(y - y0) / (torch.linalg.norm(y0) * n * EPS)) < 10
