"""GPU parity of the tall-skinny / communication-avoiding variant (SURVEY §8(f)
f3) against the oracle's tree tile QR (oracle_tileqr_factor_tree, pinned in
tests/test_oracle_tree.py): the batched TTQRT kernel, the whole tree
factorization on the dataflow kernel (R, V, T and T2 normwise 1e-10; north_star
residual / orthogonality with Q formed on the GPU), apply_qt_tree against
oracle.tileqr_apply_tree, and the one-domain tree = tileqr_factor bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle
import synth_inputs as si
from _tq import EPS, nrel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import tileqr
    return tileqr


def dev_tiles(mats):
    bufs = [torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float64).T)).cuda() for m in mats]
    return bufs, torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")


def host(buf):
    return buf.cpu().numpy().T


@pytest.mark.parametrize("nb,ib", [(32, 8), (64, 16), (64, 32), (96, 24), (128, 16), (128, 32), (192, 8),
                                   (256, 16)])
def test_ttqrt_batched_against_oracle(tq, nb, ib):
    r = [np.triu(si.uniform(nb, nb, 3000 + i)) + np.tril(np.full((nb, nb), 9.0), -1) for i in range(3)]
    b = [np.triu(si.uniform(nb, nb, 3100 + i)) + np.tril(np.full((nb, nb), 7.0), -1) for i in range(3)]
    rb, rp = dev_tiles(r)
    bb, bp = dev_tiles(b)
    tb, tp = dev_tiles([np.zeros((ib, nb))] * 3)
    tq.ttqrt_batched(nb, ib, rp, bp, tp)
    torch.cuda.synchronize()
    for i in range(3):
        ro, vo, to = oracle.ttqrt(r[i], b[i], ib)
        rg, vg = host(rb[i]), host(bb[i])
        assert np.array_equal(np.tril(rg, -1), np.tril(r[i], -1)), "R strict lower touched"
        assert np.array_equal(np.tril(vg, -1), np.tril(b[i], -1)), "A2 strict lower touched"
        assert nrel(np.triu(rg), np.triu(ro)) < 100 * nb * EPS
        assert nrel(np.triu(vg), np.triu(vo)) < 100 * nb * EPS
        assert nrel(host(tb[i]), to) < 100 * nb * EPS


TREE = [
    (2048, 256, 64, 16, 1),    # tall-skinny, binary tree over all 32 tile rows
    (2048, 256, 64, 32, 4),    # domains of 4
    (1500, 300, 64, 16, 2),    # ragged rows and columns
    (700, 700, 128, 32, 2),    # square, ragged
    (640, 1000, 64, 8, 3),     # wide
    (4096, 512, 128, 16, 1),   # 32 x 4 tiles
    (1200, 480, 96, 24, 5),
    (2000, 512, 256, 16, 2),   # NB > 128: 8-warp CTAs
]


@pytest.mark.parametrize("m,n,nb,ib,bs", TREE)
def test_factor_tree_against_oracle(tq, m, n, nb, ib, bs):
    a = si.uniform(m, n, 4000 + m + bs)
    A = tq.to_colmajor(a)
    T, info = tq.factor_tree(A, m, n, nb, ib, bs)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    fo, to, _ = oracle.tileqr_factor_tree(a, nb, ib, bs)
    f = tq.from_colmajor(A)
    assert nrel(oracle.sign_normalised_r(f), oracle.sign_normalised_r(fo)) < 1e-10
    assert nrel(f, fo) < 1e-10
    half = to.size // 2
    tg = T.cpu().numpy()
    assert nrel(tg[:half], to[:half]) < 1e-10 and nrel(tg[half:], to[half:]) < 1e-10
    # north_star tolerances with Q formed on the GPU
    Q = tq.to_colmajor(np.eye(m))
    tq.apply_qt_tree("N", A, m, n, T, nb, ib, bs, Q, m)
    torch.cuda.synchronize()
    q = tq.from_colmajor(Q)
    k = min(m, n)
    r = np.triu(f[:k, :])
    assert np.linalg.norm(a - q[:, :k] @ r) / (np.linalg.norm(a) * max(m, n) * EPS) < 10
    assert np.linalg.norm(q.T @ q - np.eye(m)) / (m * EPS) < 10


@pytest.mark.parametrize("trans", ["T", "N"])
@pytest.mark.parametrize("m,n,nrhs,nb,ib,bs", [(1024, 200, 37, 64, 16, 1), (900, 400, 130, 128, 32, 3)])
def test_apply_qt_tree_against_oracle(tq, trans, m, n, nrhs, nb, ib, bs):
    a = si.uniform(m, n, 4500 + m)
    A = tq.to_colmajor(a)
    T, _ = tq.factor_tree(A, m, n, nb, ib, bs)
    b = si.uniform(m, nrhs, 4600 + nrhs)
    B = tq.to_colmajor(b)
    tq.apply_qt_tree(trans, A, m, n, T, nb, ib, bs, B, nrhs)
    torch.cuda.synchronize()
    bo = oracle.tileqr_apply_tree(trans, tq.from_colmajor(A), T.cpu().numpy(), nb, ib, bs, b)
    assert nrel(tq.from_colmajor(B), bo) < 100 * max(m, n) * EPS


@pytest.mark.parametrize("m,n,nb,ib", [(1000, 600, 128, 16), (777, 777, 64, 32)])
def test_one_domain_tree_is_the_flat_factorization(tq, m, n, nb, ib):
    a = si.uniform(m, n, 4700 + m)
    A1, A2 = tq.to_colmajor(a), tq.to_colmajor(a)
    T1, _ = tq.factor(A1, m, n, nb, ib)
    T2, _ = tq.factor_tree(A2, m, n, nb, ib, 1 << 20)
    torch.cuda.synchronize()
    assert torch.equal(A1, A2)
    assert torch.equal(T1, T2[:T1.numel()]) and not torch.any(T2[T1.numel():] != 0)


def test_tree_deterministic(tq):
    m, n, nb, ib, bs = 3000, 384, 128, 16, 1
    a = si.uniform(m, n, 4800)
    outs = []
    for _ in range(3):
        A = tq.to_colmajor(a)
        T, _ = tq.factor_tree(A, m, n, nb, ib, bs)
        torch.cuda.synchronize()
        outs.append((A, T))
    for A, T in outs[1:]:
        assert torch.equal(A, outs[0][0]) and torch.equal(T, outs[0][1])


def test_tune_tree_picks_a_measured_bs(tq, tmp_path):
    import json
    m, n, nb, ib = 8192, 256, 128, 16
    path = tmp_path / "tt.json"
    bs, ms = tq.tune_tree(m, n, nb, ib, str(path))
    rep = json.load(open(path))
    runs = {r["bs"]: r["median_ms"] for r in rep["runs"]}
    assert set(runs) == {1, 2, 4, 8, 16, 32, 64}            # powers of two below MT = 64, and MT
    assert bs == min(runs, key=runs.get) and abs(ms - runs[bs]) < 1e-5 and rep["best_bs"] == bs
