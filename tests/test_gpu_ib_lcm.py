"""IB that the DMMA paths take only through another inner blocking IBe
(R23): lcm(IB, 8) for IB not a multiple of 8, a divisor <= 32 for
IB > 64.

tileqr_factor runs such an IB at IBe = lcm(IB, 8) (when IBe <= 64 divides NB)
and returns T at IB as the diagonal IB-blocks of T at IBe (IB > 64: runs at
IBe | IB and assembles T at IB from the factored tiles); the batched LARFB /
SSRFB entry points ('T', all NB columns, IB < 8 or > 64) form T at IBe
(assembled from V and tau, or the caller's T's diagonal blocks) and run the
packed IBe update.  Both are
compared with the oracle run at the caller's IB (V, R, T and the updated
tiles, normwise; the IBe blocking is another rounding order of the same
reflectors).
"""
import numpy as np
import pytest
import torch

import oracle
import synth_inputs as si
from _tq import EPS, nrel

pytestmark = pytest.mark.gpu

BATCH = 4
LCM_CASES = [(64, 2, 8), (128, 4, 8), (96, 12, 24), (192, 6, 24), (160, 10, 40), (160, 20, 40),
             (224, 28, 56), (224, 14, 56), (256, 1, 8),
             # IB > 64: run at the largest of 32, 24, 16, 8 dividing IB, T at IB assembled afterwards
             (128, 128, 32), (256, 128, 32), (96, 96, 32), (160, 80, 16), (224, 224, 32), (256, 256, 32)]


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import tileqr
    return tileqr


def dev_tiles(mats):
    bufs = [torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float64).T)).cuda() for m in mats]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    return bufs, ptrs


def host(buf):
    return buf.cpu().numpy().T


@pytest.mark.parametrize("nb,ib,ibe", LCM_CASES)
def test_factor_at_lcm_blocking_matches_oracle(tq, nb, ib, ibe):
    m = n = 2 * nb + nb // 2 + 3  # 3 x 3 tiles, ragged tail
    a = si.uniform(m, n, 900 + nb + ib)
    A = tq.to_colmajor(a)
    T, info = tq.factor(A, m, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    f = tq.from_colmajor(A)
    fo, to, _ = oracle.tileqr_factor(a, nb, ib)
    assert nrel(oracle.sign_normalised_r(f), oracle.sign_normalised_r(fo)) < 1e-10
    assert nrel(f, fo) < 1e-10
    t = T.cpu().numpy()
    assert t.shape == to.shape
    assert nrel(t, to) < 1e-10
    # T at IB: every IB x IB block upper triangular (strict lower part exactly 0)
    tiles = t.reshape(-1, nb, ib)  # per tile: column j of T(IB) = row j of this view
    for blk in tiles:
        for j in range(nb):
            assert np.all(blk[j, j % ib + 1:] == 0.0)


@pytest.mark.parametrize("nb,ib,ibe", [c for c in LCM_CASES if c[1] < 8 or c[1] > 64])
@pytest.mark.parametrize("larfb", [False, True])
def test_batched_update_at_lcm_blocking_matches_oracle(tq, nb, ib, ibe, larfb):
    vs, ts, c1, c2 = [], [], [], []
    for i in range(BATCH):
        x = si.uniform(nb, nb, 50 + nb + ib, offset=4 * i * nb * nb)
        y = si.uniform(nb, nb, 51 + nb + ib, offset=(4 * i + 1) * nb * nb)
        if larfb:
            f, t = oracle.geqrt(x, ib)
            vs.append(f)
        else:
            _, v2, t = oracle.tsqrt(np.triu(x), y, ib)
            vs.append(v2)
        ts.append(t)
        c1.append(si.uniform(nb, nb, 52 + nb + ib, offset=(4 * i + 2) * nb * nb))
        c2.append(si.uniform(nb, nb, 53 + nb + ib, offset=(4 * i + 3) * nb * nb))
    vb, vp = dev_tiles(vs)
    tb, tp = dev_tiles(ts)
    c1b, c1p = dev_tiles(c1)
    c2b, c2p = dev_tiles(c2)
    if larfb:
        tq.larfb_batched("T", nb, ib, vp, tp, c2p, nb)
    else:
        tq.ssrfb_batched("T", nb, ib, vp, tp, c1p, c2p, nb)
    torch.cuda.synchronize()
    tol = 100 * nb * EPS
    for i in range(BATCH):
        if larfb:
            o2 = oracle.larfb(vs[i], ts[i], c2[i], "T")
            assert nrel(host(c2b[i]), o2) < tol, i
        else:
            o1, o2 = oracle.ssrfb(vs[i], ts[i], c1[i], c2[i], "T")
            assert nrel(host(c1b[i]), o1) < tol, i
            assert nrel(host(c2b[i]), o2) < tol, i
    # the caller's V and T are inputs only
    for i in range(BATCH):
        assert np.array_equal(host(tb[i]), ts[i])
