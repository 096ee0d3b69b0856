"""GPU test of the NCCL multi-GPU path (tileqr_dist_*) at world size 1.

Only one GPU is available to this run, so the NCCL communicator has one rank
(its broadcasts are root-to-self copies); the multi-rank schedule itself is
covered by tests/test_dist_gloo.py.  The distributed factorization must be
BITWISE equal to tileqr_factor on the same matrix.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tq():
    from paper_1102_5328_b200 import tileqr
    tileqr.dist_init(1, 0, tileqr.dist_unique_id(), 0)
    yield tileqr
    tileqr.dist_finalize()


def local_to_lapack(buf, n, nb, mt, nloc):
    t = buf.cpu().numpy().reshape(nloc, mt, nb, nb)  # [j][m][jl][il]
    full = np.zeros((mt * nb, nloc * nb))
    for j in range(nloc):
        for m in range(mt):
            full[m * nb:(m + 1) * nb, j * nb:(j + 1) * nb] = t[j, m].T
    return full[:n, :n]


@pytest.mark.parametrize("n,nb,ib", [(512, 128, 32), (600, 128, 16), (700, 64, 16), (300, 96, 12),
                                     (800, 256, 16), (500, 160, 32)])
def test_dist_world1_bitwise_equals_factor(tq, n, nb, ib):
    mt = -(-n // nb)
    nloc = tq.dist_local_cols(n, nb)
    assert nloc == mt
    A = torch.empty(nloc * mt * nb * nb, dtype=torch.float64, device="cuda")
    T = torch.empty(nloc * mt * ib * nb, dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    tq.dist_fill_uniform(n, nb, A, seed=5)
    ref = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(ref, n, n, seed=5)
    torch.cuda.synchronize()
    assert np.array_equal(local_to_lapack(A, n, nb, mt, nloc), ref.cpu().numpy().T)  # same input
    tq.dist_factor(n, A, nb, ib, T, info)
    Tref, info2 = tq.factor(ref, n, n, nb, ib)
    torch.cuda.synchronize()
    assert int(info.item()) == 0 and int(info2.item()) == 0
    assert np.array_equal(local_to_lapack(A, n, nb, mt, nloc), ref.cpu().numpy().T)
    tile = ib * nb  # T tile (m, k) at (m + k*MT)*IB*NB; only m >= k is defined
    for k in range(mt):
        for m in range(k, mt):
            o = (m + k * mt) * tile
            assert torch.equal(T[o:o + tile], Tref[o:o + tile]), (m, k)


def test_dist_repeated_calls_are_deterministic(tq):
    n, nb, ib = 640, 128, 32
    mt = n // nb
    A = torch.empty(mt * mt * nb * nb, dtype=torch.float64, device="cuda")
    T = torch.empty(mt * mt * ib * nb, dtype=torch.float64, device="cuda")
    outs = []
    for _ in range(2):
        tq.dist_fill_uniform(n, nb, A, seed=6)
        tq.dist_factor(n, A, nb, ib, T)
        torch.cuda.synchronize()
        outs.append((A.clone(), T.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
