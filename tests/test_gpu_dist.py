"""GPU tests of the multi-GPU path (tileqr_dist_*).

Only one GPU is available to this run:
  * tileqr_dist_factor at world size 1 (NCCL communicator of one rank), on
    the dataflow schedule (default) and the level-synchronous NCCL baseline;
  * tileqr_dist_emulate: the multi-rank DATAFLOW factorization with 2-4
    emulated ranks on this GPU -- the same per-rank work lists and kernel
    code as a multi-GPU run, every rank with its own tile / T / slot /
    counter buffers and the COPY items pushing packed reflector tiles into
    the other ranks' buffers.
The distributed factorization must be BITWISE equal to tileqr_factor on the
same matrix.  The multi-rank host plans are also executed on
the CPU with gloo (tests/test_dist_gloo.py, tests/test_dist_dataflow_gloo.py).
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


def padded(a, nb):
    """The padded tile matrix of DESIGN.md R5 (rows >= M zero, padded column j
    is e_j when M <= j < MT*NB)."""
    m, n = a.shape
    mt, nt = -(-m // nb), -(-n // nb)
    full = np.zeros((mt * nb, nt * nb))
    full[:m, :n] = a
    for j in range(n, nt * nb):
        if m <= j < mt * nb:
            full[j, j] = 1.0
    return full


def to_local(full, nb, world, rank):
    mt, nt = full.shape[0] // nb, full.shape[1] // nb
    cols = list(range(rank, nt, world))
    buf = np.zeros((len(cols), mt, nb, nb))
    for j, c in enumerate(cols):
        for m in range(mt):
            buf[j, m] = full[m * nb:(m + 1) * nb, c * nb:(c + 1) * nb].T
    return torch.from_numpy(buf.reshape(-1)).cuda() if cols else None


def from_locals(bufs, nb, world, mt, nt):
    full = np.zeros((mt * nb, nt * nb))
    for r in range(world):
        if bufs[r] is None:
            continue
        t = bufs[r].cpu().numpy().reshape(-1, mt, nb, nb)
        for j, c in enumerate(range(r, nt, world)):
            for m in range(mt):
                full[m * nb:(m + 1) * nb, c * nb:(c + 1) * nb] = t[j, m].T
    return full


@pytest.mark.parametrize("sched", ["dataflow", "levels"])
@pytest.mark.parametrize("n,nb,ib", [(512, 128, 32), (600, 128, 16), (700, 64, 16), (300, 96, 12),
                                     (800, 256, 16), (500, 160, 32), (600, 128, 128), (500, 64, 2)])
def test_dist_world1_bitwise_equals_factor(tq, monkeypatch, sched, n, nb, ib):
    if sched == "levels":
        monkeypatch.setenv("TILEQR_DIST_SCHED", "levels")
    mt = -(-n // nb)
    nloc = tq.dist_local_cols(n, nb)
    assert nloc == mt
    A = torch.empty(nloc * mt * nb * nb, dtype=torch.float64, device="cuda")
    T = torch.empty(nloc * mt * ib * nb, dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    tq.dist_fill_uniform(n, n, nb, A, seed=5)
    ref = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(ref, n, n, seed=5)
    torch.cuda.synchronize()
    assert np.array_equal(local_to_lapack(A, n, nb, mt, nloc), ref.cpu().numpy().T)  # same input
    tq.dist_factor(n, n, A, nb, ib, T, info)
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
        tq.dist_fill_uniform(n, n, nb, A, seed=6)
        tq.dist_factor(n, n, A, nb, ib, T)
        torch.cuda.synchronize()
        outs.append((A.clone(), T.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("m,n,nb,ib,world", [
    (640, 640, 128, 32, 2),    # square
    (600, 600, 64, 16, 3),     # ragged: padded, 10 x 10 tiles
    (900, 400, 64, 16, 2),     # tall
    (400, 900, 96, 32, 4),     # wide, NB = 96
    (1000, 1000, 256, 16, 3),  # NB > 128: 8-warp CTAs
    (700, 1000, 160, 32, 2),   # NB = 160, ragged last slab
    (2048, 2048, 128, 16, 4),  # 16 x 16 tiles, thousands of items and copies
    (300, 300, 128, 16, 5),    # more ranks than some panels have consumers
])
def test_dist_emulated_ranks_bitwise_equal_factor(tq, m, n, nb, ib, world):
    import synth_inputs as si
    a = si.uniform(m, n, 80 + world)
    mt, nt = -(-m // nb), -(-n // nb)
    full = padded(a, nb)
    A = [to_local(full, nb, world, r) for r in range(world)]
    T = [torch.zeros(len(range(r, nt, world)) * mt * ib * nb, dtype=torch.float64, device="cuda")
         if A[r] is not None else None for r in range(world)]
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    for rep in range(2):  # the cached work list is reused on the second call
        if rep:
            for r in range(world):
                if A[r] is not None:
                    A[r].copy_(to_local(full, nb, world, r))
        tq.dist_emulate(world, m, n, A, nb, ib, T, info)
        torch.cuda.synchronize()
        assert int(info.item()) == 0
        ref = tq.to_colmajor(a)
        Tref, _ = tq.factor(ref, m, n, nb, ib)
        torch.cuda.synchronize()
        got = from_locals(A, nb, world, mt, nt)[:m, :n]
        assert np.array_equal(got, tq.from_colmajor(ref))
        tr = Tref.cpu().numpy()
        tile = ib * nb
        for r in range(world):
            if T[r] is None:
                continue
            tl = T[r].cpu().numpy()
            for j, k in enumerate(range(r, nt, world)):
                if k >= min(mt, nt):
                    continue
                for i in range(k, mt):
                    assert np.array_equal(tl[(i + j * mt) * tile:(i + j * mt + 1) * tile],
                                          tr[(i + k * mt) * tile:(i + k * mt + 1) * tile]), (r, i, k)


def test_tune_step2_through_dist_factor(tq, tmp_path, monkeypatch):
    """tileqr_tune's multi-GPU branch (Step 1 data set broadcast from rank 0,
    Step 2 timing tileqr_dist_factor with max-over-ranks times) on one rank,
    replayed through the oracle's tuner like the single-GPU tune."""
    import json
    from test_gpu_tune import replay
    monkeypatch.setenv("TILEQR_TUNE_DIST", "1")
    monkeypatch.setenv("TILEQR_TUNE_BATCH", "96")
    monkeypatch.setenv("TILEQR_TUNE_REPS", "3")
    path = tmp_path / "tune.json"
    nb, ib = tq.tune(768, 768, 1, 2, True, str(path))
    report = json.load(open(path))
    assert report["ngpus"] == 1
    replay(report, 2, True, nb, ib)


@pytest.mark.parametrize("m,n,nb,ib", [(640, 640, 128, 16), (900, 500, 64, 16), (500, 800, 96, 32)])
def test_dist_residual_via_apply_qt_local(tq, m, n, nb, ib):
    """The P > 1 residual check (bench.py --verify) at world size 1: Q^T A from
    the rank's own packed reflector slots equals the factor's R tiles, and
    ||Q^T A - R||_F / (||A||_F N eps) < 10 (north_star)."""
    import math
    mt = -(-m // nb)
    nloc = tq.dist_local_cols(n, nb)
    A = torch.empty(nloc * mt * nb * nb, dtype=torch.float64, device="cuda")
    tq.dist_fill_uniform(m, n, nb, A, seed=9)
    A0 = A.clone()
    T = torch.empty(nloc * mt * ib * nb, dtype=torch.float64, device="cuda")
    tq.dist_factor(m, n, A, nb, ib, T)
    B = A0.clone()
    tq.dist_apply_qt_local(m, n, B, nb, ib)
    torch.cuda.synchronize()
    res2 = float(tq.dist_residual_terms(m, n, nb, A, B, 0, 1))
    npad = sum(1 for j in range(n, nloc * nb) if m <= j < mt * nb)   # identity entries of the padding
    a2 = float(torch.sum(A0 ** 2)) - npad
    assert math.sqrt(res2) / (math.sqrt(a2) * max(m, n) * 2.0 ** -52) < 10
