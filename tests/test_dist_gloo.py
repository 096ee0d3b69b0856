"""Multi-rank schedule of the distributed tile QR, on the CPU with gloo.

The library's host planner (tileqr_dist_plan_level, the same code that drives
tileqr_dist_factor's kernels and NCCL broadcasts) is executed by world-size-2
gloo processes: each rank owns the tile columns n with n % P == rank, runs its
planned panel tasks with the oracle's kernels, broadcasts the planned V/T
tiles with torch.distributed (gloo) from the planned root, and runs its
planned update tasks reading V/T from the received panel buffers.  The result
must equal the single-process oracle factorization BITWISE (every tile sees
the same operations on the same inputs).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, nb, ib, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle
    import synth_inputs as si
    from paper_1102_5328_b200 import tileqr as tq

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mt = n // nb
        a = si.uniform(n, n, 5)
        tiles = {(m, c): np.asfortranarray(a[m * nb:(m + 1) * nb, c * nb:(c + 1) * nb])
                 for c in range(mt) if c % world == rank for m in range(mt)}
        tloc = {}
        pv, pt = {}, {}
        for t in range(3 * mt - 2):
            panel, bcast, update = tq.dist_plan_level(mt, world, rank, t)
            snap = {}
            for kind, k, m, _, _ in panel:
                if kind == 0:
                    tiles[(k, k)], tloc[(k, k)] = oracle.geqrt(tiles[(k, k)], ib)
                    snap[k] = tiles[(k, k)].copy()
                else:
                    r, v2, tt = oracle.tsqrt(tiles[(k, k)], tiles[(m, k)], ib)
                    tiles[(k, k)] = np.asfortranarray(np.triu(r) + np.tril(tiles[(k, k)], -1))
                    tiles[(m, k)], tloc[(m, k)] = v2, tt
            for _, k, m, _, src in bcast:
                # flat column-major buffers, exactly the bytes NCCL moves on the GPU
                if src == rank:
                    v = snap[k] if m == k else tiles[(m, k)]
                    tv = torch.from_numpy(np.asfortranarray(v).ravel(order="F").copy())
                    tt = torch.from_numpy(np.asfortranarray(tloc[(m, k)]).ravel(order="F").copy())
                else:
                    tv, tt = torch.empty(nb * nb, dtype=torch.float64), torch.empty(ib * nb, dtype=torch.float64)
                dist.broadcast(tv, src=src)
                dist.broadcast(tt, src=src)
                pv[(k, m)] = tv.numpy().reshape((nb, nb), order="F")
                pt[(k, m)] = tt.numpy().reshape((ib, nb), order="F")
            for kind, k, m, c, _ in update:
                assert c % world == rank
                if kind == 2:
                    tiles[(k, c)] = oracle.larfb(pv[(k, k)], pt[(k, k)], tiles[(k, c)], "T")
                else:
                    tiles[(k, c)], tiles[(m, c)] = oracle.ssrfb(pv[(k, m)], pt[(k, m)], tiles[(k, c)],
                                                                tiles[(m, c)], "T")
        q.put((rank, {key: v.copy() for key, v in tiles.items()},
               {key: v.copy() for key, v in tloc.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nb,ib,world", [(96, 16, 4, 2), (80, 16, 8, 2), (64, 16, 16, 3)])
def test_distributed_schedule_is_bitwise_the_single_process_factorization(n, nb, ib, world):
    import oracle
    import synth_inputs as si
    from paper_1102_5328_b200 import build
    build.build()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, ib, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = si.uniform(n, n, 5)
    f, t, _ = oracle.tileqr_factor(a, nb, ib)
    mt = n // nb
    seen = set()
    for rank, tiles, tloc in results:
        for (m, c), v in tiles.items():
            assert c % world == rank
            ref = f[m * nb:(m + 1) * nb, c * nb:(c + 1) * nb]
            if m == c:  # diagonal tile: R upper + V strictly lower
                assert np.array_equal(v, ref), (m, c)
            else:
                assert np.array_equal(v, ref), (m, c)
            seen.add((m, c))
        for (m, k), tt in tloc.items():
            assert np.array_equal(tt, oracle.t_tile(t, n, n, nb, ib, m, k)), (m, k)
    assert seen == {(m, c) for m in range(mt) for c in range(mt)}


def test_plan_covers_every_task_exactly_once():
    """Union over ranks and levels of the planned tasks is the whole DAG, each
    task on the owner of its column; broadcast roots own column k."""
    from oracle.tuner import dag_levels
    from paper_1102_5328_b200 import tileqr as tq
    for mt, world in [(5, 2), (7, 3), (4, 4), (6, 1)]:
        got = {}
        for rank in range(world):
            for t in range(3 * mt - 2):
                panel, bcast, update = tq.dist_plan_level(mt, world, rank, t)
                for kind, k, m, c, root in panel:
                    key = ("G", k) if kind == 0 else ("T", k, m)
                    assert k % world == rank and key not in got
                    got[key] = t
                for kind, k, m, c, root in update:
                    key = ("L", k, c) if kind == 2 else ("S", k, m, c)
                    assert c % world == rank and key not in got
                    got[key] = t
                for kind, k, m, c, root in bcast:
                    assert root == k % world
        assert got == dag_levels(mt, mt)
