"""The multi-rank DATAFLOW plan (tileqr_dist_plan_items: the per-rank work
lists of the persistent kernel, with the panel broadcast as COPY items) run
on the CPU by world-size-2/3 gloo processes.

Each rank walks its own work list IN CLAIM ORDER with one worker, executing
the items with the oracle's tile kernels: GEQRT / TSQRT on its panels (the
packed slot of reflector tile (k, m) = the V / T the panel produced), COPY
as a non-blocking gloo send of that slot to the destination rank, LARFB /
SSRFB column slabs reading the slot -- received from the owner when the
item's dependency is an ARRIVE.  This checks the host plan itself:
  * every local dependency is already complete when an item is reached
    (the claim order is topological on every rank);
  * walking the per-rank orders with one worker each never deadlocks across
    ranks (the orders are restrictions of one global order, sched.h);
  * the result is BITWISE the single-process oracle factorization (every
    tile sees the same operations on the same inputs).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GEQRT, TSQRT, LARFB, SSRFB, COPY = 0, 1, 2, 3, 7


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m_, n_, nb, ib, workers, q):
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
        mt, nt = m_ // nb, n_ // nb
        cols = {32: 32, 64: 32, 96: 64, 128: 64}[nb]   # update columns per item (dag_item.h dag_cols)
        a = si.uniform(m_, n_, 9)
        tiles = {(m, c): np.asfortranarray(a[m * nb:(m + 1) * nb, c * nb:(c + 1) * nb])
                 for c in range(nt) if c % world == rank for m in range(mt)}
        tloc, slot, sends = {}, {}, []
        rows = tq.dist_plan_items(m_, n_, nb, ib, world, rank, workers, nb)
        mine = {r[5] for r in rows}
        parts = {}
        for r in rows:
            parts[r[5]] = parts.get(r[5], 0) + 1
        count = {}
        done = set()
        for kind, k, m, c, s, task, deps in rows:
            for d in deps:
                if d in mine:
                    assert d in done, ("claimed before its input", kind, k, m, c, d)
            remote = [d for d in deps if d not in mine]
            if remote:  # ARRIVE: the copy of reflector tile (k, m) from its owner
                key = (k, k) if kind == LARFB else (k, m)
                assert kind in (LARFB, SSRFB) and k % world != rank and len(remote) == 1
                if key not in slot:
                    v = torch.empty(nb * nb, dtype=torch.float64)
                    t = torch.empty(ib * nb, dtype=torch.float64)
                    dist.recv(v, src=k % world, tag=2 * (key[0] * mt + key[1]))
                    dist.recv(t, src=k % world, tag=2 * (key[0] * mt + key[1]) + 1)
                    slot[key] = (v.numpy().reshape((nb, nb), order="F"), t.numpy().reshape((ib, nb), order="F"))
            if kind == GEQRT:
                assert k % world == rank
                tiles[(k, k)], tloc[(k, k)] = oracle.geqrt(tiles[(k, k)], ib)
                slot[(k, k)] = (tiles[(k, k)].copy(), tloc[(k, k)].copy())
            elif kind == TSQRT:
                assert k % world == rank
                r_, v2, tt = oracle.tsqrt(tiles[(k, k)], tiles[(m, k)], ib)
                tiles[(k, k)] = np.asfortranarray(np.triu(r_) + np.tril(tiles[(k, k)], -1))
                tiles[(m, k)], tloc[(m, k)] = v2, tt
                slot[(k, m)] = (v2.copy(), tt.copy())
            elif kind == COPY:
                assert k % world == rank and s != rank
                v, t = slot[(k, m)]
                sends.append(dist.isend(torch.from_numpy(v.ravel(order="F").copy()), dst=s, tag=2 * (k * mt + m)))
                sends.append(dist.isend(torch.from_numpy(t.ravel(order="F").copy()), dst=s, tag=2 * (k * mt + m) + 1))
            elif kind == LARFB:
                assert c % world == rank
                v, t = slot[(k, k)]
                j0, j1 = s * cols, min(nb, (s + 1) * cols)
                cur = tiles[(k, c)].copy()
                cur[:, j0:j1] = oracle.larfb(v, t, cur[:, j0:j1], "T")
                tiles[(k, c)] = np.asfortranarray(cur)
            elif kind == SSRFB:
                assert c % world == rank
                v, t = slot[(k, m)]
                j0, j1 = s * cols, min(nb, (s + 1) * cols)
                c1, c2 = tiles[(k, c)].copy(), tiles[(m, c)].copy()
                c1[:, j0:j1], c2[:, j0:j1] = oracle.ssrfb(v, t, c1[:, j0:j1], c2[:, j0:j1], "T")
                tiles[(k, c)], tiles[(m, c)] = np.asfortranarray(c1), np.asfortranarray(c2)
            else:
                raise AssertionError(kind)
            count[task] = count.get(task, 0) + 1
            if count[task] == parts[task]:
                done.add(task)
        for h in sends:
            h.wait()
        assert done == mine
        q.put((rank, {key: v.copy() for key, v in tiles.items()},
               {key: v.copy() for key, v in tloc.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,nb,ib,world,workers", [
    (384, 384, 64, 16, 2, 4),     # square, 6 x 6 tiles, 2 update slabs per tile
    (512, 256, 64, 32, 3, 3),     # tall
    (256, 448, 64, 8, 2, 2),      # wide
    (320, 320, 32, 8, 3, 8),      # 10 x 10 tiles, one slab
])
def test_dataflow_plan_executes_to_the_oracle_factorization(m, n, nb, ib, world, workers):
    import oracle
    import synth_inputs as si
    from paper_1102_5328_b200 import build
    build.build()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, nb, ib, workers, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = si.uniform(m, n, 9)
    f, t, _ = oracle.tileqr_factor(a, nb, ib)
    mt, nt = m // nb, n // nb
    seen = set()
    for rank, tiles, tloc in results:
        for (i, c), v in tiles.items():
            assert c % world == rank
            assert np.array_equal(v, f[i * nb:(i + 1) * nb, c * nb:(c + 1) * nb]), (i, c)
            seen.add((i, c))
        for (i, k), tt in tloc.items():
            assert np.array_equal(tt, oracle.t_tile(t, m, n, nb, ib, i, k)), (i, k)
    assert seen == {(i, c) for i in range(mt) for c in range(nt)}


def test_dataflow_plan_structure():
    """Every task of the flat-tree DAG runs exactly once, on the owner of its
    column (panels: column k), with one COPY per (reflector tile, consumer
    rank) and no COPY to a rank that owns no later column."""
    from paper_1102_5328_b200 import tileqr as tq
    for m, n, nb, ib, world in [(512, 512, 64, 16, 3), (640, 256, 128, 32, 4), (256, 640, 64, 8, 2)]:
        mt, nt = -(-m // nb), -(-n // nb)
        kt = min(mt, nt)
        seen, copies = {}, set()
        for rank in range(world):
            for kind, k, i, c, s, task, deps in tq.dist_plan_items(m, n, nb, ib, world, rank, 4, 32):
                if kind in (GEQRT, TSQRT):
                    assert k % world == rank
                    seen[(kind, k, i, s)] = seen.get((kind, k, i, s), 0) + 1
                elif kind in (LARFB, SSRFB):
                    assert c % world == rank
                    seen[(kind, k, i, c, s)] = seen.get((kind, k, i, c, s), 0) + 1
                else:
                    assert kind == COPY and k % world == rank and s != rank
                    assert any(cc % world == s for cc in range(k + 1, nt))
                    assert (k, i, s) not in copies
                    copies.add((k, i, s))
        assert all(v == 1 for v in seen.values())
        nslab = 2 if nb == 128 else 2 if nb == 64 else 1
        ns = nb // 32
        want = kt * ns + sum((mt - k - 1) * ns for k in range(kt)) + \
            nslab * sum((nt - k - 1) + (mt - k - 1) * (nt - k - 1) for k in range(kt))
        assert len(seen) == want
        want_cp = sum((mt - k) * len({cc % world for cc in range(k + 1, nt)} - {k % world}) for k in range(kt))
        assert len(copies) == want_cp
