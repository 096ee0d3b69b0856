"""Bitwise check of the dataflow kernel against the level launcher at scale.

    python tools/dag_check.py [--n 10000] [--nb 128] [--ib 16] [--reps 3]
Prints, per DAG run, whether A and T equal the level-synchronous result and
the first differing tiles (tile row, tile column) in tile-column order.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--nb", type=int, default=128)
ap.add_argument("--ib", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n, nb, ib = a.n, a.nb, a.ib
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)


def run(sched):
    tq.finalize()
    if sched:
        os.environ["TILEQR_SCHED"] = sched
    else:
        os.environ.pop("TILEQR_SCHED", None)
    A = A0.clone()
    T, info = tq.factor(A, n, n, nb, ib)
    torch.cuda.synchronize()
    return A, T


Ar, Tr = run("levels")
mt = -(-n // nb)
for r in range(a.reps):
    A, T = run(None)
    eqA, eqT = torch.equal(A, Ar), torch.equal(T, Tr)
    msg = f"rep {r}: A equal {eqA}, T equal {eqT}"
    if not eqA:
        d = (A != Ar)  # column-major storage: row index of the tensor = column of the matrix
        cols, rows = torch.nonzero(d, as_tuple=True)
        tiles = sorted({(int(rr) // nb, int(cc) // nb) for rr, cc in zip(rows[:200000].tolist(), cols[:200000].tolist())},
                       key=lambda x: (x[1], x[0]))
        msg += f"; {int(d.sum())} entries differ, max |diff| {float((A - Ar).abs().max()):.3e}, first tiles {tiles[:12]}"
    print(msg, flush=True)
