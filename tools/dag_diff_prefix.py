"""Compare the result of a dataflow prefix between 2 CTAs/SM and 1 CTA/SM runs
and describe where it differs (diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

n, nb, ib = 4096, 128, 16
prefix = int(sys.argv[1])
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)
T = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64, device="cuda")


def run(grid):
    os.environ["TILEQR_DAG_NITEMS"] = str(prefix)
    os.environ["TILEQR_DAG_GRID"] = str(grid)
    A = A0.clone()
    tq.factor(A, n, n, nb, ib, T=T)
    torch.cuda.synchronize()
    return A


ref = run(148)
for rep in range(6):
    A = run(296)
    d = (A != ref)
    if not bool(d.any()):
        print(rep, "same")
        continue
    cols, rows = torch.nonzero(d, as_tuple=True)   # storage (col, row)
    tiles = {}
    for r, c in zip(rows.tolist(), cols.tolist()):
        key = (r // nb, c // nb)
        tiles.setdefault(key, []).append((r % nb, c % nb))
    for key, lst in sorted(tiles.items()):
        rs = sorted({x[0] for x in lst})
        cs = sorted({x[1] for x in lst})
        print(rep, "tile", key, len(lst), "rows", rs[0], "-", rs[-1], "cols", cs[0], "-", cs[-1],
              "max", float((A - ref).abs().max()))
