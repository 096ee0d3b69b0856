"""Find the shortest prefix of the dataflow claim order whose result differs
between a run with 2 CTAs per SM and a run with 1 CTA per SM (diagnostics).

    python tools/dag_bisect.py [--n 4096] [--nb 128] [--ib 16]
"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--nb", type=int, default=128)
ap.add_argument("--ib", type=int, default=16)
a = ap.parse_args()
n, nb, ib = a.n, a.nb, a.ib
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)
T = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64, device="cuda")


def run(prefix, grid):
    os.environ["TILEQR_DAG_NITEMS"] = str(prefix)
    os.environ["TILEQR_DAG_GRID"] = str(grid)
    A = A0.clone()
    tq.factor(A, n, n, nb, ib, T=T)
    torch.cuda.synchronize()
    return A


def differs(prefix):
    ref = run(prefix, 148)
    for _ in range(3):
        if not torch.equal(run(prefix, 296), ref):
            return True
    return False


run(1, 148)
f = tq._lib.tileqr_debug_dag_item
f.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]
nitems = 0
out = (ctypes.c_int * 5)()
while f(n, n, nb, ib, nitems, out) == 0:
    nitems += 1
print("items", nitems, flush=True)
lo, hi = 0, nitems
if not differs(hi):
    print("no difference at full length")
    sys.exit(0)
while hi - lo > 1:
    mid = (lo + hi) // 2
    d = differs(mid)
    print(f"prefix {mid}: {'DIFF' if d else 'same'}", flush=True)
    if d:
        hi = mid
    else:
        lo = mid
names = ["G", "T", "L", "S"]
for i in range(max(0, hi - 6), hi):
    f(n, n, nb, ib, i, out)
    print(i, names[out[0]], list(out)[1:])
