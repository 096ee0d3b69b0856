"""Phase cycles of the panel sub-tasks inside the DAG kernel (prof build:
TILEQR_LIB=paper_1102_5328_b200/libtileqr_prof.so), summed over all GEQRT and
TSQRT items of one 10000^2 NB=128 factorization."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

ib = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n, nb = int(sys.argv[2]) if len(sys.argv) > 2 else 10000, 128
f = tq._lib.tileqr_debug_dag_panel_prof
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = (ctypes.c_ulonglong * 16)()
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)
A = A0.clone()
tq.factor(A, n, n, nb, ib)
torch.cuda.synchronize()
f(out, 1)
A = A0.clone()
tq.factor(A, n, n, nb, ib)
torch.cuda.synchronize()
f(out, 1)
names = {0: "stage", 1: "factor", 2: "writeV", 5: "gram", 6: "Tdiag", 7: "Tmerge", 3: "Twrite+pack", 4: "trailing"}
nt = -(-n // nb)
for label, off, npan in (("TSQRT", 0, nt * (nt - 1) // 2 * (nb // ib)), ("GEQRT", 8, nt * (nb // ib))):
    ph = {v: out[k + off] for k, v in names.items()}
    tot = sum(ph.values())
    print(label, {k: round(v / npan) for k, v in ph.items()}, "cycles per inner panel, total %.0f" % (tot / npan))
