"""GEQRT / TSQRT sub-task durations versus the step k in one dataflow run."""
import ctypes, json, os, sys, collections
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402
n, nb, ib = 10000, 128, 16
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)
tq.set_kernel_timing(True)
for _ in range(2):
    A = A0.clone(); tq.factor(A, n, n, nb, ib); torch.cuda.synchronize()
recs = tq.kernel_trace(n, n, nb, ib, max_recs=1 << 22)
tq.set_kernel_timing(False)
f = tq._lib.tileqr_debug_dag_item
f.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]
out = (ctypes.c_int * 5)()
g = collections.defaultdict(list); t = collections.defaultdict(list)
for i, r in enumerate(recs):
    f(n, n, nb, ib, i, out)
    kind, k, m, nn, s = list(out)
    if kind == 0: g[(k // 10, s)].append(r[1] - r[0])
    if kind == 1: t[(k // 10, s)].append(r[1] - r[0])
for key in sorted(g):
    tv = t.get(key, [0])
    print("k %2d-%2d sub %d: G %.1f us  T %.1f us" % (key[0] * 10, key[0] * 10 + 9, key[1],
          1e3 * sum(g[key]) / len(g[key]), 1e3 * sum(tv) / len(tv)))
