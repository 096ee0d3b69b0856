"""Critical path of one dataflow factorization, reconstructed from the
per-item trace: walks back from the last task through the dependency that
finished last and splits the path into item run time (per kind) and gaps
(dependency done -> item started: hand-off, claim order, co-residency).

    python tools/critical_path.py [--n 10000] [--nb 128] [--ib 16]
"""
import argparse
import collections
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--nb", type=int, default=128)
ap.add_argument("--ib", type=int, default=16)
a = ap.parse_args()
n, nb, ib = a.n, a.nb, a.ib
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)
tq.set_kernel_timing(True)
for _ in range(2):
    A = A0.clone()
    tq.factor(A, n, n, nb, ib)
    torch.cuda.synchronize()
recs = tq.kernel_trace(n, n, nb, ib, max_recs=1 << 22)
tq.set_kernel_timing(False)
f = tq._lib.tileqr_debug_dag_item
f.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]
out = (ctypes.c_int * 5)()
names = ["G", "T", "L", "S"]
task_start, task_end, task_claim = {}, {}, {}
for i, r in enumerate(recs):
    f(n, n, nb, ib, i, out)
    kind, k, m, nn, s = list(out)
    key = (names[kind], k, m, nn, s if kind < 2 else 0)
    task_start[key] = min(task_start.get(key, 1e30), r[0])
    task_end[key] = max(task_end.get(key, 0.0), r[1])
    task_claim[key] = max(task_claim.get(key, 0.0), r[4] * 1e-6)
NS = max(key[4] for key in task_end if key[0] == "G") + 1


def deps(t):
    kind, k, m, nn, s = t
    d = []
    if kind == "G":
        d.append(("G", k, k, k, s - 1) if s > 0 else ("S", k - 1, k, k, 0))
    elif kind == "L":
        d += [("G", k, k, k, NS - 1), ("S", k - 1, k, nn, 0)]
    elif kind == "T":
        d.append(("T", k, m, k, s - 1) if s > 0 else ("S", k - 1, m, k, 0))
        d.append(("G", k, k, k, s) if m == k + 1 else ("T", k, m - 1, k, s))
    else:
        d += [("T", k, m, k, NS - 1), ("L", k, k, nn, 0) if m == k + 1 else ("S", k, m - 1, nn, 0),
              ("S", k - 1, m, nn, 0)]
    return [x for x in d if x in task_end]


t = max(task_end, key=task_end.get)
span = task_end[t]
run = collections.Counter()
gap = collections.Counter()
late_claim = collections.Counter()  # part of the gap: the item was claimed after its input was final
tail = collections.Counter()        # run / gap of path tasks starting in the last 10 % of the span
path = []
while True:
    ds = deps(t)
    path.append(t)
    run[t[0]] += task_end[t] - task_start[t]
    if not ds:
        gap["start"] += task_start[t]
        break
    d = max(ds, key=task_end.get)
    gap[t[0]] += max(0.0, task_start[t] - task_end[d])
    late_claim[t[0]] += max(0.0, task_claim[t] - task_end[d])
    if task_start[t] > 0.9 * span:
        tail["run_" + t[0]] += task_end[t] - task_start[t]
        tail["gap_" + t[0]] += max(0.0, task_start[t] - task_end[d])
    t = d
print(json.dumps({"span_ms": round(span, 3), "path_tasks": len(path),
                  "run_ms": {k: round(v, 3) for k, v in run.items()},
                  "gap_ms_before": {k: round(v, 3) for k, v in gap.items()},
                  "late_claim_ms": {k: round(v, 3) for k, v in late_claim.items()},
                  "last_10pct": {k: round(v, 3) for k, v in sorted(tail.items())},
                  "kinds_on_path": dict(collections.Counter(x[0] for x in path))}))
