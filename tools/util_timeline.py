"""Slot utilisation of one dataflow factorization over time: per bin, the
fraction of the grid's CTA slots running an item (inputs ready -> done), by
kind, plus the fraction claimed but waiting on inputs.

    python tools/util_timeline.py [--n 10000] [--ib 16] [--bin 1.0]
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
ap.add_argument("--bin", type=float, default=1.0)
a = ap.parse_args()
A0 = torch.empty((a.n, a.n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, a.n, a.n, seed=4)
tq.set_kernel_timing(True)
for _ in range(2):
    A = A0.clone()
    tq.factor(A, a.n, a.n, a.nb, a.ib)
    torch.cuda.synchronize()
recs = tq.kernel_trace(a.n, a.n, a.nb, a.ib, max_recs=1 << 22)
tq.set_kernel_timing(False)
slots = torch.cuda.get_device_properties(0).multi_processor_count * (2 if a.nb <= 128 else 1)
span = max(r[1] for r in recs)
nb = int(span / a.bin) + 1
kinds = ["geqrt", "tsqrt", "larfb", "ssrfb", "load", "store", "wait"]
busy = {k: [0.0] * nb for k in kinds}


def add(key, t0, t1):
    b = int(t0 / a.bin)
    while t0 < t1:
        e = min(t1, (b + 1) * a.bin)
        busy[key][b] += e - t0
        t0, b = e, b + 1


for t0, t1, kind, _, claim_ns in recs:
    add(kind, t0, t1)
    add("wait", claim_ns * 1e-6, t0)
print("span %.3f ms, %d slots" % (span, slots))
print("  ms  " + " ".join("%6s" % k for k in kinds) + "   idle")
for b in range(nb):
    f = [busy[k][b] / (slots * a.bin) for k in kinds]
    print("%5.1f " % (b * a.bin) + " ".join("%6.3f" % x for x in f) + "  %6.3f" % (1 - sum(f)))
tot = {k: sum(busy[k]) / (slots * span) for k in kinds}
print("total " + " ".join("%6.3f" % tot[k] for k in kinds) + "  %6.3f" % (1 - sum(tot.values())))
