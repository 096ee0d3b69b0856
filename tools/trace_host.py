"""Trace of tileqr_factor_host (host-buffer pipeline): DAG items incl. LOAD /
STORE, the kernel span and the whole call's span (diagnostics)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

n, nb, ib = 10000, 128, 16
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, n, n, seed=4)
hA = A0.cpu().pin_memory()
hR = torch.empty_like(hA).pin_memory()
hT = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64).pin_memory()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for timing in (False, True):
    tq.set_kernel_timing(timing)
    for _ in range(2):
        e0.record()
        tq.factor_host(hA, n, n, nb, ib, hR=hR, hT=hT)
        e1.record()
        torch.cuda.synchronize()
    print(json.dumps({"timing": timing, "call_ms": round(e0.elapsed_time(e1), 3)}))
print(json.dumps({"dag_kernel_ms": round(tq.kernel_times(n, n, nb, ib, "dag")[0], 3)}))
recs = tq.kernel_trace(n, n, nb, ib, max_recs=1 << 21)
tq.set_kernel_timing(False)
json.dump({"n": n, "nb": nb, "ib": ib, "recs": recs}, open("gpurun_out/trace_host.json", "w"))
ld = sorted([r for r in recs if r[2] == "load"], key=lambda r: r[0])
st = sorted([r for r in recs if r[2] == "store"], key=lambda r: r[1])
print("load items: first start %.3f last end %.3f" % (ld[0][0], max(r[1] for r in ld)))
print("store items: first end %.3f last end %.3f" % (st[0][1], st[-1][1]))
print("span %.3f" % max(r[1] for r in recs))
# utilisation of the CTA slots per 2 ms (all kinds) -- where the host pipeline waits
slots = torch.cuda.get_device_properties(0).multi_processor_count * 2
span = max(r[1] for r in recs)
nb_ = int(span / 2.0) + 1
busy = [0.0] * nb_
for r in recs:
    t0, t1 = r[0], r[1]
    b = int(t0 / 2.0)
    while t0 < t1:
        e = min(t1, (b + 1) * 2.0)
        busy[b] += e - t0
        t0, b = e, b + 1
print("busy fraction per 2 ms:", " ".join("%.2f" % (x / (slots * 2.0)) for x in busy))
