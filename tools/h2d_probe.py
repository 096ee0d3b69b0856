"""H2D copy throughput of the factor_host input pipeline, alone and while the
dataflow kernel runs (diagnostics)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

n, nb = 10000, 128
h = torch.empty((n, n), dtype=torch.float64).pin_memory()
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for trial in ("alone", "with_dag"):
    A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(A0, n, n, seed=4)
    torch.cuda.synchronize()
    if trial == "with_dag":
        tq.factor(A0, n, n, nb, 16)  # on the default stream, runs ~55 ms
    with torch.cuda.stream(s):
        e0.record(s)
        for c in range(0, n, nb):
            d[c:c + nb].copy_(h[c:c + nb], non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(trial, "H2D 800 MB in %.2f ms = %.1f GB/s" % (ms, 0.8 / (ms * 1e-3)))
