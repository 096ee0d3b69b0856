"""Where the CTAs of tileqr_factor_host's dataflow kernel are during the ramp:
per 1 ms bin, CTA-time busy (inputs ready -> done) and parked (claimed, inputs
not ready), the parked time split by the kind of the item claimed
(diagnostics; needs the timed build's per-item claim/start/end trace)."""
import collections
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
tq.set_kernel_timing(True)
for _ in range(2):
    tq.factor_host(hA, n, n, nb, ib, hR=hR, hT=hT)
    torch.cuda.synchronize()
recs = tq.kernel_trace(n, n, nb, ib, max_recs=1 << 21)   # (start, end, kind, level, claim_ns)
tq.set_kernel_timing(False)
bins = 20
busy = [0.0] * bins
parked = [collections.Counter() for _ in range(bins)]
for t0, t1, kind, lvl, claim_ns in recs:
    c = claim_ns * 1e-6
    for lo, hi, acc in ((c, t0, "parked"), (t0, t1, "busy")):
        b = int(lo)
        while lo < hi and b < bins:
            e = min(hi, b + 1.0)
            if acc == "busy":
                busy[b] += e - lo
            else:
                parked[b][kind] += e - lo
            lo, b = e, b + 1
slots = torch.cuda.get_device_properties(0).multi_processor_count * 2
for b in range(bins):
    print(json.dumps({"ms": b, "busy": round(busy[b] / slots, 3),
                      "parked": {k: round(v / slots, 3) for k, v in parked[b].most_common(4)}}))
