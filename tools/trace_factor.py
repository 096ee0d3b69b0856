"""Per-level launch trace of one tileqr_factor (CUDA events around every launch).

    python tools/trace_factor.py [--n 10000] [--nb 128] [--ib 16] [--out gpurun_out/trace.json]

Prints a summary: per-kind totals, panel-stream busy time, and the levels
grouped in bands with their wall time (first start .. last end of the level).
"""
import argparse
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--ib", type=int, default=16)
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--band", type=int, default=16)
    a = ap.parse_args()
    n, nb, ib = a.n, a.nb, a.ib
    A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(A0, n, n, seed=4)
    A = A0.clone()
    T = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    for timing in (False, True):
        tq.set_kernel_timing(timing)
        for _ in range(3):
            A.copy_(A0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tq.factor(A, n, n, nb, ib, T=T, info=info)
            e1.record()
            torch.cuda.synchronize()
        print(json.dumps({"timing": timing, "ms": round(e0.elapsed_time(e1), 3)}), flush=True)
    recs = tq.kernel_trace(n, n, nb, ib, max_recs=1 << 21)
    try:
        print(json.dumps({"dag_kernel_ms": round(tq.kernel_times(n, n, nb, ib, "dag")[0], 3)}))
    except tq.TileQRError:
        pass
    tq.set_kernel_timing(False)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump({"n": n, "nb": nb, "ib": ib, "recs": recs}, open(a.out, "w"))
    per = collections.defaultdict(float)
    for t0, t1, k, lv, nt in recs:
        per[k] += t1 - t0
    print(json.dumps({k: round(v, 3) for k, v in per.items()}))
    lv = collections.defaultdict(list)
    for r in recs:
        lv[r[3]].append(r)
    levels = sorted(lv)
    span = max(r[1] for r in recs) - min(r[0] for r in recs)
    print(f"levels {len(levels)}  span {span:.3f} ms")
    for b0 in range(0, len(levels), a.band):
        band = levels[b0:b0 + a.band]
        st = min(r[0] for l in band for r in lv[l])
        en = max(r[1] for l in band for r in lv[l])
        pan = sum(r[1] - r[0] for l in band for r in lv[l] if r[2] in ("geqrt", "tsqrt"))
        upd = sum(r[1] - r[0] for l in band for r in lv[l] if r[2] in ("larfb", "ssrfb"))
        ns = sum(r[4] for l in band for r in lv[l] if r[2] == "ssrfb")
        print(f"levels {band[0]:4d}-{band[-1]:4d}: wall {en - st:7.3f} ms  panel {pan:7.3f}  update {upd:7.3f}"
              f"  ssrfb tasks {ns:6d}  ({ns * 4 * nb ** 3 / max(upd, 1e-9) / 1e9:6.1f} TF in update)")


if __name__ == "__main__":
    main()
