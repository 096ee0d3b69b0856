"""Quick performance scan of tileqr_factor and the batched SSRFB kernel.

    python tools/perf_scan.py [--n 10000] [--pairs 64:16,128:32,...] [--ssrfb]

Prints one JSON line per case: factor median ms, GFLOP/s (4/3 N^3), per-kind
kernel time shares (CUDA events inside the graph), and for --ssrfb the
4096-pair batched SSRFB rate.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402


def time_factor(n, nb, ib, reps=3, timing=False):
    A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(A0, n, n, seed=4)
    A = A0.clone()
    T = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    tq.set_kernel_timing(timing)
    times = []
    for r in range(reps + 1):
        A.copy_(A0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tq.factor(A, n, n, nb, ib, T=T, info=info)
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    times.sort()
    med = times[len(times) // 2]
    out = {"n": n, "nb": nb, "ib": ib, "ms": round(med, 3), "gflops": round(4 / 3 * n ** 3 / med / 1e6, 1)}
    if timing:
        for k in ("geqrt", "tsqrt", "larfb", "ssrfb"):
            tot, nl, nt = tq.kernel_times(n, n, nb, ib, k)
            out[k + "_ms"] = round(tot, 3)
            out[k + "_launches"] = nl
        tot, nl, nt = tq.kernel_times(n, n, nb, ib, "ssrfb")
        out["ssrfb_tflops_inkernel"] = round(nt * 4 * nb ** 3 / (tot * 1e-3) / 1e12, 2)
    tq.set_kernel_timing(False)
    return out


def time_ssrfb(nb, ib, batch=4096, reps=20):
    tile = nb * nb
    buf = torch.empty(batch * 5 * tile, dtype=torch.float64, device="cuda")
    tq.rng_uniform(buf, tile, batch * 5, seed=2)
    base = buf.data_ptr()
    idx = torch.arange(batch, dtype=torch.int64, device="cuda") * 5 * tile * 8 + base
    R, V, C1, C2, T = (idx + j * tile * 8 for j in range(5))
    tq.tsqrt_batched(nb, ib, R, V, T)
    tq.ssrfb_batched("T", nb, ib, V, T, C1, C2, nb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tq.ssrfb_batched("T", nb, ib, V, T, C1, C2, nb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"nb": nb, "ib": ib, "batch": batch, "ms": round(ms, 3),
            "tflops_nominal": round(batch * 4 * nb ** 3 / (ms * 1e-3) / 1e12, 2),
            "tflops_executed": round(batch * (4 * nb ** 3 + ib * nb * nb) / (ms * 1e-3) / 1e12, 2)}


def time_ssrfb_packed(nb, ib, batch=4096, reps=20):
    """The factorization's kernel alone: packed reflector tiles prepared once."""
    tile = nb * nb
    pk = tq.packed_size(nb, ib)
    buf = torch.empty(batch * 5 * tile, dtype=torch.float64, device="cuda")
    tq.rng_uniform(buf, tile, batch * 5, seed=2)
    pbuf = torch.empty(batch * pk, dtype=torch.float64, device="cuda")
    base = buf.data_ptr()
    idx = torch.arange(batch, dtype=torch.int64, device="cuda") * 5 * tile * 8 + base
    R, V, C1, C2, T = (idx + j * tile * 8 for j in range(5))
    P = torch.arange(batch, dtype=torch.int64, device="cuda") * pk * 8 + pbuf.data_ptr()
    tq.tsqrt_batched(nb, ib, R, V, T)
    tq.pack_batched(False, nb, ib, V, T, P)
    tq.update_packed_batched(False, nb, ib, P, C1, C2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tq.update_packed_batched(False, nb, ib, P, C1, C2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"kernel": "packed", "nb": nb, "ib": ib, "batch": batch, "ms": round(ms, 3),
            "tflops_nominal": round(batch * 4 * nb ** 3 / (ms * 1e-3) / 1e12, 2)}


def time_panel(nb, ib, batch=1, reps=50, kind="tsqrt"):
    tile = nb * nb
    buf = torch.empty(batch * 3 * tile, dtype=torch.float64, device="cuda")
    base = buf.data_ptr()
    idx = torch.arange(batch, dtype=torch.int64, device="cuda") * 3 * tile * 8 + base
    R, A2, T = (idx + j * tile * 8 for j in range(3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for r in range(reps + 1):
        tq.rng_uniform(buf, tile, batch * 3, seed=7 + r)
        e0.record()
        if kind == "tsqrt":
            tq.tsqrt_batched(nb, ib, R, A2, T)
        else:
            tq.geqrt_batched(nb, ib, R, T)
        e1.record()
        torch.cuda.synchronize()
        if r:
            tot += e0.elapsed_time(e1)
    us = 1e3 * tot / reps
    return {"kind": kind, "nb": nb, "ib": ib, "batch": batch, "us": round(us, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[10000])
    ap.add_argument("--pairs", default="64:16,96:32,128:32,160:32,192:32,256:32")
    ap.add_argument("--ssrfb", action="store_true")
    ap.add_argument("--timing", action="store_true")
    ap.add_argument("--panel", action="store_true")
    a = ap.parse_args()
    pairs = [tuple(int(v) for v in p.split(":")) for p in a.pairs.split(",")]
    if a.panel:
        for nb, ib in pairs:
            for kind in ("geqrt", "tsqrt"):
                print(json.dumps(time_panel(nb, ib, kind=kind)), flush=True)
    if a.ssrfb:
        for nb, ib in pairs:
            if tq.packed_size(nb, ib):
                print(json.dumps(time_ssrfb_packed(nb, ib)), flush=True)
            os.environ["TILEQR_NO_V2"] = "1"
            print(json.dumps(time_ssrfb(nb, ib)), flush=True)
            os.environ.pop("TILEQR_NO_V2")
    for n in a.n:
        for nb, ib in pairs:
            print(json.dumps(time_factor(n, nb, ib, timing=a.timing)), flush=True)


if __name__ == "__main__":
    main()
