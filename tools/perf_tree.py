"""Flat tree vs reduction tree on tall-skinny and square
shapes: median of 5 timed tileqr_factor / tileqr_factor_tree calls after one
warm-up, CUDA events, input restored from a pristine device copy outside the
events.  Rate = (2MN^2 - 2N^3/3) / t.

    python tools/perf_tree.py [--shapes 65536x512,...] [--nb 128 --ib 16] [--bs 1,4,16]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402


def flops(m, n):
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0 if m >= n else 2.0 * n * m * m - 2.0 * m ** 3 / 3.0


def timeit(fn, A, A0, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(reps + 1):
        A.copy_(A0)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="131072x256,65536x512,32768x1024,16384x2048,2048x2048,10000x10000")
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--ib", type=int, default=16)
    ap.add_argument("--bs", default="1,2,4,8,16")
    a = ap.parse_args()
    for sh in a.shapes.split(","):
        m, n = (int(x) for x in sh.split("x"))
        for nb, ib in ([(a.nb, a.ib), (64, 16)] if m > 4 * n else [(a.nb, a.ib)]):
            A0 = torch.empty((n, m), dtype=torch.float64, device="cuda")
            tq.rng_uniform(A0, m, n, seed=6)
            A = torch.empty_like(A0)
            T = torch.empty(tq.t_size(m, n, nb, ib), dtype=torch.float64, device="cuda")
            ms = timeit(lambda: tq.factor(A, m, n, nb, ib, T=T), A, A0)
            row = {"m": m, "n": n, "nb": nb, "ib": ib, "flat_ms": round(ms, 3),
                   "flat_gflops": round(flops(m, n) / ms / 1e6, 1), "tree": []}
            T2 = torch.empty(tq.t_size_tree(m, n, nb, ib), dtype=torch.float64, device="cuda")
            for bs in (int(x) for x in a.bs.split(",")):
                if bs >= -(-m // nb):
                    continue
                mt = timeit(lambda: tq.factor_tree(A, m, n, nb, ib, bs, T=T2), A, A0)
                row["tree"].append({"bs": bs, "ms": round(mt, 3), "gflops": round(flops(m, n) / mt / 1e6, 1),
                                    "speedup": round(ms / mt, 2)})
            tq.finalize()
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
