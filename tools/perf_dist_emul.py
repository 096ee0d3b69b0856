"""The multi-rank dataflow factorization with P EMULATED ranks on one GPU
(tileqr_dist_emulate: every rank's work list in one launch, COPY items
pushing packed panel tiles between the ranks' buffers in HBM) against the
single-GPU tileqr_factor of the same matrix: bitwise check and time.  This
measures the plan's overhead (copies, per-rank claim restrictions, arrival
counters), not NVLink.

    python tools/perf_dist_emul.py [--n 10000] [--nb 128 --ib 16] [--ranks 1,2,4,8]
"""
import argparse
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
    ap.add_argument("--ranks", default="1,2,4,8")
    a = ap.parse_args()
    n, nb, ib = a.n, a.nb, a.ib
    mt = -(-n // nb)
    ref = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(ref, n, n, seed=5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    A = ref.clone()
    T = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64, device="cuda")
    ts = []
    for r in range(4):
        A.copy_(ref)
        e0.record()
        tq.factor(A, n, n, nb, ib, T=T)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    single = sorted(ts)[1]
    print(json.dumps({"n": n, "nb": nb, "ib": ib, "single_gpu_ms": round(single, 3)}), flush=True)
    full = A  # the factored matrix (column-major storage)
    for P in (int(x) for x in a.ranks.split(",")):
        # local tile buffers of every rank from the padded input
        inp = ref.t()  # the matrix
        locs, Ts = [], []
        for rk in range(P):
            cols = list(range(rk, mt, P))
            buf = torch.zeros((len(cols), mt, nb, nb), dtype=torch.float64, device="cuda")
            for j, c in enumerate(cols):
                for m in range(mt):
                    blk = inp[m * nb:min(n, (m + 1) * nb), c * nb:min(n, (c + 1) * nb)]
                    buf[j, m, :blk.shape[1], :blk.shape[0]] = blk.t()
                    for d in range(nb):  # padded columns: e_j (R5)
                        g = c * nb + d
                        if g >= n and m * nb <= g < (m + 1) * nb:
                            buf[j, m, d, g - m * nb] = 1.0
            locs.append(buf.reshape(-1))
            Ts.append(torch.zeros(len(cols) * mt * ib * nb, dtype=torch.float64, device="cuda"))
        pristine = [x.clone() for x in locs]
        tq.dist_emulate(P, n, n, locs, nb, ib, Ts)   # builds the plan (host) and runs once
        torch.cuda.synchronize()
        ts = []
        for r in range(3):
            for x, p0 in zip(locs, pristine):
                x.copy_(p0)
            e0.record()
            tq.dist_emulate(P, n, n, locs, nb, ib, Ts)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = True
        fm = full.t()
        for rk in range(P):
            v = locs[rk].view(-1, mt, nb, nb)
            for j, c in enumerate(range(rk, mt, P)):
                for m in range(mt):
                    i1, j1 = min(n, (m + 1) * nb) - m * nb, min(n, (c + 1) * nb) - c * nb
                    ok = ok and bool(torch.equal(v[j, m].t()[:i1, :j1], fm[m * nb:m * nb + i1, c * nb:c * nb + j1]))
        ms = sorted(ts)[1]
        print(json.dumps({"ranks": P, "emulated_ms": round(ms, 3), "vs_single": round(single / ms, 3),
                          "bitwise_equal_to_single_gpu": ok}), flush=True)
        del locs, pristine, Ts
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
