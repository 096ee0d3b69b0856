"""Single-kernel cases for ncu captures (measurement only; no timing printed).

    python tools/kernel_cases.py ssrfb NB IB [--batch 4096] [--reps 3]
        the factorization's packed update kernel (update_v2_kernel) on a
        BASELINE configs[1] batch: 4096 independent tile pairs, V2/T from a
        TSQRT of uniform data, packed once; `reps` launches after one warm-up
    python tools/kernel_cases.py layout N NB IB
        one tileqr_factor of the N x N configs[3]-style matrix (layout_to_tiles,
        the DAG, tiles_to_layout)
    python tools/kernel_cases.py panel KIND NB IB [--batch B]
        one batched GEQRT / TSQRT launch (panel_fast_kernel) of B tasks
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402


def ssrfb(nb, ib, batch, reps):
    tile = nb * nb
    pk = tq.packed_size(nb, ib)
    buf = torch.empty(batch * 5 * tile, dtype=torch.float64, device="cuda")
    tq.rng_uniform(buf, tile, batch * 5, seed=2)
    pbuf = torch.empty(batch * pk, dtype=torch.float64, device="cuda")
    idx = torch.arange(batch, dtype=torch.int64, device="cuda") * 5 * tile * 8 + buf.data_ptr()
    R, V, C1, C2, T = (idx + j * tile * 8 for j in range(5))
    P = torch.arange(batch, dtype=torch.int64, device="cuda") * pk * 8 + pbuf.data_ptr()
    tq.tsqrt_batched(nb, ib, R, V, T)
    tq.pack_batched(False, nb, ib, V, T, P)
    for _ in range(1 + reps):
        tq.update_packed_batched(False, nb, ib, P, C1, C2)
    torch.cuda.synchronize()


def layout(n, nb, ib):
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(A, n, n, seed=4)
    tq.factor(A, n, n, nb, ib)
    torch.cuda.synchronize()


def panel(kind, nb, ib, batch):
    tile = nb * nb
    buf = torch.empty(batch * 3 * tile, dtype=torch.float64, device="cuda")
    tq.rng_uniform(buf, tile, batch * 3, seed=7)
    idx = torch.arange(batch, dtype=torch.int64, device="cuda") * 3 * tile * 8 + buf.data_ptr()
    R, A2, T = (idx + j * tile * 8 for j in range(3))
    for _ in range(2):
        if kind == "tsqrt":
            tq.tsqrt_batched(nb, ib, R, A2, T)
        else:
            tq.geqrt_batched(nb, ib, R, T)
    torch.cuda.synchronize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("args", nargs="*")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    v = [x for x in a.args]
    if a.case == "ssrfb":
        ssrfb(int(v[0]), int(v[1]), a.batch or 4096, a.reps)
    elif a.case == "layout":
        layout(int(v[0]), int(v[1]), int(v[2]))
    elif a.case == "panel":
        panel(v[0], int(v[1]), int(v[2]), a.batch or 148)
    else:
        ap.error("unknown case")
    print("ok")


if __name__ == "__main__":
    main()
