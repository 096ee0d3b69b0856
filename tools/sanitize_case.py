"""Small cases for compute-sanitizer runs (one tool per gpurun call).

    python tools/sanitize_case.py [dag|levels|all]

dag:    configs[0] (256^2, NB=64, IB=16) and 384^2 at NB=128 through the
        persistent dataflow kernel, the host-buffer pipeline (LOAD / STORE
        items), apply_qt both ways, and 2 emulated ranks of the multi-rank
        dataflow kernel (COPY items);
levels: the same shapes through the level-synchronous batched launcher and
        the batched kernels (GEQRT / TSQRT / LARFB / SSRFB, packed update).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth_inputs as si  # noqa: E402
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402


def factor_cases():
    for (m, n, nb, ib) in [(256, 256, 64, 16), (384, 384, 128, 16), (300, 200, 64, 32)]:
        a = si.uniform(m, n, 1)
        A = tq.to_colmajor(a)
        T, info = tq.factor(A, m, n, nb, ib)
        B = tq.to_colmajor(si.uniform(m, 5, 2))
        tq.apply_qt("T", A, m, n, T, nb, ib, B, 5)
        tq.apply_qt("N", A, m, n, T, nb, ib, B, 5)
        hA = torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory()
        hR = torch.empty_like(hA).pin_memory()
        hT = torch.empty(T.numel(), dtype=torch.float64).pin_memory()
        tq.factor_host(hA, m, n, nb, ib, hR=hR, hT=hT, info=info)
        torch.cuda.synchronize()
        assert int(info.item()) == 0
        print("factor ok", m, n, nb, ib, flush=True)


def emulated():
    m = n = 384
    nb, ib, world = 128, 16, 2
    mt = nt = 3
    A = []
    for r in range(world):
        cols = len(range(r, nt, world))
        buf = torch.empty(cols * mt * nb * nb, dtype=torch.float64, device="cuda")
        buf.copy_(torch.rand(buf.numel(), dtype=torch.float64))
        A.append(buf)
    T = [torch.zeros(len(range(r, nt, world)) * mt * ib * nb, dtype=torch.float64, device="cuda")
         for r in range(world)]
    tq.dist_emulate(world, m, n, A, nb, ib, T)
    torch.cuda.synchronize()
    print("emulated ranks ok", flush=True)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    if mode == "levels":
        os.environ["TILEQR_SCHED"] = "levels"
    factor_cases()
    if mode != "levels":
        emulated()
    print("done")
