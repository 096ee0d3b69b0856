"""Run tileqr_factor of an N x N uniform matrix a few times (for ncu captures).

    python tools/run_factor.py [--n 10000] [--nb 128] [--ib 16] [--reps 2]
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
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
A0 = torch.empty((a.n, a.n), dtype=torch.float64, device="cuda")
tq.rng_uniform(A0, a.n, a.n, seed=4)
A = A0.clone()
T = torch.empty(tq.t_size(a.n, a.n, a.nb, a.ib), dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    A.copy_(A0)
    tq.factor(A, a.n, a.n, a.nb, a.ib, T=T)
torch.cuda.synchronize()
print("ok")
