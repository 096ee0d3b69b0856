"""Install-time autotuning on the GPU (BASELINE configs[1..3]).

    python tools/autotune.py [--n 2048 10000] [--es 2048] [--out profiles/tune_r01.json]

For every N: tileqr_tune (Step 1 SSRFB sweep over the (NB, IB) grid, Property 1,
upper hull, Heuristic 2, Step 2 with prune-as-you-go) -> decision table
paper_1102_5328_b200/tuned_table.json (nearest-point lookup).
With --es N0: exhaustive search over the full 74-pair grid at N0 (BASELINE
configs[2]) and the tuned pick's rate as % of the ES optimum (Table 2 style).
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

GRID = {nb: [d for d in range(1, nb + 1) if nb % d == 0] for nb in (64, 96, 128, 160, 192, 224, 256)}


def factor_rate(n, nb, ib, reps=6):
    A0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tq.rng_uniform(A0, n, n, seed=3)
    A = torch.empty_like(A0)
    T = torch.empty(tq.t_size(n, n, nb, ib), dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for r in range(reps + 1):
        A.copy_(A0)
        e0.record()
        tq.factor(A, n, n, nb, ib, T=T, info=info)
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    times.sort()
    med = 0.5 * (times[(reps - 1) // 2] + times[reps // 2])
    return 4.0 / 3.0 * n ** 3 / (med * 1e-3) / 1e9, med


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[500, 1000, 2000, 2048, 4000, 6000, 8000, 10000])  # P:612-623 grid + configs[2]
    ap.add_argument("--es", type=int, default=2048)
    ap.add_argument("--heuristic", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "tune_r01.json"))
    ap.add_argument("--table", default=os.path.join(ROOT, "gpurun_out", "tuned_table.json"))
    a = ap.parse_args()
    report = {"gpu": torch.cuda.get_device_name(0), "heuristic": a.heuristic, "payg": True, "runs": []}
    entries = []
    for n in a.n:
        path = os.path.join(ROOT, "gpurun_out", f"tune_{n}.json")
        t0 = time.time()
        nb, ib = tq.tune(n, n, 1, a.heuristic, True, path)
        wall = time.time() - t0
        detail = json.load(open(path))
        g, ms = factor_rate(n, nb, ib)
        report["runs"].append({"n": n, "nb": nb, "ib": ib, "gflops": g, "ms": ms, "tune_wall_s": wall,
                               "candidates": detail["candidates"], "step2": detail["step2"],
                               "step1": detail["step1"]})
        entries.append({"n": n, "ngpus": 1, "nb": nb, "ib": ib, "gflops": g})
        print(json.dumps({"n": n, "nb": nb, "ib": ib, "gflops": round(g, 1), "tune_wall_s": round(wall, 1)}),
              flush=True)
    if a.es:
        es = []
        for nb, ibs in GRID.items():
            for ib in ibs:
                g, ms = factor_rate(a.es, nb, ib)
                es.append({"nb": nb, "ib": ib, "gflops": g, "ms": ms})
        best = max(es, key=lambda r: r["gflops"])
        tuned = next((r for r in report["runs"] if r["n"] == a.es), None)
        res = {"n": a.es, "pairs": len(es), "es_best": best, "all": es}
        if tuned:
            g_t = next(r["gflops"] for r in es if r["nb"] == tuned["nb"] and r["ib"] == tuned["ib"])
            res["tuned_pick"] = {"nb": tuned["nb"], "ib": tuned["ib"], "gflops": g_t,
                                 "pct_of_es": 100.0 * g_t / best["gflops"],
                                 "optimum_found": (tuned["nb"], tuned["ib"]) == (best["nb"], best["ib"])}
        report["exhaustive_search"] = res
        print(json.dumps({k: v for k, v in res.items() if k != "all"}), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(report, open(a.out + ".tmp", "w"), indent=1)
    os.replace(a.out + ".tmp", a.out)
    table = {"format_version": 1, "machine": torch.cuda.get_device_name(0), "heuristic": a.heuristic,
             "payg": True, "entries": entries}
    tmp = a.table + ".tmp"  # written atomically: a reader never sees a partial table
    json.dump(table, open(tmp, "w"), indent=1)
    os.replace(tmp, a.table)


if __name__ == "__main__":
    main()
