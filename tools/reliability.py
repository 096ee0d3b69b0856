"""Tuner reliability study (Tables 2-3 style):
for several N, the exhaustive search (ES) over the full (NB, IB) grid and the
pick of the two-step tuner with Heuristics 0/1/2 (prune-as-you-go) and with
H2 without PAYG; each pick's rate as % of the ES optimum.

    python tools/reliability.py [--n 1024 2048 4096] [--out gpurun_out/reliability.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402
from tools.autotune import GRID, factor_rate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="*", default=[1024, 2048, 4096])
ap.add_argument("--out", default="gpurun_out/reliability.json")
ap.add_argument("--table", default=None, help="decision table: also score its nearest-point pick (on/off grid)")
ap.add_argument("--no-tune", action="store_true", help="score only the table's pick (no per-N tuning)")
a = ap.parse_args()
rows = []
for n in a.n:
    t0 = time.time()
    es = {}
    for nb, ibs in GRID.items():
        for ib in ibs:
            es[(nb, ib)] = factor_rate(n, nb, ib)[0]
            tq.finalize()
    best = max(es, key=es.get)
    es_wall = time.time() - t0
    row = {"n": n, "es_best": {"nb": best[0], "ib": best[1], "gflops": es[best]}, "es_pairs": len(es),
           "es_wall_s": round(es_wall, 1), "tuners": []}
    if a.table:
        os.environ["TILEQR_TUNED_TABLE"] = a.table
        grid_n = sorted({e["n"] for e in json.load(open(a.table))["entries"]})
        nb, ib, found = tq.lookup(n, n, 1)
        g = es.get((nb, ib), factor_rate(n, nb, ib)[0])
        row["table_pick"] = {"nb": nb, "ib": ib, "gflops": g, "pct_of_es": 100.0 * g / es[best],
                             "optimum": (nb, ib) == best, "on_grid": n in grid_n, "table_n": grid_n,
                             "from_table": found}
        print(json.dumps({"n": n, "table_pick": row["table_pick"]}), flush=True)
    for name, h, payg in (() if a.no_tune else
                          (("H0+PAYG", 0, True), ("H1+PAYG", 1, True), ("H2+PAYG", 2, True), ("H2", 2, False))):
        t1 = time.time()
        nb, ib = tq.tune(n, n, 1, h, payg, None)
        wall = time.time() - t1
        g = es.get((nb, ib), factor_rate(n, nb, ib)[0])
        row["tuners"].append({"method": name, "nb": nb, "ib": ib, "gflops": g,
                              "pct_of_es": 100.0 * g / es[best], "optimum": (nb, ib) == best,
                              "wall_s": round(wall, 1)})
        tq.finalize()
    rows.append(row)
    print(json.dumps({"n": n, "es_best": row["es_best"],
                      "tuners": [(t["method"], t["nb"], t["ib"], round(t["pct_of_es"], 1)) for t in row["tuners"]]}),
          flush=True)
json.dump({"rows": rows}, open(a.out, "w"), indent=1)
