"""Step 1 with and without L2 flushing:
runs tileqr_tune twice at one N and compares the Step-1 rates, the
pre-selected candidates and the final pick.

    python tools/step1_flush.py [--n 10000] [--out gpurun_out/step1_flush.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--out", default="gpurun_out/step1_flush.json")
a = ap.parse_args()
res = {}
for mode in ("no_flush", "flush"):
    os.environ["TILEQR_TUNE_FLUSH"] = "1" if mode == "flush" else "0"
    path = f"gpurun_out/tune_{mode}_{a.n}.json"
    nb, ib = tq.tune(a.n, a.n, 1, 2, True, path)
    d = json.load(open(path))
    res[mode] = {"pick": [nb, ib], "candidates": d["candidates"],
                 "step1": {f"{p['nb']}:{p['ib']}": round(p["gflops"], 1) for p in d["step1"]}}
common = sorted(set(res["flush"]["step1"]) & set(res["no_flush"]["step1"]))
ratio = {k: round(res["flush"]["step1"][k] / res["no_flush"]["step1"][k], 4) for k in common}
out = {"n": a.n, "no_flush": res["no_flush"], "flush": res["flush"], "flush_over_no_flush": ratio,
       "same_candidates": [(c["nb"], c["ib"]) for c in res["flush"]["candidates"]] ==
                          [(c["nb"], c["ib"]) for c in res["no_flush"]["candidates"]],
       "same_pick": res["flush"]["pick"] == res["no_flush"]["pick"]}
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps({k: out[k] for k in ("n", "same_candidates", "same_pick")}),
      "ratio min/max", min(ratio.values()), max(ratio.values()))
