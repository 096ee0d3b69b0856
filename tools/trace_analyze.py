"""Analyse a dataflow-kernel trace (tools/trace_factor.py output): SM
utilisation over time, claim->ready wait per kind, head/tail idle.

    python tools/trace_analyze.py gpurun_out/trace.json [--nsm 148] [--bins 20]
"""
import argparse
import collections
import json

ap = argparse.ArgumentParser()
ap.add_argument("path")
ap.add_argument("--nsm", type=int, default=148)
ap.add_argument("--bins", type=int, default=20)
a = ap.parse_args()
d = json.load(open(a.path))
recs = d["recs"]  # (start_ms, end_ms, kind, level, claim_ns)
span = max(r[1] for r in recs)
print(f"items {len(recs)}  span {span:.3f} ms  (NB={d['nb']} IB={d['ib']})")
busy = collections.defaultdict(float)
wait = collections.defaultdict(float)
cnt = collections.Counter()
for s, e, k, lv, c in recs:
    busy[k] += e - s
    wait[k] += s - c * 1e-6
    cnt[k] += 1
tot_busy = sum(busy.values())
print(f"SM busy fraction {tot_busy / (a.nsm * span):.3f}; dependency wait (claim->ready) "
      f"{sum(wait.values()) / (a.nsm * span):.3f} of SM time")
for k in busy:
    print(f"  {k:6s} n={cnt[k]:7d} busy {busy[k]:9.2f} ms ({1e3 * busy[k] / cnt[k]:7.2f} us/item) "
          f"wait {wait[k]:8.2f} ms ({1e3 * wait[k] / cnt[k]:7.2f} us/item)")
# utilisation over time
B = a.bins
bb = [0.0] * B
wb = [0.0] * B
w = span / B
for s, e, k, lv, c in recs:
    for arr, t0, t1 in ((bb, s, e), (wb, c * 1e-6, s)):
        i0, i1 = int(t0 / w), min(B - 1, int(t1 / w))
        for i in range(i0, i1 + 1):
            lo, hi = max(t0, i * w), min(t1, (i + 1) * w)
            if hi > lo:
                arr[i] += hi - lo
print("time bins: busy SMs / waiting SMs")
for i in range(B):
    print(f"  {i * w:7.2f}-{(i + 1) * w:7.2f} ms: busy {bb[i] / w:6.1f}  waiting {wb[i] / w:6.1f}")
