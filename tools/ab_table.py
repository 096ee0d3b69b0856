"""Summarise an A/B log of perf_scan lines grouped by '== variant' headers:
    python tools/ab_table.py gpurun_out/r02z/ab.log"""
import collections
import json
import sys

cur, d, order = None, collections.defaultdict(list), []
for line in open(sys.argv[1]):
    line = line.strip()
    if line.startswith("=="):
        cur = line[3:]
        if cur not in order:
            order.append(cur)
        continue
    if not line.startswith("{"):
        continue
    r = json.loads(line)
    key = (r.get("kind", "factor"), r.get("n") or 0, r["nb"], r["ib"])
    d[(key, cur)].append(r.get("ms", r.get("us")))
for k in sorted(set(k for k, _ in d)):
    meds = {v: sorted(d[(k, v)])[len(d[(k, v)]) // 2] for v in order if d[(k, v)]}
    base = meds.get(order[-1])
    print(k, "  ".join(f"{v}={m:g}" for v, m in meds.items()),
          f"  ({(meds[order[0]] / base - 1) * 100:+.1f} %)" if base else "")
