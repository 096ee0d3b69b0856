"""Per-SM analysis of a dataflow-kernel trace (tools/trace_factor.py output,
claim field tagged by dag.cuh: SM id | fast hand-off << 8 | C2 staged << 9).

    python tools/trace_sm.py gpurun_out/trace.json

Reports: how often the fast hand-off and the C2 staging happened; SSRFB item
durations by what the SM's other CTA was doing meanwhile (update item, panel
item, nothing); the per-CTA gaps between consecutive items; the SM time split
into both-update / update+panel / update alone / other.
"""
import collections
import json
import sys

d = json.load(open(sys.argv[1]))
recs = d["recs"]
nb = d["nb"]
per_sm = collections.defaultdict(list)
flags = collections.Counter()
for s, e, k, lv, c in recs:
    tag = c & 0x3FF
    sm, fast, staged = tag & 0xFF, (tag >> 8) & 1, (tag >> 9) & 1
    per_sm[sm].append((s, e, k, fast, staged))
    if k == "ssrfb":
        flags["ssrfb"] += 1
        flags["fast"] += fast
        flags["staged"] += staged
print(f"items {len(recs)} on {len(per_sm)} SMs; SSRFB {flags['ssrfb']}: fast hand-off {flags['fast'] / flags['ssrfb']:.3f}, "
      f"C2 staged {flags['staged'] / flags['ssrfb']:.3f}")
span = max(r[1] for r in recs)
upd = ("ssrfb", "larfb")
cat = collections.defaultdict(list)  # SSRFB durations by neighbour state
gaps = collections.defaultdict(list)
tsplit = collections.Counter()
for sm, its in per_sm.items():
    its.sort()
    # two CTAs per SM: split into two non-overlapping chains
    chains = [[], []]
    for it in its:
        ends = [ch[-1][1] if ch else -1.0 for ch in chains]
        cand = [i for i in range(2) if ends[i] <= it[0] + 1e-6]
        i = max(cand, key=lambda j: ends[j]) if cand else min(range(2), key=lambda j: ends[j])
        chains[i].append(it)
    for ci, ch in enumerate(chains):
        other = chains[1 - ci]
        for a, b in zip(ch, ch[1:]):
            gaps[(a[2] in upd, b[2] in upd, b[3])].append(b[0] - a[1])
        j = 0
        for it in ch:
            if it[2] != "ssrfb":
                continue
            s, e = it[0], it[1]
            ov = collections.Counter()
            for o in other:
                lo, hi = max(s, o[0]), min(e, o[1])
                if hi > lo:
                    ov["upd" if o[2] in upd else "panel"] += hi - lo
            dur = e - s
            fu = ov["upd"] / dur
            fp = ov["panel"] / dur
            key = "co-update>=0.95" if fu >= 0.95 else ("panel>=0.5" if fp >= 0.5 else
                   ("idle>=0.5" if 1 - fu - fp >= 0.5 else "mixed"))
            cat[(key, it[3])].append(dur)
    # SM time split: sweep over the two chains' boundaries
    ev = sorted({0.0, span} | {x for ch in chains for it in ch for x in it[:2]})
    idx = [0, 0]
    for t0, t1 in zip(ev, ev[1:]):
        mid = 0.5 * (t0 + t1)
        st = []
        for ci, ch in enumerate(chains):
            while idx[ci] < len(ch) and ch[idx[ci]][1] <= mid:
                idx[ci] += 1
            it = ch[idx[ci]] if idx[ci] < len(ch) else None
            st.append("-" if it is None or it[0] > mid else ("U" if it[2] in upd else "P"))
        tsplit["".join(sorted(st))] += t1 - t0
dur = collections.defaultdict(list)
for sm, its in per_sm.items():
    for it in its:
        if it[2] == "ssrfb":
            dur[it[4]].append(1e3 * (it[1] - it[0]))
for k in sorted(dur):
    v = sorted(dur[k])
    q = lambda f: v[min(len(v) - 1, int(f * len(v)))]
    print(f"SSRFB duration (us), C2 staged={k}: n={len(v)} p10 {q(0.1):.1f} p50 {q(0.5):.1f} p90 {q(0.9):.1f} "
          f"p99 {q(0.99):.1f} mean {sum(v) / len(v):.2f}")
print("SSRFB item duration (us) by the SM's other CTA [fast hand-off flag]:")
for k in sorted(cat):
    v = sorted(cat[k])
    print(f"  {k[0]:16s} fast={k[1]}  n={len(v):6d}  mean {1e3 * sum(v) / len(v):7.2f}  median {1e3 * v[len(v) // 2]:7.2f}")
print("gaps between consecutive items of one CTA (us) [prev update, next update, next fast]:")
for k in sorted(gaps):
    v = sorted(gaps[k])
    print(f"  {str(k):22s} n={len(v):6d}  mean {1e3 * sum(v) / len(v):7.2f}  median {1e3 * v[len(v) // 2]:7.2f}")
tot = sum(tsplit.values())
print("SM time split (U update item, P panel item, - nothing), both CTAs:")
for k, v in tsplit.most_common():
    print(f"  {k}: {v / tot:.3f}")
