"""Hot regions of an ncu source-page CSV (SASS view): samples per chunk of
consecutive instructions with the dominant stall reasons and opcodes.
    python tools/sass_hot.py file.source.csv.gz [chunk]"""
import collections
import csv
import gzip
import io
import sys

path = sys.argv[1]
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ix[S]] or 0) for r in data)
print("instructions", len(data), "samples", tot)
agg = collections.Counter()
for r in data:
    for h in stalls:
        agg[h[6:]] += int(r[ix[h]] or 0)
print("stalls:", ", ".join(f"{k} {v / tot:.1%}" for k, v in agg.most_common(8)))
for i0 in range(0, len(data), chunk):
    blk = data[i0:i0 + chunk]
    s = sum(int(r[ix[S]] or 0) for r in blk)
    if s < tot * 0.01:
        continue
    st = collections.Counter()
    ops = collections.Counter()
    for r in blk:
        for h in stalls:
            st[h[6:]] += int(r[ix[h]] or 0)
        op = r[1].strip().split()[0]
        if op.startswith("@"):
            op = r[1].strip().split()[1]
        ops[op.split(".")[0]] += 1
    print(f"[{i0:5d}-{i0 + len(blk) - 1:5d}] {s / tot:6.1%}  "
          + ", ".join(f"{k} {v / s:.0%}" for k, v in st.most_common(3)) + "  | "
          + " ".join(f"{k}:{v}" for k, v in ops.most_common(5)))
