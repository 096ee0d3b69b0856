import sys, os, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import perf_scan as ps
for nb, ib in [(160, 10), (160, 40), (128, 4), (128, 8)]:
    print(json.dumps(ps.time_ssrfb(nb, ib, reps=5)), flush=True)
