import ctypes, torch, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '.')
from paper_1102_5328_b200 import tileqr as tq
f = tq._lib.tileqr_debug_panel_prof; f.argtypes=[ctypes.c_void_p, ctypes.c_int]
out = (ctypes.c_ulonglong * 16)()
from tools.perf_scan import time_panel
for nb, ib in [(64,16),(128,32)]:
    for kind in ("tsqrt","geqrt"):
        f(out, 1)
        r = time_panel(nb, ib, reps=20, kind=kind)
        f(out, 1)
        reps = 21
        print(r, "cycles/launch [stage, factor, writeV, G, trailing, base, merge, Twrite, sync, Twrite2+sync]:", [round(out[i]/reps) for i in range(10)])
