"""Phase cycles of the fast GEQRT/TSQRT kernel (needs the diagnostic build:
TILEQR_BUILD_VARIANT=prof python -m paper_1102_5328_b200.build; run with
TILEQR_LIB=paper_1102_5328_b200/libtileqr_prof.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_5328_b200 import tileqr as tq  # noqa: E402
from tools.perf_scan import time_panel  # noqa: E402

f = tq._lib.tileqr_debug_panel_prof
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = (ctypes.c_ulonglong * 16)()
names = {0: "stage", 1: "factor", 2: "writeV", 5: "gram", 6: "Tdiag", 7: "Tmerge", 3: "Twrite+pack", 4: "trailing"}
for nb, ib in [(128, 16), (64, 16), (64, 32)]:
    for kind in ("tsqrt", "geqrt"):
        f(out, 1)
        r = time_panel(nb, ib, reps=20, kind=kind)
        f(out, 1)
        reps = 21
        off = 0 if kind == "tsqrt" else 8  # GEQRT phases are counted at index 8 + k
        ph = {v: round(out[off + k] / reps) for k, v in names.items()}
        ph["total"] = sum(ph.values())
        print(r, ph, flush=True)
