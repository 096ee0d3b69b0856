"""Summarise ncu evidence into small JSON files under profiles/.

    python tools/ncu_summary.py rep  <file.ncu-rep> <out.json> [--label ...]
    python tools/ncu_summary.py launches <launches.csv> <out.json>

`rep`: key counters of each profiled kernel (duration, DMMA pipe utilisation,
DRAM bytes, stall reasons, registers, occupancy).  `launches`: per-kernel
totals and shares from a `--metrics gpu__time_duration.sum` launch list.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
]


def rep_summary(path, label=None):
    if path.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` output brought back from the box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v / tot > 0.01}
        out.append(d)
    return {"source": path, "label": label, "kernels": out}


def launches_summary(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    grand = sum(tot.values()) or 1.0
    per = sorted(({"kernel": k, "launches": cnt[k], "total_ns": tot[k], "share": round(tot[k] / grand, 4)}
                  for k in tot), key=lambda d: -d["total_ns"])
    return {"source": path, "launches": sum(cnt.values()), "total_ns": grand, "per_kernel": per,
            "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised "
                    "launches; compare shares, not absolute times"}


if __name__ == "__main__":
    mode, src, dst = sys.argv[1], sys.argv[2], sys.argv[3]
    label = sys.argv[5] if len(sys.argv) > 5 and sys.argv[4] == "--label" else None
    res = rep_summary(src, label) if mode == "rep" else launches_summary(src)
    json.dump(res, open(dst, "w"), indent=1)
    print(dst)
