"""bench.py -- tile-QR FP64 throughput of libtileqr on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tileqr|reference]
                    [--workload 3|2|0|4] [--nb NB --ib IB]

One "step" = one whole tile QR factorization (tileqr_factor: layout in, every
DAG level of GEQRT/TSQRT/LARFB/SSRFB, layout out, T copy) of the workload's
matrix.  At N=1 every timed step factors its own pristine copy of the input,
staged in HBM before the timed region (800 MB each, > L2); when the copies
do not fit (and at N>1, and in the warm-up), the step first restores A from
one pristine device copy, inside the step.

Workload at N=1: BASELINE.json configs[3] (10000 x 10000, uniform(-0.5,0.5),
seed 4, NB/IB from the tuner's decision table) -- the largest single-GPU
tile-QR configuration (configs[1] is a kernel sweep, not a factorization).
At N>1 (torchrun): configs[4], 40000 x 40000 with tile columns 1D
block-cyclic over the ranks (tileqr_dist_factor; strong scaling).

Metric: GFLOP/s = (4/3 N^3) / t (unpadded N, IB extra
flops not credited), also as % of the measured B200 FP64 (DMMA) peak.
Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the
plain C tile QR in oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.0   # measured: tools/peak_fp64.cu, profiles/peak_fp64_r01.json (DMMA, sustained)
FP64_PEAK_SRC = "measured here: mma.sync.m8n8k4.f64 register loop on 148 SMs at 1965 MHz (profiles/peak_fp64_r01.json)"

WORKLOADS = {
    0: dict(name="qr256_nb64_ib16 (BASELINE configs[0])", M=256, N=256, seed=1, nb=64, ib=16),
    2: dict(name="qr2048 (BASELINE configs[2])", M=2048, N=2048, seed=3),
    3: dict(name="qr10000_tuned (BASELINE configs[3])", M=10000, N=10000, seed=4),
    4: dict(name="qr40000_dist (BASELINE configs[4])", M=40000, N=40000, seed=5),
    # not a BASELINE config: the tall-skinny case of SURVEY §8(f) f3 (reduction tree, BS tuned)
    5: dict(name="tall_skinny_131072x256_tree (SURVEY f3; not a BASELINE config)", M=131072, N=256, seed=6,
            nb=128, ib=16, tree=True),
}
TUNED = os.path.join(ROOT, "paper_1102_5328_b200", "tuned_table.json")


def qr_flops(m: int, n: int) -> float:
    if m >= n:
        return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
    return 2.0 * n * m * m - 2.0 * m ** 3 / 3.0


def tuned_pair(n: int, ngpus: int):
    """Nearest-point lookup in the decision table."""
    if os.path.exists(TUNED):
        tab = json.load(open(TUNED))["entries"]
        ns = sorted({e["n"] for e in tab})
        cs = sorted({e["ngpus"] for e in tab})
        nn = min(ns, key=lambda v: (abs(v - n), -v))
        cc = min(cs, key=lambda v: (abs(v - ngpus), -v))
        for e in tab:
            if e["n"] == nn and e["ngpus"] == cc:
                return e["nb"], e["ib"], "tuned_table.json (tileqr_tune, nearest point)"
    return 64, 16, "default (no tuned table)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for name, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_oracle_sample(m, n, nb, ib, seed, target_gflop=150.0, threads=None, full=False):
    """Time the CPU oracle (as it stands) on the workload: the whole
    factorization (full=True) or its first kmax panels (useful flops =
    flops(m, n) - flops of the untouched trailing part)."""
    import numpy as np  # noqa: F401
    import oracle
    import synth_inputs as si
    cores = threads or len(os.sched_getaffinity(0))
    npan = -(-min(m, n) // nb)
    kmax = npan if full else min(npan, max(1, int(target_gflop * 1e9 / (4.0 * m * n * nb))))
    a = si.uniform(m, n, seed)
    t0 = time.perf_counter()
    oracle.tileqr_factor(a, nb, ib, nthreads=cores, kmax=0 if kmax >= npan else kmax)
    dt = time.perf_counter() - t0
    done = kmax * nb
    fl = qr_flops(m, n) - (qr_flops(m - done, n - done) if done < min(m, n) else 0.0)
    what = (f"the whole {m}x{n} NB={nb} IB={ib} factorization" if kmax >= npan else
            f"first {kmax} of {npan} panels (k < {kmax}) of the {m}x{n} NB={nb} IB={ib} factorization")
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "cpu": _cpu_model(),
            "sample": f"{what}, oracle/tileqr_oracle.c with {cores} OpenMP thread(s); "
                      f"{fl / 1e9:.1f} useful GFLOP in {dt:.2f} s"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    wl = WORKLOADS[args.workload if args.workload is not None else (3 if world == 1 else 4)]
    m, n = wl["M"], wl["N"]
    nb, ib = (args.nb, args.ib) if args.nb else tuned_pair(n, world)[:2]
    if "nb" in wl and not args.nb:
        nb, ib = wl["nb"], wl["ib"]
    target = float(os.environ.get("TILEQR_REF_GFLOP", 60.0))
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        cpu_oracle_sample(min(m, 1024), min(n, 1024), nb, ib, wl["seed"], target_gflop=1.0)
    vals, samples = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_oracle_sample(m, n, nb, ib, wl["seed"], target_gflop=target)
        vals.append(r["value"])
        samples.append(r)
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    line = {"metric": "tile-QR FP64 GFLOP/s", "value": v, "unit": "GFLOP/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["name"], "M": m, "N": n, "NB": nb, "IB": ib},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": samples[0]["cores"],
                             "kind": "oracle", "sample": samples[0]["sample"]},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _traffic(key, nb, ib):
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        return json.load(open(prof)).get(key, {}).get(f"{nb}:{ib}")
    return None


def measure_dag(tq, m, n, nb, ib, step, step_ms, launch=None):
    """Roofline of the persistent dataflow kernel (the one launch that runs the
    whole DAG): algorithmic flops = the factorization's useful flops
     per launch / the kernel's average duration over the
    timed steps (`launch`: CUDA events around every launch, on its stream).
    Per-kind item busy times come from the device clock (globaltimer) in one
    traced step after the timed region."""
    tq.set_kernel_timing(True)
    step()
    import torch
    torch.cuda.synchronize()
    dag_ms, slots, _ = tq.kernel_times(m, n, nb, ib, "dag")   # slots = resident CTAs
    traced_ms = dag_ms
    if launch:
        dag_ms = launch[0]
    kinds = {"note": "dataflow kernel: per kind, items, busy ms summed over CTAs (inputs ready -> done), "
                     "one step after the timed region"}
    busy = {}
    for k in ("geqrt", "tsqrt", "larfb", "ssrfb"):
        tk, lk, nk = tq.kernel_times(m, n, nb, ib, k)
        busy[k] = tk
        kinds[k] = {"busy_ms_sum": round(tk, 3), "items": lk, "tasks": nk}
    tq.set_kernel_timing(False)
    s_tasks = kinds["ssrfb"]["tasks"]
    # SSRFB rate while running: its flops over its CTA-time, scaled to all slots
    kinds["ssrfb"]["tflops_while_running"] = round(
        s_tasks * 4.0 * nb ** 3 / (busy["ssrfb"] * 1e-3 / slots) / 1e12, 3) if busy["ssrfb"] else None
    kinds["cta_slots"] = slots
    kinds["slot_busy_frac"] = round(sum(busy.values()) / (slots * traced_ms), 4) if traced_ms else None
    kinds["traced_launch_ms"] = round(traced_ms, 4)
    flops = qr_flops(m, n)
    achieved = flops / (dag_ms * 1e-3) / 1e12 if dag_ms > 0 else 0.0
    roofline = {"kernel": "dag_kernel (persistent dataflow: GEQRT/TSQRT/LARFB/SSRFB items)",
                "bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": _traffic("dag", nb, ib),
                "flops_per_launch": flops, "avg_launch_ms": round(dag_ms, 4),
                "peak_source": FP64_PEAK_SRC, "share_of_step": round(dag_ms / step_ms, 4),
                "launches_timed": launch[1] if launch else 1,
                "measured": ("CUDA events around every dag_kernel launch of the timed steps (on the caller's "
                             "stream), averaged" if launch else
                             "CUDA events around the dag_kernel launch of one step after the timed region") +
                            "; flops = useful 4/3 N^3 (2MN^2-2N^3/3); "
                            "traffic = ncu dram read+write bytes of one launch (profiles/ncu_traffic.json)"}
    return roofline, kinds


def measure_levels(tq, m, n, nb, ib, step, step_ms):
    """Roofline of the SSRFB launches of the level-synchronous schedule."""
    import torch
    # SSRFB launch durations: CUDA events (event-record nodes in the captured graph,
    # on the update stream the kernels run on) in one measurement step right after
    # the timed region -- the nodes cost ~5% of a step, so the timed region has none
    tq.set_kernel_timing(True, kinds=("ssrfb",))
    step()
    torch.cuda.synchronize()
    tot, nl, nt = tq.kernel_times(m, n, nb, ib, "ssrfb")
    s = {"ms": round(tot, 3), "launches": nl, "tasks": nt}
    # per-kind breakdown from one more step with events around every launch
    tq.set_kernel_timing(True)
    step()
    torch.cuda.synchronize()
    kinds = {"note": "one extra step after the timed region, events around every launch"}
    for k in ("geqrt", "tsqrt", "larfb", "ssrfb"):
        tk, lk, nk = tq.kernel_times(m, n, nb, ib, k)
        kinds[k] = {"ms": round(tk, 3), "launches": lk, "tasks": nk}
    tq.set_kernel_timing(False)
    ssrfb_flops = s["tasks"] * 4.0 * nb ** 3          # useful 4 NB^3 per pair
    achieved = ssrfb_flops / (s["ms"] * 1e-3) / 1e12 if s["ms"] > 0 else 0.0
    per_task = _traffic("ssrfb_per_task", nb, ib)
    traffic = per_task * s["tasks"] / s["launches"] if (per_task and s["launches"]) else None
    roofline = {"kernel": "ssrfb (update kernel)", "bound": "tensor",
                "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": traffic,
                "flops_per_launch": ssrfb_flops / max(1, s["launches"]),
                "avg_launch_ms": round(s["ms"] / max(1, s["launches"]), 4),
                "peak_source": FP64_PEAK_SRC,
                "share_of_step": round(s["ms"] / step_ms, 4),
                "measured": "CUDA events around each SSRFB launch (graph event-record nodes on the update "
                            "stream) in the step right after the timed region; traffic = ncu dram bytes per "
                            "task (profiles/ncu_traffic.json) x this run's tasks per launch"}
    return roofline, kinds


def run_tileqr(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1102_5328_b200 import tileqr as tq

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1 or args.force_dist:
        return run_tileqr_dist(args, rank, world, local_rank)
    wl = WORKLOADS[args.workload if args.workload is not None else 3]
    m, n, seed = wl["M"], wl["N"], wl["seed"]
    if args.nb:
        nb, ib, src = args.nb, args.ib, "command line"
    elif "nb" in wl:
        nb, ib, src = wl["nb"], wl["ib"], ("fixed for the f3 tall-skinny line" if wl.get("tree")
                                           else "BASELINE configs[0]")
    else:
        nb, ib, src = tuned_pair(n, world)
    plan = tq.factor_plan(m, n, nb, ib)
    tree_bs = None
    if wl.get("tree"):  # domain size: tileqr_tune_tree ("p domains"), before any timing
        tree_bs, _ = tq.tune_tree(m, n, nb, ib)

    A0 = torch.empty((n, m), dtype=torch.float64, device=dev)   # column-major m x n
    tq.rng_uniform(A0, m, n, seed=seed)
    A = torch.empty_like(A0)
    T = torch.empty(max(1, tq.t_size(m, n, nb, ib)), dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    if tree_bs:
        T = torch.empty(max(1, tq.t_size_tree(m, n, nb, ib)), dtype=torch.float64, device=dev)

    def factor_once(buf):
        if tree_bs:
            tq.factor_tree(buf, m, n, nb, ib, tree_bs, T=T, info=info)
        else:
            tq.factor(buf, m, n, nb, ib, T=T, info=info)

    def step():
        A.copy_(A0)
        factor_once(A)

    tq.set_kernel_timing(False)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(info.item()) != 0:
        raise RuntimeError("tileqr_factor reported a non-finite input")

    # the timed steps factor their own pristine copies of A, staged in HBM
    # before the timed region (each > L2); if they do not fit, every step
    # restores A from the pristine copy inside the timed region instead
    free, _ = torch.cuda.mem_get_info(dev)
    staged = args.steps * A0.numel() * 8 < 0.5 * free
    bufs = [A0.clone() for _ in range(args.steps)] if staged else []
    sched = tq.factor_schedule(nb, ib)
    live = sched == "dag" and not tree_bs
    if live:  # CUDA events around every dataflow-kernel launch of the timed steps (no device-clock trace)
        tq.set_kernel_timing(True, kinds=(), launch_events=True)
        tq.kernel_times(m, n, nb, ib, "dag_launches")   # reset
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.steps):
            if staged:
                factor_once(bufs[i])
            else:
                step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launch = None
    if live:
        tot, cnt, _ = tq.kernel_times(m, n, nb, ib, "dag_launches")
        launch = (tot / cnt, cnt) if cnt else None
        tq.set_kernel_timing(False)
    del bufs
    flops = qr_flops(m, n)
    value = flops / (ms * 1e-3) / 1e9

    if tree_bs:
        sched = f"dag (reduction tree, BS={tree_bs})"
        ach = qr_flops(m, n) / (ms * 1e-3) / 1e12
        roofline = {"kernel": "dag_kernel (tree mode) + layout kernels: the whole step", "bound": "tensor",
                    "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": round(ach / FP64_PEAK_TFLOPS, 4), "traffic": None, "peak_source": FP64_PEAK_SRC,
                    "measured": "useful flops / the step's CUDA-event time (an upper bound on the kernel's "
                                "duration)"}
        kinds = None
    elif sched == "dag":
        roofline, kinds = measure_dag(tq, m, n, nb, ib, step, ms, launch)
    else:
        roofline, kinds = measure_levels(tq, m, n, nb, ib, step, ms)

    # e2e: same metric through the public host-buffer API (tileqr_factor_host):
    # pinned host A in, R/V and T back to pinned host buffers, the copies
    # overlapped with the factorization inside the call; every step moves the
    # whole input in and the whole result out inside the timed region
    e2e = None
    if not args.no_e2e and not tree_bs:
        hA = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        hA.copy_(A0)
        hR = torch.empty_like(hA, pin_memory=True)
        hT = torch.empty(T.numel(), dtype=torch.float64, pin_memory=True)
        e2e_steps = max(1, args.steps)

        def step_e2e():
            tq.factor_host(hA, m, n, nb, ib, hR=hR, hT=hT, info=info)

        step_e2e()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(e2e_steps):
            step_e2e()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1) / e2e_steps
        e2e = {"value": flops / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": hA.numel() * 8, "d2h_bytes_per_step": (hR.numel() + hT.numel()) * 8,
               "ms_per_step": ms_e2e, "steps": e2e_steps,
               "api": "tileqr_factor_host (copies overlapped with the dataflow kernel)"}

    cpu = None
    if not args.no_cpu_baseline and tree_bs:
        import oracle
        import synth_inputs as si
        a_h = si.uniform(m, n, seed)
        cores = len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        oracle.tileqr_factor_tree(a_h, nb, ib, tree_bs, nthreads=cores)
        dt = time.perf_counter() - t0
        cpu = {"value": qr_flops(m, n) / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
               "cpu": _cpu_model(), "sample": f"the whole {m}x{n} tree factorization (BS={tree_bs}), "
                                             f"oracle_tileqr_factor_tree with {cores} threads, {dt:.2f} s"}
    elif not args.no_cpu_baseline:
        # the whole factorization on every host core (about 30 s at 10000^2 on 16 cores), plus a
        # 1-thread sample of its first panel
        cpu = cpu_oracle_sample(m, n, nb, ib, seed, full=True)
        one = cpu_oracle_sample(m, n, nb, ib, seed, target_gflop=1.0, threads=1)
        cpu["one_thread"] = {"value": one["value"], "unit": one["unit"], "sample": one["sample"]}

    line = {"metric": "tile-QR FP64 GFLOP/s", "value": round(value, 2), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: i.i.d. uniform(-0.5,0.5), splitmix64 counter generator, seed {seed}",
            "config": {"workload": wl["name"], "M": m, "N": n, "NB": nb, "IB": ib, "nb_ib_source": src,
                       "BS": tree_bs,
                       "parallelism": "single GPU", "levels": plan["levels"], "schedule": sched,
                       "l2": (f"input {m * n * 8 / 1e6:.0f} MB > 126 MB L2; " +
                              ("each timed step factors its own pristine copy of A, staged in HBM before "
                               "the timed region" if staged else
                               "A restored from a pristine device copy at the start of every step "
                               "(inside the timed region)"))},
            "pct_fp64_peak": round(100 * value / (FP64_PEAK_TFLOPS * 1e3), 2),
            "roofline": roofline, "kernels": kinds, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": plan["launches"] * args.steps,
            "clocks": clk.summary(), "lib": tq.LIB_PATH}
    print(json.dumps(line), flush=True)


def run_tileqr_dist(args, rank, world, local_rank):
    """N>1: BASELINE configs[4] (40000^2) with tile columns 1D block-cyclic over
    the ranks; panel V/T broadcast with NCCL inside tileqr_dist_factor."""
    import torch
    import torch.distributed as dist
    from paper_1102_5328_b200 import tileqr as tq

    dev = torch.device("cuda", local_rank)
    if world == 1:  # --force-dist without torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=dev)
    wl = WORKLOADS[args.workload if args.workload is not None else 4]
    n, seed = wl["N"], wl["seed"]
    nb, ib, src = (args.nb, args.ib, "command line") if args.nb else tuned_pair(n, world)
    uid = [tq.dist_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    tq.dist_init(world, rank, uid[0], local_rank)
    mt = -(-n // nb)
    nloc = tq.dist_local_cols(n, nb)
    A0 = torch.empty(max(1, nloc * mt * nb * nb), dtype=torch.float64, device=dev)
    tq.dist_fill_uniform(n, n, nb, A0, seed)
    A = torch.empty_like(A0)
    T = torch.empty(max(1, nloc * mt * ib * nb), dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    dataflow = tq.factor_schedule(nb, ib) == "dag" and os.environ.get("TILEQR_DIST_SCHED") != "levels"

    def step():
        A.copy_(A0)
        tq.dist_factor(n, n, A, nb, ib, T, info)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)   # max over ranks
    ms = float(ms.item())
    bad = torch.tensor([int(info.item())], device=dev)
    dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    flops = qr_flops(n, n)
    value = flops / (ms * 1e-3) / 1e9
    if dataflow:  # zero-info, non-finite scan, the persistent dataflow kernel
        launches = 3
    else:
        launches = 2  # zero-info + non-finite scan
        for t in range(3 * mt - 2):
            panel, _, upd = tq.dist_plan_level(mt, world, rank, t)
            launches += len({q[0] for q in panel}) + len({q[0] for q in upd})
    verify = verify_dist(tq, dist, args, rank, world, dev, n, nb, ib, seed, A, T, mt, nloc, dataflow) \
        if args.verify else None
    if rank == 0:
        line = {"metric": "tile-QR FP64 GFLOP/s", "value": round(value, 2), "unit": "GFLOP/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": f"synthetic: i.i.d. uniform(-0.5,0.5), splitmix64 counter generator, seed {seed}",
                "config": {"workload": wl["name"], "M": n, "N": n, "NB": nb, "IB": ib, "nb_ib_source": src,
                           "parallelism": (f"1D block-cyclic tile columns over {world} GPUs; each rank runs its "
                                           "share of the DAG in the persistent dataflow kernel, packed panel "
                                           "V/T tiles pushed to the consumers over peer memory (NVLink)")
                           if dataflow else (f"1D block-cyclic tile columns over {world} GPUs, NCCL broadcast "
                                             "of panel V/T per DAG level"),
                           "schedule": "dataflow" if dataflow else "levels",
                           "l2": "per-rank input > 126 MB L2; A restored from a pristine device copy each step"},
                "pct_fp64_peak": round(100 * value / (world * FP64_PEAK_TFLOPS * 1e3), 2),
                "roofline": None, "cpu_baseline": None, "e2e": None, "nonfinite": int(bad.item()),
                "gpu_launches": launches * args.steps, "clocks": clk.summary(), "verify": verify}
        print(json.dumps(line), flush=True)
    tq.dist_finalize()
    dist.destroy_process_group()


def verify_dist(tq, dist, args, rank, world, dev, n, nb, ib, seed, A, T, mt, nloc, dataflow=True):
    """P>1 verification: every rank's factored tile columns and T tiles are
    sent to rank 0, which factors the same matrix on its own GPU with
    tileqr_factor and compares BITWISE (the distributed result must be
    identical for the same (NB, IB))."""
    import torch
    torch.cuda.synchronize()
    ok = True
    if rank == 0:
        ref = torch.empty((n, n), dtype=torch.float64, device=dev)
        tq.rng_uniform(ref, n, n, seed=seed)
        Tref, _ = tq.factor(ref, n, n, nb, ib)
        torch.cuda.synchronize()
        refm = ref.t()   # the factored matrix (column-major storage)
        nt = mt
        for r in range(world):
            cols = list(range(r, nt, world))
            if not cols:
                continue
            if r == 0:
                buf, tb = A, T
            else:
                buf = torch.empty(len(cols) * mt * nb * nb, dtype=torch.float64, device=dev)
                tb = torch.empty(len(cols) * mt * ib * nb, dtype=torch.float64, device=dev)
                dist.recv(buf, src=r)
                dist.recv(tb, src=r)
            v = buf.view(len(cols), mt, nb, nb)
            tv = tb.view(len(cols), mt, nb * ib)
            for j, c in enumerate(cols):
                for m in range(mt):
                    i0, i1 = m * nb, min(n, (m + 1) * nb)
                    j0, j1 = c * nb, min(n, (c + 1) * nb)
                    got = v[j, m].t()[: i1 - i0, : j1 - j0]
                    ok = ok and bool(torch.equal(got, refm[i0:i1, j0:j1]))
                    if m >= c:
                        o = (m + c * mt) * ib * nb
                        ok = ok and bool(torch.equal(tv[j, m], Tref[o:o + ib * nb]))
        del ref, Tref
    elif nloc > 0:
        dist.send(A, dst=0)
        dist.send(T, dst=0)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, src=0)
    if not dataflow:  # the level-synchronous baseline keeps no reflector slots to apply Q^T from
        return {"bitwise_equal_to_single_gpu": bool(flag.item()), "residual_ratio": None,
                "how": "all ranks' tile columns and T gathered on rank 0 and compared with tileqr_factor of the "
                       "same matrix on rank 0's GPU"}
    # residual without the single GPU: every rank applies Q^T (its packed reflector slots) to its
    # pristine columns; ||Q^T A - R||^2 and ||A||^2 summed over ranks (all-reduce)
    B = torch.empty(max(1, nloc * mt * nb * nb), dtype=torch.float64, device=dev)
    tq.dist_fill_uniform(n, n, nb, B, seed)
    a2 = torch.sum(B ** 2) if nloc else torch.zeros((), dtype=torch.float64, device=dev)
    if nloc:
        tq.dist_apply_qt_local(n, n, B, nb, ib)
        r2 = tq.dist_residual_terms(n, n, nb, A, B, rank, world)
    else:
        r2 = torch.zeros((), dtype=torch.float64, device=dev)
    tot = torch.stack([r2, a2]).reshape(2)
    dist.all_reduce(tot)
    npad = sum(1 for j in range(n, mt * nb) if j < mt * nb)
    res = float(torch.sqrt(tot[0]) / (torch.sqrt(tot[1] - npad) * n * 2.0 ** -52))
    return {"bitwise_equal_to_single_gpu": bool(flag.item()),
            "residual_ratio": res, "residual_ok": res < 10,
            "how": "all ranks' tile columns and T gathered on rank 0 and compared with tileqr_factor of the same "
                   "matrix on rank 0's GPU; residual ||Q^T A - R||_F / (||A||_F N eps) from every rank's own "
                   "reflector slots (tileqr_dist_apply_qt_local), sums of squares all-reduced"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tileqr", choices=["tileqr", "reference"])
    ap.add_argument("--workload", type=int, default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--nb", type=int, default=None)
    ap.add_argument("--ib", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verify", action="store_true", help="N>1: bitwise check against a 1-GPU tileqr_factor")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU path even at world size 1 (exercises its code on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "tileqr":
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_tileqr(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
