"""Build libtileqr.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1102_5328_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# TILEQR_BUILD_VARIANT=prof builds a diagnostic copy (-DTILEQR_PANEL_PROF) as
# libtileqr_prof.so (loaded when TILEQR_LIB points at it); the default build is
# the product library
VARIANT = os.environ.get("TILEQR_BUILD_VARIANT", "")
BUILD = os.path.join(HERE, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(HERE, "libtileqr" + (f"_{VARIANT}" if VARIANT else "") + ".so")
EXTRA = (["-DTILEQR_PANEL_PROF"] if VARIANT == "prof" else []) + os.environ.get("TILEQR_EXTRA_FLAGS", "").split()
SOURCES = ["kernels_layout.cu", "kernels_panel.cu", "kernels_panel_fast.cu", "kernels_update.cu",
           "api.cu", "tune.cu", "dist.cu", "table.cu", "dist_dag.cu", "tree.cu"] + [f"update_nb{nb}.cu" for nb in (32, 64, 96, 128, 160, 192, 224, 256)]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def _nccl_dirs():
    try:
        import nvidia.nccl as n  # torch's NCCL (the one torch.distributed uses)
        root = list(n.__path__)[0]
        return os.path.join(root, "include"), os.path.join(root, "lib")
    except Exception:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = _nccl_dirs()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "tileqr.h"))
    hdr_mtime = max(os.path.getmtime(h) for h in headers)
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_mtime):
            jobs.append([NVCC, *ARCH, *FLAGS, *EXTRA, "-I", inc, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        log = os.path.join(BUILD, os.path.basename(cmd[-1]) + ".log")
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        return r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for r in ex.map(run, jobs):
            if verbose:
                sys.stdout.write(r.stderr)
    if jobs or force or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L", libdir, "-l:libnccl.so.2",
               "-Xlinker", "-rpath=" + libdir, "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
