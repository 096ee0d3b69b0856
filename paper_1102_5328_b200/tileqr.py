"""Thin ctypes binding of libtileqr.so (include/tileqr.h).

Argument marshalling only: every step of the factorization runs in the CUDA
kernels of libtileqr.so.  PyTorch supplies device memory, streams and process
groups.  There is no CPU fallback: if the library is missing, importing this
module raises.

Names follow the C ABI (tileqr_factor -> factor, ...).  Matrices are FP64
column-major; torch tensors are passed as Fortran-ordered views, i.e. a
torch tensor ``A`` of shape (N, M) row-major IS the column-major M x N matrix
``A.T``.  The helpers :func:`colmajor_empty` / :func:`to_colmajor` /
:func:`from_colmajor` do that bookkeeping.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("TILEQR_LIB") or os.path.join(_HERE, "libtileqr.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libtileqr.so not built ({_LIB_PATH}); run `python -m paper_1102_5328_b200.build`")

_lib = ctypes.CDLL(_LIB_PATH)

_i, _i64, _u64, _c, _d = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_char, ctypes.c_double
_p, _sz = ctypes.c_void_p, ctypes.c_size_t
_PI = ctypes.POINTER(ctypes.c_int)
_PD = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "tileqr_version": ([], ctypes.c_char_p),
    "tileqr_last_error": ([], ctypes.c_char_p),
    "tileqr_t_size": ([_i64, _i64, _i, _i, ctypes.POINTER(_sz)], _i),
    "tileqr_lookup": ([_i64, _i64, _i, _PI, _PI], _i),
    "tileqr_factor": ([_i64, _i64, _p, _i64, _i, _i, _p, _p, _p], _i),
    "tileqr_factor_host": ([_i64, _i64, _p, _i64, _i, _i, _p, _i64, _p, _p, _p], _i),
    "tileqr_apply_qt": ([_c, _i64, _i64, _i64, _p, _i64, _p, _i, _i, _p, _i64, _p], _i),
    "tileqr_geqrt_batched": ([_i, _i, _i, _p, _p, _p], _i),
    "tileqr_tsqrt_batched": ([_i, _i, _i, _p, _p, _p, _p], _i),
    "tileqr_larfb_batched": ([_c, _i, _i, _i, _p, _p, _p, _i, _p], _i),
    "tileqr_ssrfb_batched": ([_c, _i, _i, _i, _p, _p, _p, _p, _i, _p], _i),
    "tileqr_packed_size": ([_i, _i, ctypes.POINTER(_sz)], _i),
    "tileqr_pack_batched": ([_i, _i, _i, _i, _p, _p, _p, _p], _i),
    "tileqr_update_packed_batched": ([_i, _i, _i, _i, _p, _p, _p, _p], _i),
    "tileqr_tune": ([_i64, _i64, _i, _i, _i, _PI, _PI, ctypes.c_char_p], _i),
    "tileqr_preselect": ([_i, _PI, _PI, _PD, _i, _i, _PI, _PI, _PD, _PI], _i),
    "tileqr_preselect_tie": ([_i, _PI, _PI, _PD, _i, _i, ctypes.c_double, _PI, _PI, _PD, _PI], _i),
    "tileqr_payg_prune": ([_i, _PI, _PD, _PI], _i),
    "tileqr_num_levels": ([_i64, _i64, ctypes.POINTER(_i64)], _i),
    "tileqr_dist_init": ([_i, _i, _p, _i], _i),
    "tileqr_dist_unique_id": ([_p], _i),
    "tileqr_dist_local_cols": ([_i64, _i, _PI], _i),
    "tileqr_dist_fill_uniform": ([_i64, _i64, _i, _p, _u64, _p], _i),
    "tileqr_dist_factor": ([_i64, _i64, _p, _i, _i, _p, _p, _p], _i),
    "tileqr_dist_emulate": ([_i, _i64, _i64, _p, _i, _i, _p, _p, _p], _i),
    "tileqr_dist_apply_qt_local": ([_i64, _i64, _p, _i, _i, _p], _i),
    "tileqr_dist_plan_items": ([_i64, _i64, _i, _i, _i, _i, _i, _i, ctypes.POINTER(_i64), _i64,
                                ctypes.POINTER(_i64)], _i),
    "tileqr_dist_plan_level": ([_i64, _i, _i, _i64, ctypes.POINTER(_i64), _i64, ctypes.POINTER(_i64)], _i),
    "tileqr_dist_finalize": ([], None),
    "tileqr_rng_uniform": ([_i64, _i64, _p, _i64, _u64, _u64, _p], _i),
    "tileqr_ssrfb_impl": ([_i, _i], ctypes.c_char_p),
    "tileqr_factor_schedule": ([_i, _i], ctypes.c_char_p),
    "tileqr_factor_plan": ([_i64, _i64, _i, _i, ctypes.POINTER(_i64)], _i),
    "tileqr_set_kernel_timing": ([_i], None),
    "tileqr_kernel_times": ([_i64, _i64, _i, _i, _i, _PD, ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _i),
    "tileqr_kernel_trace": ([_i64, _i64, _i, _i, _i64, _PD, _PD, _PI, ctypes.POINTER(_i64),
                             ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _i),
    "tileqr_finalize": ([], None),
    "tileqr_factor_tree": ([_i64, _i64, _p, _i64, _i, _i, _i64, _p, _p, _p], _i),
    "tileqr_t_size_tree": ([_i64, _i64, _i, _i, ctypes.POINTER(_sz)], _i),
    "tileqr_apply_qt_tree": ([_c, _i64, _i64, _i64, _p, _i64, _p, _i, _i, _i64, _p, _i64, _p], _i),
    "tileqr_ttqrt_batched": ([_i, _i, _i, _p, _p, _p, _p], _i),
    "tileqr_tree_finalize": ([], None),
    "tileqr_tune_tree": ([_i64, _i64, _i, _i, ctypes.POINTER(_i64), _PD, ctypes.c_char_p], _i),
    "tileqr_tree_plan_items": ([_i64, _i64, _i, _i, _i64, _i, _i, ctypes.POINTER(_i64), _i64,
                                ctypes.POINTER(_i64)], _i),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
LIB_PATH = _LIB_PATH


class TileQRError(RuntimeError):
    pass


def _check(rc: int, fn: str):
    if rc != 0:
        msg = _lib.tileqr_last_error().decode()
        raise TileQRError(f"{fn} returned {rc}: {msg}")


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def version() -> str:
    return _lib.tileqr_version().decode()


def last_error() -> str:
    return _lib.tileqr_last_error().decode()


def t_size(m: int, n: int, nb: int, ib: int) -> int:
    out = _sz()
    _check(_lib.tileqr_t_size(m, n, nb, ib, ctypes.byref(out)), "tileqr_t_size")
    return out.value


def lookup(m: int, n: int, ngpus: int = 1):
    """(nb, ib, from_table): the installed decision table's pair for this shape
    (built-in default and from_table False when no table is installed)."""
    nb, ib = ctypes.c_int(), ctypes.c_int()
    rc = _lib.tileqr_lookup(m, n, ngpus, ctypes.byref(nb), ctypes.byref(ib))
    if rc not in (0, 4):
        _check(rc, "tileqr_lookup")
    return nb.value, ib.value, rc == 0


def num_levels(mt: int, nt: int) -> int:
    out = _i64()
    _check(_lib.tileqr_num_levels(mt, nt, ctypes.byref(out)), "tileqr_num_levels")
    return out.value


def ssrfb_impl(nb: int, ib: int) -> str:
    return _lib.tileqr_ssrfb_impl(nb, ib).decode()


# ---------------------------------------------------------------------------
# column-major helpers
# ---------------------------------------------------------------------------
def colmajor_empty(m: int, n: int, device="cuda") -> torch.Tensor:
    """Storage of a column-major m x n FP64 matrix: a (n, m) row-major tensor."""
    return torch.empty((n, m), dtype=torch.float64, device=device)


def to_colmajor(x, device="cuda") -> torch.Tensor:
    """numpy/torch m x n matrix -> device storage (n, m) holding it column-major."""
    t = torch.as_tensor(x, dtype=torch.float64)
    return t.t().contiguous().to(device)


def from_colmajor(buf: torch.Tensor):
    """device storage (n, m) -> numpy m x n matrix (Fortran order)."""
    import numpy as np
    return np.asfortranarray(buf.detach().cpu().numpy().T)


# ---------------------------------------------------------------------------
# entry points
# ---------------------------------------------------------------------------
def factor(A: torch.Tensor, m: int, n: int, nb: int, ib: int, T: torch.Tensor | None = None,
           info: torch.Tensor | None = None, lda: int | None = None, stream=None):
    """tileqr_factor on the column-major m x n matrix stored in A (in place).

    Returns (T, info) device tensors."""
    assert A.dtype == torch.float64 and A.is_cuda and A.is_contiguous()
    if T is None:
        T = torch.empty(max(1, t_size(m, n, nb, ib)), dtype=torch.float64, device=A.device)
    if info is None:
        info = torch.zeros(1, dtype=torch.int32, device=A.device)
    rc = _lib.tileqr_factor(m, n, A.data_ptr(), lda if lda is not None else max(1, m), nb, ib,
                            T.data_ptr(), info.data_ptr(), _stream(stream))
    _check(rc, "tileqr_factor")
    return T, info


def factor_host(hA: torch.Tensor, m: int, n: int, nb: int, ib: int, hR: torch.Tensor | None = None,
                hT: torch.Tensor | None = None, info: torch.Tensor | None = None, lda: int | None = None,
                ldr: int | None = None, stream=None):
    """tileqr_factor_host: the column-major m x n matrix in HOST tensor hA
    (pin it for overlap) -> R/V in host tensor hR (default: in place in hA) and
    T in host tensor hT.  Stream-ordered; returns (hR, hT, info)."""
    assert hA.dtype == torch.float64 and not hA.is_cuda and hA.is_contiguous()
    if hR is None:
        hR = hA
    own = hT is None or info is None
    if hT is None:
        hT = torch.empty(max(1, t_size(m, n, nb, ib)), dtype=torch.float64, pin_memory=hA.is_pinned())
    if info is None:
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = _stream(stream)
    rc = _lib.tileqr_factor_host(m, n, hA.data_ptr(), lda if lda is not None else max(1, m), nb, ib,
                                 hR.data_ptr(), ldr if ldr is not None else max(1, m), hT.data_ptr(),
                                 info.data_ptr(), s)
    _check(rc, "tileqr_factor_host")
    if own:
        # buffers this wrapper allocated are still being written by queued
        # copies: finish the call before handing them out, so dropping them
        # cannot return a block to torch's allocator under an in-flight DMA
        torch.cuda.ExternalStream(s).synchronize() if s else torch.cuda.synchronize()
    return hR, hT, info


def apply_qt(trans: str, A: torch.Tensor, m: int, k: int, T: torch.Tensor, nb: int, ib: int,
             B: torch.Tensor, nrhs: int, lda: int | None = None, ldb: int | None = None,
             stream=None):
    """B <- Q^T B ('T') or Q B ('N') in place (B column-major m x nrhs)."""
    rc = _lib.tileqr_apply_qt(trans.encode(), m, nrhs, k, A.data_ptr(),
                              lda if lda is not None else max(1, m), T.data_ptr(), nb, ib,
                              B.data_ptr(), ldb if ldb is not None else max(1, m), _stream(stream))
    _check(rc, "tileqr_apply_qt")
    return B


def _ptrs(tiles) -> torch.Tensor:
    return torch.tensor([t.data_ptr() for t in tiles], dtype=torch.int64, device="cuda")


def geqrt_batched(nb: int, ib: int, A_ptrs: torch.Tensor, T_ptrs: torch.Tensor, stream=None):
    _check(_lib.tileqr_geqrt_batched(nb, ib, A_ptrs.numel(), A_ptrs.data_ptr(), T_ptrs.data_ptr(),
                                     _stream(stream)), "tileqr_geqrt_batched")


def tsqrt_batched(nb: int, ib: int, R_ptrs, A2_ptrs, T_ptrs, stream=None):
    _check(_lib.tileqr_tsqrt_batched(nb, ib, R_ptrs.numel(), R_ptrs.data_ptr(), A2_ptrs.data_ptr(),
                                     T_ptrs.data_ptr(), _stream(stream)), "tileqr_tsqrt_batched")


def larfb_batched(trans: str, nb: int, ib: int, V_ptrs, T_ptrs, C_ptrs, ncols: int, stream=None):
    _check(_lib.tileqr_larfb_batched(trans.encode(), nb, ib, V_ptrs.numel(), V_ptrs.data_ptr(),
                                     T_ptrs.data_ptr(), C_ptrs.data_ptr(), ncols, _stream(stream)),
           "tileqr_larfb_batched")


def ssrfb_batched(trans: str, nb: int, ib: int, V2_ptrs, T_ptrs, C1_ptrs, C2_ptrs, ncols: int,
                  stream=None):
    _check(_lib.tileqr_ssrfb_batched(trans.encode(), nb, ib, V2_ptrs.numel(), V2_ptrs.data_ptr(),
                                     T_ptrs.data_ptr(), C1_ptrs.data_ptr(), C2_ptrs.data_ptr(),
                                     ncols, _stream(stream)), "tileqr_ssrfb_batched")


def packed_size(nb: int, ib: int) -> int:
    out = _sz()
    _check(_lib.tileqr_packed_size(nb, ib, ctypes.byref(out)), "tileqr_packed_size")
    return out.value


def pack_batched(larfb: bool, nb: int, ib: int, V_ptrs, T_ptrs, Pk_ptrs, stream=None):
    _check(_lib.tileqr_pack_batched(int(larfb), nb, ib, V_ptrs.numel(), V_ptrs.data_ptr(), T_ptrs.data_ptr(),
                                    Pk_ptrs.data_ptr(), _stream(stream)), "tileqr_pack_batched")


def update_packed_batched(larfb: bool, nb: int, ib: int, Pk_ptrs, C1_ptrs, C2_ptrs, stream=None):
    _check(_lib.tileqr_update_packed_batched(int(larfb), nb, ib, Pk_ptrs.numel(), Pk_ptrs.data_ptr(),
                                             C1_ptrs.data_ptr() if C1_ptrs is not None else None,
                                             C2_ptrs.data_ptr(), _stream(stream)),
           "tileqr_update_packed_batched")


def rng_uniform(A: torch.Tensor, m: int, n: int, seed: int, offset: int = 0, lda: int | None = None,
                stream=None):
    _check(_lib.tileqr_rng_uniform(m, n, A.data_ptr(), lda if lda is not None else max(1, m), seed,
                                   offset, _stream(stream)), "tileqr_rng_uniform")
    return A


def tune(m: int, n: int, ngpus: int = 1, heuristic: int = 2, payg: bool = True,
         report_json_path: str | None = None):
    nb, ib = ctypes.c_int(), ctypes.c_int()
    rc = _lib.tileqr_tune(m, n, ngpus, heuristic, int(payg), ctypes.byref(nb), ctypes.byref(ib),
                          report_json_path.encode() if report_json_path else None)
    _check(rc, "tileqr_tune")
    return nb.value, ib.value


def preselect(samples, heuristic: int = 2, cap: int = 8, tie_rel: float = 0.0):
    """Host-only Step-1 pre-selection; samples [(nb, ib, gflops)]; tie_rel: Property-1 tie width."""
    n = len(samples)
    nb = (ctypes.c_int * n)(*[s[0] for s in samples])
    ib = (ctypes.c_int * n)(*[s[1] for s in samples])
    g = (ctypes.c_double * n)(*[s[2] for s in samples])
    onb, oib, og = (ctypes.c_int * n)(), (ctypes.c_int * n)(), (ctypes.c_double * n)()
    cnt = ctypes.c_int()
    _check(_lib.tileqr_preselect_tie(n, nb, ib, g, heuristic, cap, tie_rel, onb, oib, og, ctypes.byref(cnt)),
           "tileqr_preselect_tie")
    return [(onb[i], oib[i], og[i]) for i in range(cnt.value)]


def payg_prune(results):
    """Host-only Property-3 prune; results [(nb, ib, gflops)] -> survivors."""
    n = len(results)
    nb = (ctypes.c_int * n)(*[r[0] for r in results])
    g = (ctypes.c_double * n)(*[r[2] for r in results])
    keep = (ctypes.c_int * n)()
    _check(_lib.tileqr_payg_prune(n, nb, g, keep), "tileqr_payg_prune")
    return [r for r, k in zip(results, keep) if k]


def factor_plan(m: int, n: int, nb: int, ib: int) -> dict:
    out = (_i64 * 8)()
    _check(_lib.tileqr_factor_plan(m, n, nb, ib, out), "tileqr_factor_plan")
    keys = ["levels", "launches", "geqrt", "tsqrt", "larfb", "ssrfb", "MT", "NT"]
    return dict(zip(keys, list(out)))


def factor_schedule(nb: int, ib: int) -> str:
    return _lib.tileqr_factor_schedule(nb, ib).decode()


KINDS = {"geqrt": 0, "tsqrt": 1, "larfb": 2, "ssrfb": 3, "dag": 4, "dag_launches": 5}


def set_kernel_timing(on, kinds=("geqrt", "tsqrt", "larfb", "ssrfb"), launch_events=False):
    """Enable CUDA-event timing of the given kernel kinds (False/0: off).
    launch_events: only CUDA events around every dataflow-kernel launch (no
    device-clock trace), read back with kernel_times(..., "dag_launches")."""
    mask = 0 if not on else sum(1 << KINDS[k] for k in kinds)
    if launch_events:
        mask |= 16
    _lib.tileqr_set_kernel_timing(mask)


def kernel_times(m: int, n: int, nb: int, ib: int, kind: str):
    """(total_ms, launches, tasks) of one kernel kind in the last timed factor."""
    tot, nl, nt = _d(), _i64(), _i64()
    _check(_lib.tileqr_kernel_times(m, n, nb, ib, KINDS[kind], ctypes.byref(tot), ctypes.byref(nl),
                                    ctypes.byref(nt)), "tileqr_kernel_times")
    return tot.value, nl.value, nt.value


def kernel_trace(m: int, n: int, nb: int, ib: int, max_recs: int = 1 << 16):
    """Per-launch records of the last timed factor: list of (t0_ms, t1_ms, kind, level, tasks)."""
    t0 = (ctypes.c_double * max_recs)()
    t1 = (ctypes.c_double * max_recs)()
    kd = (ctypes.c_int * max_recs)()
    lv = (ctypes.c_int64 * max_recs)()
    nt = (ctypes.c_int64 * max_recs)()
    cnt = _i64()
    _check(_lib.tileqr_kernel_trace(m, n, nb, ib, max_recs, t0, t1, kd, lv, nt, ctypes.byref(cnt)),
           "tileqr_kernel_trace")
    names = {0: "geqrt", 1: "tsqrt", 2: "larfb", 3: "ssrfb", 4: "load", 5: "store"}
    return [(t0[i], t1[i], names[kd[i]], lv[i], nt[i]) for i in range(min(cnt.value, max_recs))]


def finalize():
    _lib.tileqr_finalize()
    _lib.tileqr_tree_finalize()


# ---------------------------------------------------------------------------
# tall-skinny / communication-avoiding variant (reduction tree)
# ---------------------------------------------------------------------------
def t_size_tree(m: int, n: int, nb: int, ib: int) -> int:
    out = _sz()
    _check(_lib.tileqr_t_size_tree(m, n, nb, ib, ctypes.byref(out)), "tileqr_t_size_tree")
    return out.value


def factor_tree(A: torch.Tensor, m: int, n: int, nb: int, ib: int, bs: int, T: torch.Tensor | None = None,
                info: torch.Tensor | None = None, lda: int | None = None, stream=None):
    """tileqr_factor_tree on the column-major m x n matrix stored in A (in place);
    bs = domain size in tile rows.  Returns (T (T then T2), info)."""
    assert A.dtype == torch.float64 and A.is_cuda and A.is_contiguous()
    if T is None:
        T = torch.empty(max(1, t_size_tree(m, n, nb, ib)), dtype=torch.float64, device=A.device)
    if info is None:
        info = torch.zeros(1, dtype=torch.int32, device=A.device)
    _check(_lib.tileqr_factor_tree(m, n, A.data_ptr(), lda if lda is not None else max(1, m), nb, ib, bs,
                                   T.data_ptr(), info.data_ptr(), _stream(stream)), "tileqr_factor_tree")
    return T, info


def apply_qt_tree(trans: str, A: torch.Tensor, m: int, k: int, T: torch.Tensor, nb: int, ib: int, bs: int,
                  B: torch.Tensor, nrhs: int, lda: int | None = None, ldb: int | None = None, stream=None):
    _check(_lib.tileqr_apply_qt_tree(trans.encode(), m, nrhs, k, A.data_ptr(), lda if lda is not None else max(1, m),
                                     T.data_ptr(), nb, ib, bs, B.data_ptr(), ldb if ldb is not None else max(1, m),
                                     _stream(stream)), "tileqr_apply_qt_tree")
    return B


def tune_tree(m: int, n: int, nb: int, ib: int, report_json_path: str | None = None):
    """(best BS, its median ms) of tileqr_factor_tree over BS = 1, 2, 4, ..., MT."""
    bs, ms = _i64(), _d()
    _check(_lib.tileqr_tune_tree(m, n, nb, ib, ctypes.byref(bs), ctypes.byref(ms),
                                 report_json_path.encode() if report_json_path else None), "tileqr_tune_tree")
    return bs.value, ms.value


def tree_plan_items(m: int, n: int, nb: int, ib: int, bs: int, workers: int, sub_cols: int):
    """Host-only claim-ordered work list of the tree variant: (kind, a, b, k, n, s, task, deps)."""
    cnt = _i64()
    _check(_lib.tileqr_tree_plan_items(m, n, nb, ib, bs, workers, sub_cols, None, 0, ctypes.byref(cnt)),
           "tileqr_tree_plan_items")
    out = (_i64 * (11 * max(1, cnt.value)))()
    _check(_lib.tileqr_tree_plan_items(m, n, nb, ib, bs, workers, sub_cols, out, 11 * cnt.value, ctypes.byref(cnt)),
           "tileqr_tree_plan_items")
    rows = []
    for i in range(cnt.value):
        r = list(out[11 * i: 11 * i + 11])
        rows.append((r[0], r[1], r[2], r[3], r[4], r[5], r[6], tuple(r[8:8 + r[7]])))
    return rows


def ttqrt_batched(nb: int, ib: int, R_ptrs, A2_ptrs, T_ptrs, stream=None):
    _check(_lib.tileqr_ttqrt_batched(nb, ib, R_ptrs.numel(), R_ptrs.data_ptr(), A2_ptrs.data_ptr(),
                                     T_ptrs.data_ptr(), _stream(stream)), "tileqr_ttqrt_batched")


# ---------------------------------------------------------------------------
# multi-GPU (one process per GPU; 1D block-cyclic tile columns)
# ---------------------------------------------------------------------------
def dist_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.tileqr_dist_unique_id(buf), "tileqr_dist_unique_id")
    return buf.raw


def dist_init(nranks: int, rank: int, unique_id: bytes, device: int):
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(_lib.tileqr_dist_init(nranks, rank, buf, device), "tileqr_dist_init")


def dist_local_cols(n: int, nb: int) -> int:
    out = ctypes.c_int()
    _check(_lib.tileqr_dist_local_cols(n, nb, ctypes.byref(out)), "tileqr_dist_local_cols")
    return out.value


def dist_fill_uniform(m: int, n: int, nb: int, A_local: torch.Tensor, seed: int, stream=None):
    _check(_lib.tileqr_dist_fill_uniform(m, n, nb, A_local.data_ptr(), seed, _stream(stream)),
           "tileqr_dist_fill_uniform")


def dist_factor(m: int, n: int, A_local: torch.Tensor, nb: int, ib: int, T_local: torch.Tensor,
                info: torch.Tensor | None = None, stream=None):
    _check(_lib.tileqr_dist_factor(m, n, A_local.data_ptr(), nb, ib, T_local.data_ptr(),
                                   info.data_ptr() if info is not None else None, _stream(stream)),
           "tileqr_dist_factor")


def dist_apply_qt_local(m: int, n: int, B_local: torch.Tensor, nb: int, ib: int, stream=None):
    """B <- Q^T B on this rank's local tile columns (after a dataflow dist_factor of the shape)."""
    _check(_lib.tileqr_dist_apply_qt_local(m, n, B_local.data_ptr(), nb, ib, _stream(stream)),
           "tileqr_dist_apply_qt_local")


def dist_residual_terms(m: int, n: int, nb: int, A_fact: torch.Tensor, QtA: torch.Tensor, rank: int,
                        nranks: int):
    """(||Q^T A - R||^2, ||A||^2-part) on this rank's local columns: R tile (i, j) is the whole tile
    above the diagonal tile, its upper triangle on it, zero below (the V tiles)."""
    mt = -(-m // nb)
    a = A_fact.view(-1, mt, nb, nb)      # [local col][tile row][jl][il]
    q = QtA.view(-1, mt, nb, nb)
    tot = torch.zeros((), dtype=torch.float64, device=A_fact.device)
    for j in range(a.shape[0]):
        c = rank + j * nranks
        for i in range(mt):
            r = a[j, i].t()
            if i == c:
                r = torch.triu(r)
            elif i > c:
                r = torch.zeros_like(r)
            tot += torch.sum((q[j, i].t() - r) ** 2)
    return tot


def dist_emulate(nranks: int, m: int, n: int, A_locals, nb: int, ib: int, T_locals,
                 info: torch.Tensor | None = None, stream=None):
    """Multi-rank dataflow factorization with `nranks` emulated ranks on this GPU."""
    pa = (ctypes.c_void_p * nranks)(*[a.data_ptr() if a is not None else None for a in A_locals])
    pt = (ctypes.c_void_p * nranks)(*[t.data_ptr() if t is not None else None for t in T_locals])
    _check(_lib.tileqr_dist_emulate(nranks, m, n, ctypes.cast(pa, ctypes.c_void_p), nb, ib,
                                    ctypes.cast(pt, ctypes.c_void_p),
                                    info.data_ptr() if info is not None else None, _stream(stream)),
           "tileqr_dist_emulate")


def dist_plan_items(m: int, n: int, nb: int, ib: int, nranks: int, rank: int, workers: int, sub_cols: int):
    """Host-only dataflow work list of one rank: list of
    (kind, k, m, n, s, task, deps) in claim order (KINDS_DIST names)."""
    cnt = _i64()
    _check(_lib.tileqr_dist_plan_items(m, n, nb, ib, nranks, rank, workers, sub_cols, None, 0,
                                       ctypes.byref(cnt)), "tileqr_dist_plan_items")
    out = (_i64 * (10 * max(1, cnt.value)))()
    _check(_lib.tileqr_dist_plan_items(m, n, nb, ib, nranks, rank, workers, sub_cols, out, 10 * cnt.value,
                                       ctypes.byref(cnt)), "tileqr_dist_plan_items")
    rows = []
    for i in range(cnt.value):
        r = list(out[10 * i: 10 * i + 10])
        rows.append((r[0], r[1], r[2], r[3], r[4], r[5], tuple(d for d in r[7:7 + r[6]])))
    return rows


KINDS_DIST = {0: "geqrt", 1: "tsqrt", 2: "larfb", 3: "ssrfb", 6: "arrive", 7: "copy"}


def dist_finalize():
    _lib.tileqr_dist_finalize()


def dist_plan_level(mt: int, nranks: int, rank: int, level: int):
    """Host-only plan of one level: (panel, bcast, update) lists of
    (kind, k, m, n, root) tuples."""
    cap = 5 * (mt * mt + 4 * mt + 8)
    out = (_i64 * cap)()
    cnt = (_i64 * 3)()
    _check(_lib.tileqr_dist_plan_level(mt, nranks, rank, level, out, cap, cnt), "tileqr_dist_plan_level")
    tup = [tuple(out[5 * i: 5 * i + 5]) for i in range(cnt[0] + cnt[1] + cnt[2])]
    return tup[:cnt[0]], tup[cnt[0]:cnt[0] + cnt[1]], tup[cnt[0] + cnt[1]:]
