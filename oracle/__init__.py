"""CPU oracle for the tile Householder QR of arxiv 1102.5328 (RR-7526).

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
this package.  The product package ``paper_1102_5328_b200`` never imports,
links or executes it; the two share no code (only ``synth_inputs`` seeds both).

Three parts:
  * ``tileqr_oracle.c`` (plain C loops, fp64) -- the tile kernels GEQRT,
    TSQRT, LARFB, SSRFB, the whole tile factorization and the Q application
    (P:147-187 of /root/reference/PAPER.md; S:58-106 of SPEC.md).  Wrapped
    here with ctypes; built by :func:`build` (gcc -O2 -fopenmp).
  * the tall-skinny / communication-avoiding variant:
    TTQRT / TTMQRT and the tree tile QR of DESIGN.md R20 (same C file);
  * ``oracle.tuner`` -- the paper's pruning rules (Properties 1-3,
    Heuristics 0/1/2, nearest-point lookup) and the DAG level schedule by an
    explicit dependency DP, in plain Python.

Parity status: every function here is pinned by tests/test_oracle_*.py
(see DESIGN.md "Oracle pins"); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tileqr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile the C oracle into oracle/liboracle.so (plain gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i, i64, c, d = ctypes.c_int, ctypes.c_int64, ctypes.c_char, ctypes.c_double
        lib.oracle_larfg.argtypes = [i, _dp, _dp, i]
        lib.oracle_larfg.restype = d
        lib.oracle_geqrt.argtypes = [i, i, _dp, i, _dp, i]
        lib.oracle_tsqrt.argtypes = [i, i, _dp, i, _dp, i, _dp, i]
        lib.oracle_larfb.argtypes = [c, i, i, _dp, i, _dp, i, _dp, i, i]
        lib.oracle_ssrfb.argtypes = [c, i, i, _dp, i, _dp, i, _dp, i, _dp, i, i]
        lib.oracle_tileqr_factor.argtypes = [i64, i64, _dp, i64, i, i, _dp, i, i]
        lib.oracle_tileqr_factor.restype = i
        lib.oracle_tileqr_apply.argtypes = [c, i64, i64, i64, _dp, i64, _dp, i, i, _dp, i64, i]
        lib.oracle_tileqr_apply.restype = i
        lib.oracle_ttqrt.argtypes = [i, i, _dp, i, _dp, i, _dp, i]
        lib.oracle_ttmqrt.argtypes = [c, i, i, _dp, i, _dp, i, _dp, i, _dp, i, i]
        lib.oracle_tileqr_factor_tree.argtypes = [i64, i64, _dp, i64, i, i, i64, _dp, i]
        lib.oracle_tileqr_factor_tree.restype = i
        lib.oracle_tileqr_apply_tree.argtypes = [c, i64, i64, i64, _dp, i64, _dp, i, i, i64, _dp, i64, i]
        lib.oracle_tileqr_apply_tree.restype = i
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.f_contiguous, "oracle arrays are fp64 Fortran-ordered"
    return a.ctypes.data_as(_dp)


def _f(a) -> np.ndarray:
    return np.array(a, dtype=np.float64, order="F", copy=True)


def larfg(alpha: float, x2):
    """Reflector rule (R1). Returns (beta, tau, v2)."""
    a = np.array([alpha], dtype=np.float64)
    x = _f(np.atleast_1d(x2))
    tau = _load().oracle_larfg(x.size, _ptr(a), _ptr(x), 1)
    return float(a[0]), float(tau), x


def geqrt(a, ib: int):
    """GEQRT of one NB x NB tile. Returns (tile with R/V, T (IB x NB))."""
    a = _f(a)
    nb = a.shape[0]
    t = np.zeros((ib, nb), order="F")
    _load().oracle_geqrt(nb, ib, _ptr(a), nb, _ptr(t), ib)
    return a, t


def tsqrt(r, b, ib: int):
    """TSQRT of [R; B]. Returns (R updated (upper part), V2, T)."""
    r, b = _f(r), _f(b)
    nb = r.shape[0]
    t = np.zeros((ib, nb), order="F")
    _load().oracle_tsqrt(nb, ib, _ptr(r), nb, _ptr(b), nb, _ptr(t), ib)
    return r, b, t


def larfb(v, t, c, trans: str = "T"):
    """C <- Q^T C ('T') or Q C ('N') with GEQRT reflectors (V, T)."""
    v, t, c = _f(v), _f(t), _f(c)
    nb, ib = v.shape[0], t.shape[0]
    _load().oracle_larfb(trans.encode(), nb, ib, _ptr(v), nb, _ptr(t), ib, _ptr(c), nb, c.shape[1])
    return c


def ssrfb(v2, t, c1, c2, trans: str = "T"):
    """[C1; C2] <- Q^T [C1; C2] ('T') or Q [C1; C2] ('N') with TSQRT reflectors."""
    v2, t, c1, c2 = _f(v2), _f(t), _f(c1), _f(c2)
    nb, ib = v2.shape[0], t.shape[0]
    _load().oracle_ssrfb(trans.encode(), nb, ib, _ptr(v2), nb, _ptr(t), ib, _ptr(c1), nb,
                         _ptr(c2), nb, c1.shape[1])
    return c1, c2


def ttqrt(r1, r2, ib: int):
    """TTQRT of [R1; R2] (both upper triangular; strict lower parts untouched).
    Returns (R1 updated (upper part), R2 with V2 in its upper triangle, T)."""
    r1, r2 = _f(r1), _f(r2)
    nb = r1.shape[0]
    t = np.zeros((ib, nb), order="F")
    _load().oracle_ttqrt(nb, ib, _ptr(r1), nb, _ptr(r2), nb, _ptr(t), ib)
    return r1, r2, t


def ttmqrt(v2, t, c1, c2, trans: str = "T"):
    """[C1; C2] <- Q^T [C1; C2] ('T') or Q [C1; C2] ('N') with TTQRT reflectors
    (the upper triangle of v2)."""
    v2, t, c1, c2 = _f(v2), _f(t), _f(c1), _f(c2)
    nb, ib = v2.shape[0], t.shape[0]
    _load().oracle_ttmqrt(trans.encode(), nb, ib, _ptr(v2), nb, _ptr(t), ib, _ptr(c1), nb,
                          _ptr(c2), nb, c1.shape[1])
    return c1, c2


def tileqr_factor_tree(a, nb: int, ib: int, bs: int, nthreads: int = 0):
    """Tile QR with the reduction tree of DESIGN.md R20 (domains of bs tile rows,
    flat inside, binary tree over the heads).  Returns (A with R and V, T flat
    array of 2 * t_size doubles: T then T2, info)."""
    a = _f(a)
    m, n = a.shape
    t = np.zeros(max(1, 2 * t_size(m, n, nb, ib)), dtype=np.float64)
    info = _load().oracle_tileqr_factor_tree(m, n, _ptr(a), max(1, m), nb, ib, bs, t.ctypes.data_as(_dp),
                                             nthreads)
    if info < 0:
        raise MemoryError("oracle allocation failed")
    return a, t, info


def tileqr_apply_tree(trans: str, a, t, nb: int, ib: int, bs: int, b, nthreads: int = 0):
    """B <- Q^T B ('T') or Q B ('N') for the Q of a tileqr_factor_tree output."""
    a = _f(a)
    b = _f(b)
    m, k = a.shape
    t = np.ascontiguousarray(t, dtype=np.float64)
    rc = _load().oracle_tileqr_apply_tree(trans.encode(), m, b.shape[1], k, _ptr(a), max(1, m),
                                          t.ctypes.data_as(_dp), nb, ib, bs, _ptr(b), max(1, m), nthreads)
    if rc < 0:
        raise MemoryError("oracle allocation failed")
    return b


def tree_heads(mt: int, k: int, bs: int):
    """Domain heads of panel k (R20)."""
    return [max(d * bs, k) for d in range(k // bs, -(-mt // bs))]


def t_size(m: int, n: int, nb: int, ib: int) -> int:
    mt, nt = -(-m // nb), -(-n // nb)
    return mt * nt * ib * nb


def tileqr_factor(a, nb: int, ib: int, nthreads: int = 0, kmax: int = 0):
    """Whole tile QR. Returns (A overwritten with R and V, T flat array, info)."""
    a = _f(a)
    m, n = a.shape
    t = np.zeros(max(1, t_size(m, n, nb, ib)), dtype=np.float64)
    info = _load().oracle_tileqr_factor(m, n, _ptr(a), max(1, m), nb, ib,
                                        t.ctypes.data_as(_dp), nthreads, kmax)
    if info < 0:
        raise MemoryError("oracle allocation failed")
    return a, t, info


def tileqr_apply(trans: str, a, t, nb: int, ib: int, b, nthreads: int = 0):
    """B <- Q^T B ('T') or Q B ('N') for the Q of a tileqr_factor output."""
    a = _f(a)
    b = _f(b)
    m, k = a.shape
    t = np.ascontiguousarray(t, dtype=np.float64)
    rc = _load().oracle_tileqr_apply(trans.encode(), m, b.shape[1], k, _ptr(a), max(1, m),
                                     t.ctypes.data_as(_dp), nb, ib, _ptr(b), max(1, m), nthreads)
    if rc < 0:
        raise MemoryError("oracle allocation failed")
    return b


def t_tile(t, m: int, n: int, nb: int, ib: int, mi: int, ki: int):
    """The IB x NB T factor of tile (mi, ki) inside a flat T array."""
    mt = -(-m // nb)
    off = (mi + ki * mt) * ib * nb
    return np.asarray(t[off: off + ib * nb]).reshape((ib, nb), order="F")


def sign_normalised_r(a_fact, n_cols: int | None = None):
    """R = triu(A[0:min(M,N), 0:N]) scaled by diag(sign(R_jj)), sign(0)=+1 (reading R10)."""
    m, n = a_fact.shape
    k = min(m, n)
    r = np.triu(np.asarray(a_fact)[:k, :n])
    s = np.where(np.diag(r) < 0, -1.0, 1.0)
    return s[:, None] * r
