"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no Householder, no tile
kernels): only the counter-based generator and the workload recipes of
BASELINE.json ``configs``.  The CUDA library
re-implements the same generator on the device (``tileqr_rng_uniform``);
tests check the two agree bit for bit.

Generator:
    x[idx] = (splitmix64(splitmix64(seed) + idx) >> 11) * 2^-53 - 0.5
with idx = i + j*M (global column-major index, independent of lda), i.e.
i.i.d. uniform(-0.5, 0.5) as BASELINE.json configs state.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """splitmix64 finaliser on uint64 numpy arrays/scalars (wrapping)."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + _GOLDEN
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def uniform(m: int, n: int, seed: int, offset: int = 0) -> np.ndarray:
    """m x n float64 Fortran-ordered matrix of i.i.d. uniform(-0.5, 0.5).

    Entry (i, j) uses counter idx = offset + i + j*m.
    """
    key = splitmix64(np.uint64(seed))
    out = np.empty((m, n), dtype=np.float64, order="F")
    flat = out.reshape(-1, order="F")
    chunk = 1 << 24
    total = m * n
    with np.errstate(over="ignore"):
        for s in range(0, total, chunk):
            e = min(total, s + chunk)
            idx = np.arange(s + offset, e + offset, dtype=np.uint64)
            bits = splitmix64(key + idx) >> np.uint64(11)
            flat[s:e] = bits.astype(np.float64) * (2.0 ** -53) - 0.5
    return out


# Workloads of BASELINE.json "configs" (indices 0..4).  Seeds per SURVEY §8(d).
CONFIGS = {
    0: dict(name="qr256_nb64_ib16", M=256, N=256, NB=64, IB=16, seed=1),
    1: dict(name="ssrfb_sweep_4096", batch=4096, seed=2,
            grid={64: [8, 16, 32, 64], 96: [8, 12, 16, 24, 32, 48, 96],
                  128: [8, 16, 32, 64, 128], 160: [8, 10, 16, 20, 32, 40, 80, 160],
                  192: [8, 12, 16, 24, 32, 48, 64, 96, 192],
                  256: [8, 16, 32, 64, 128, 256]}),
    2: dict(name="qr2048_grid", M=2048, N=2048, seed=3,
            nb_values=[64, 96, 128, 160, 192, 224, 256]),
    3: dict(name="qr10000_tuned", M=10000, N=10000, seed=4),
    4: dict(name="qr40000_dist", M=40000, N=40000, seed=5),
}


def divisors(nb: int, minimum: int = 1) -> list[int]:
    return [d for d in range(minimum, nb + 1) if nb % d == 0]


def ssrfb_pair_operands(nb: int, pair: int, seed: int = 2):
    """Operands of SSRFB-sweep pair `pair` (config [1]): the TSQRT inputs
    (top = triu(uniform), bottom = uniform) and the update tiles C1, C2.
    Operand o of pair p uses counters offset (4p + o) * nb^2."""
    base = 4 * pair * nb * nb
    top = np.triu(uniform(nb, nb, seed, base))
    bot = uniform(nb, nb, seed, base + nb * nb)
    c1 = uniform(nb, nb, seed, base + 2 * nb * nb)
    c2 = uniform(nb, nb, seed, base + 3 * nb * nb)
    return np.asfortranarray(top), bot, c1, c2
