"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the t-product's arithmetic: it only draws i.i.d. N(0,1) numbers and
lays them out.  Recipe (SURVEY.md 8(c) reading #10):

  numpy.random.default_rng(seed).standard_normal(n1*n2*n3) in float64, filled in Matlab
  linear order (element (i,j,k) at i + n1*j + n1*n2*k), then rounded RN to float32
  for the fp32 configs.  The fp64 oracle always consumes the *rounded* values the GPU saw.

Chunked generation from one Generator yields the same stream as one big draw, so large tensors
are produced chunk by chunk to bound host memory.
"""
from __future__ import annotations

import numpy as np

# the lateral-slice partition (pure index arithmetic, one definition): re-exported for tests/bench
from paper_1806_07247_b200.dist import lateral_shard  # noqa: F401

# BASELINE.json configs (shape tuples (n1, n2, n3, n4), dtype, seeds)
CONFIGS = {
    "c1": dict(n1=20, n2=30, n3=10, n4=15, dtype="f64", seedA=0, seedB=1, seedD=2),
    "c2": dict(n1=256, n2=256, n3=32, n4=256, dtype="f32", seedA=10, seedB=11),
    "c3": dict(n1=1024, n2=1024, n3=31, n4=512, dtype="f32", seedA=20, seedB=21,
               seedU=22, seedV=23, rank=5),
    "c4": dict(n1=64, n2=64, n3=4096, n4=64, dtype="f32", seedA=30, seedB=31),
    "c5": dict(n1=4096, n2=4096, n3=64, n4=8192, dtype="f32", seedA=40, seedB=41),
}

_CHUNK = 1 << 24


def normal(shape, seed: int, dtype=np.float32) -> np.ndarray:
    """i.i.d. N(0,1) tensor of ``shape`` from ``default_rng(seed)``, Matlab (Fortran) order.

    Returns a Fortran-ordered numpy array, so ``arr[i, j, k]`` is the paper's a_{ijk} and the
    memory layout is the C-ABI's (i fastest, then j, then k)."""
    n = int(np.prod(shape))
    rng = np.random.default_rng(seed)
    out = np.empty(n, dtype=dtype)
    for s in range(0, n, _CHUNK):
        e = min(n, s + _CHUNK)
        out[s:e] = rng.standard_normal(e - s)  # float64 draw, RN cast on assignment
    return out.reshape(shape, order="F")


def normal_lateral(shape, seed: int, j0: int, j1: int, dtype=np.float32) -> np.ndarray:
    """Lateral slices [j0, j1) of ``normal(shape, seed, dtype)``, without holding the whole tensor.

    The full stream is drawn chunk by chunk in Matlab order (so the values are bit-identical to the
    corresponding columns of ``normal(shape, seed)``) and only the wanted columns are kept."""
    n2, n4, n3 = shape
    w = j1 - j0
    out = np.empty((n2, w, n3), dtype=dtype, order="F")
    flat = out.reshape(-1, order="F")                 # view: column-major (i, j - j0, k)
    rng = np.random.default_rng(seed)
    slab = n2 * n4                                    # one frontal slice of the stream
    lo, hi = n2 * j0, n2 * j1                         # wanted window inside each slice
    pos = 0                                           # stream position
    total = slab * n3
    while pos < total:
        e = min(total, pos + _CHUNK)
        vals = rng.standard_normal(e - pos).astype(dtype)
        # copy the part of [pos, e) that falls in the window of each slice it touches
        k0, k1 = pos // slab, (e - 1) // slab
        for k in range(k0, k1 + 1):
            a = max(pos, k * slab + lo)
            b = min(e, k * slab + hi)
            if a < b:
                d = k * n2 * w + (a - k * slab - lo)
                flat[d:d + (b - a)] = vals[a - pos:b - pos]
        pos = e
    return out


def sample_columns(n4: int, count: int = 64, seed: int = 42) -> np.ndarray:
    """Fixed lateral-slice sample J for full-size parity: the first and last
    column, every shard boundary for world sizes 2/4/8, plus random others."""
    must = {0, n4 - 1}
    for w in (2, 4, 8):
        for r in range(1, w):
            s, _ = lateral_shard(n4, w, r)
            must.update({s - 1, s})
    must = sorted(x for x in must if 0 <= x < n4)
    rest = np.setdiff1d(np.arange(n4), must)
    k = max(0, min(len(rest), count - len(must)))
    extra = np.random.default_rng(seed).choice(rest, size=k, replace=False) if k else []
    return np.array(sorted(set(must) | set(int(x) for x in extra)), dtype=np.int64)
