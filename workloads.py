"""Synthetic inputs of the five BASELINE configurations.

The generators restate the reference's seeded fixtures (random.py:28-40 for
TT chains; the explicit hybrid of config 5) with the TNTZ_SEED convention
(config.py:5-18).  tests/test_workloads.py checks that they produce exactly
the numbers pinned from the real reference (tests/golden/configs.npz) and
the oracle's generators, so bench.py measures the same inputs the
reference would see.
"""

from __future__ import annotations

import os

import numpy as np

CONFIGS = {
    # name: (description, shape, rank)
    "cfg1": ("Pure TT, N=6 modes of size 16, ranks 8; full() 16^6 + t[idx] on 2^20 tuples",
             (16,) * 6, 8),
    "cfg2": ("Batched entry evaluation: TT N=10 modes of size 32, ranks 32; 2^24 int64 index "
             "tuples; output [2^24] fp32", (32,) * 10, 32),
    "cfg3": ("Dense decompression full(): TT N=4 modes of size 256, ranks 64; output 256^4 fp32 "
             "(17.18 GB)", (256,) * 4, 64),
    "cfg4": ("Batched dot/norm: 4096 pairs of TTs, N=16 modes of size 64, ranks 16",
             (64,) * 16, 16),
    "cfg5": ("Hybrid CP-TT-Tucker: N=8 modes of size 128 (factors 128x16), modes 0-3 TT rank 24, "
             "modes 4-7 CP rank 24; t[idx] on 2^26 tuples", (128,) * 8, 24),
}


def base_seed() -> int:
    return int(os.environ.get("TNTZ_SEED", "0"))


def tt_cores(shape, rank, seed, batch_size=None, scale=None, dtype=np.float32):
    """random_tt(shape, rank, seed, batch_size, scale) cores (random.py:28-40),
    drawn in float64 from one default_rng stream and cast to fp32."""
    rng = np.random.default_rng(seed)
    n = len(shape)
    ranks = [1] + [rank] * (n - 1) + [1]
    scale = rank ** -0.5 if scale is None else scale
    cores = []
    for k, isz in enumerate(shape):
        dims = (ranks[k], isz, ranks[k + 1])
        if batch_size is not None:
            dims = (batch_size,) + dims
        cores.append((scale * rng.standard_normal(dims)).astype(dtype))
    return cores


def hybrid_nodes(seed, dtype=np.float32):
    """Config 5: per mode draw the core then the factor, N(0, 1/24)."""
    rng = np.random.default_rng(seed)
    s = 24 ** -0.5
    nodes = []
    for k in range(8):
        if k < 4:
            core = rng.standard_normal((1 if k == 0 else 24, 16, 24)) * s
            kind = "tt"
        else:
            core = rng.standard_normal((16, 24)) * s
            kind = "cp"
        fac = rng.standard_normal((128, 16)) * s
        nodes.append((kind, core.astype(dtype), fac.astype(dtype)))
    return nodes


def indices(shape, m, seed):
    """int64 [m, N], uniform per mode (default_rng(seed).integers)."""
    rng = np.random.default_rng(seed)
    if len(set(shape)) == 1:
        return rng.integers(0, shape[0], size=(m, len(shape)), dtype=np.int64)
    return np.stack([rng.integers(0, s, size=m, dtype=np.int64) for s in shape], axis=1)


def entry_flops(modes) -> int:
    """Algorithmic FLOP per entry with factors pre-absorbed:
    2*r_l*r_r per dense mode, R per diagonal (interior CP) mode."""
    f = 0
    for layout, rl, rr in modes:
        f += rl if layout == "diag" else 2 * rl * rr
    return f
