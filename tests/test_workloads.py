"""bench.py's input generators produce the reference's pinned numbers."""

import numpy as np

import workloads as W
from oracle import tntz_oracle as O
from tests import golden_cases as G


def _stats(cores):
    out = []
    for c in cores:
        c64 = np.asarray(c, np.float64)
        out.append(np.concatenate([[c64.sum(), (c64 ** 2).sum()], c64.ravel()[:16]]))
    return np.stack(out)


def test_generators_match_reference_pins():
    z = G.configs()
    np.testing.assert_allclose(_stats(W.tt_cores((16,) * 6, 8, 0)), z["cfg1/core_stats"], rtol=1e-12)
    np.testing.assert_allclose(_stats(W.tt_cores((32,) * 10, 32, 0)), z["cfg2/core_stats"], rtol=1e-12)
    np.testing.assert_allclose(_stats(W.tt_cores((256,) * 4, 64, 0)), z["cfg3/core_stats"], rtol=1e-12)
    h = W.hybrid_nodes(0)
    np.testing.assert_allclose(_stats([n[1] for n in h] + [n[2] for n in h]), z["cfg5/core_stats"],
                               rtol=1e-12)
    assert np.array_equal(W.indices((32,) * 10, 4096, 2)[:64], z["cfg2/idx_head"])
    assert np.array_equal(W.indices((128,) * 8, 4096, 2)[:64], z["cfg5/idx_head"])


def test_generators_match_oracle():
    for a, b in zip(W.tt_cores((4, 5, 3), 2, 7), O.random_tt((4, 5, 3), 2, seed=7, scale=2 ** -0.5)):
        assert np.array_equal(a, b)
    for (k1, c1, f1), (k2, c2, f2) in zip(W.hybrid_nodes(3), O.cfg5_nodes(seed=3)):
        assert k1 == k2 and np.array_equal(c1, c2) and np.array_equal(f1, f2)
    assert np.array_equal(W.indices((5, 7), 100, 1), O.uniform_indices((5, 7), 100, 1))


def test_entry_flops():
    cfg2 = [("dense", 1, 32)] + [("dense", 32, 32)] * 8 + [("dense", 32, 1)]
    assert W.entry_flops(cfg2) == 16512
    cfg5 = [("dense", 1, 24)] + [("dense", 24, 24)] * 3 + [("diag", 24, 24)] * 3 + [("dense", 24, 1)]
    assert W.entry_flops(cfg5) == 48 + 3 * 1152 + 72 + 48
