"""Pins the CPU oracle (oracle/tntz_oracle.py) to the real reference's outputs.

Every golden case was produced by tntz itself (tests/golden/make_golden.py);
here the numpy restatement must reproduce them at the reference's own float64
tolerances (pkg/tests/test_core.py:89 uses 1e-12 * max(|ref|, 1)).
"""

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests import golden_cases as G

TOL = 1e-12


def close(got, ref, tol=TOL):
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape
    scale = max(float(np.abs(ref).max()) if ref.size else 0.0, 1.0)
    assert float(np.abs(got - ref).max() if ref.size else 0.0) <= tol * scale


@pytest.mark.parametrize("name", G.CASE_NAMES)
def test_oracle_matches_reference(name):
    c = G.case(name)
    t = O.make_chain(c["nodes"], c["batch"])
    out = c["out"]
    if "full" in out:
        close(O.full(t), out["full"])
    close(np.asarray(O.norm(t)), out["norm"])
    if "entries" in out:
        close(O.entries(t, out["idx"]), out["entries"])
    if "dot" in out:
        o = O.make_chain(*c["other"])
        close(np.asarray(O.chain_dot(t, o)), out["dot"], 1e-10)


@pytest.mark.parametrize("name", [n for n in G.CASE_NAMES if "hybrid" not in n])
def test_bruteforce_agrees_with_reference_full(name):
    # the independent summation oracle (restating pkg/tests/oracles.py:49-73)
    c = G.case(name)
    if "full" not in c["out"]:
        pytest.skip("no full")
    t = O.make_chain(c["nodes"], c["batch"])
    close(O.dense_bruteforce(t), c["out"]["full"], 1e-11)


def test_known_answers():
    # test_core.py:62-64: all-ones CP of rank 3 -> every entry 3.0
    c = G.case("kat_ones_cp")
    assert np.array_equal(c["out"]["full"], np.full((2, 2), 3.0))
    # test_core.py:66-72: rank-1 TT is the outer product
    c = G.case("kat_outer")
    assert np.array_equal(c["out"]["full"], np.outer([1.0, 2.0, 3.0], [4.0, 5.0]))
    # test_core.py:127-130: zero tensor norm is exactly 0; dot with zero is 0
    c = G.case("kat_zero")
    assert float(c["out"]["norm"]) == 0.0 and float(c["out"]["dot"]) == 0.0


def test_index_semantics():
    t = O.make_chain([("tt", np.arange(8.0).reshape(1, 4, 2)),
                      ("tt", np.arange(10.0).reshape(2, 5, 1))])
    f = O.full(t)
    # test_core.py:187-190: negatives normalise
    assert O.entries(t, np.array([[-1, -2]]))[0] == f[3, 3]
    # -size wraps to 0; -size-1 raises (SURVEY §8(a) probed quirks)
    assert O.entries(t, np.array([[-4, -5]]))[0] == f[0, 0]
    with pytest.raises(O.OracleError, match="mode 1"):
        O.entries(t, np.array([[0, -6]]))
    # lowest offending mode is reported (core.py:409-416)
    with pytest.raises(O.OracleError, match="mode 0"):
        O.entries(t, np.array([[4, 9], [0, 0]]))
    # 1-D index is one sample; empty gives shape (0,)
    assert O.entries(t, np.array([1, 1])).shape == (1,)
    assert O.entries(t, np.zeros((0, 2), dtype=np.int64)).shape == (0,)
    with pytest.raises(O.OracleError):
        O.entries(t, np.zeros((3, 3), dtype=np.int64))


def _stats_match(cores, stats):
    got = []
    for c in cores:
        c64 = np.asarray(c, dtype=np.float64)
        got.append(np.concatenate([[c64.sum(), (c64 ** 2).sum()], c64.ravel()[:16]]))
    np.testing.assert_allclose(np.stack(got), stats, rtol=1e-12, atol=0)


def test_config_generators_pinned():
    z = G.configs()
    _stats_match(O.random_tt((16,) * 6, 8, seed=0, scale=8 ** -0.5), z["cfg1/core_stats"])
    _stats_match(O.random_tt((32,) * 10, 32, seed=0, scale=32 ** -0.5), z["cfg2/core_stats"])
    _stats_match(O.random_tt((256,) * 4, 64, seed=0, scale=64 ** -0.5), z["cfg3/core_stats"])
    n5 = O.cfg5_nodes(seed=0)
    _stats_match([n[1] for n in n5] + [n[2] for n in n5], z["cfg5/core_stats"])
    # index streams: the first rows do not depend on the total sample count
    assert np.array_equal(O.uniform_indices((16,) * 6, 1 << 14, 2)[:64], z["cfg1/idx_head"])
    assert np.array_equal(O.uniform_indices((32,) * 10, 1 << 14, 2)[:64], z["cfg2/idx_head"])
    assert np.array_equal(O.uniform_indices((128,) * 8, 1 << 14, 2)[:64], z["cfg5/idx_head"])


def test_config_outputs_pinned():
    z = G.configs()
    t1 = O.make_chain([("tt", c) for c in O.random_tt((16,) * 6, 8, seed=0, scale=8 ** -0.5)])
    i1 = O.uniform_indices((16,) * 6, 4096, 2)
    close(O.entries(t1, i1), z["cfg1/entries"])
    close(O.norm(t1), z["cfg1/norm"])
    slab = O.full_slab(t1, 0, 1)
    close(slab.ravel()[:256], z["cfg1/slab0_head"])
    t2 = O.make_chain([("tt", c) for c in O.random_tt((32,) * 10, 32, seed=0, scale=32 ** -0.5)])
    close(O.entries(t2, O.uniform_indices((32,) * 10, 2048, 2)), z["cfg2/entries"])
    t5 = O.make_chain(O.cfg5_nodes(seed=0))
    close(O.entries(t5, O.uniform_indices((128,) * 8, 2048, 2)), z["cfg5/entries"])
    close(O.norm(t5), z["cfg5/norm"], 1e-10)


def test_cfg3_pinned():
    z = G.configs()
    t3 = O.make_chain([("tt", c) for c in O.random_tt((256,) * 4, 64, seed=0, scale=64 ** -0.5)])
    close(O.norm(t3), z["cfg3/norm"], 1e-10)
    slab = O.full_slab(t3, 255, 256).ravel()
    close(slab[z["cfg3/slab255_pos"]], z["cfg3/slab255_val"])


def test_cfg4_pinned():
    z = G.configs()
    if "cfg4/pairs" not in z.files:
        pytest.skip("cfg4 pin not generated (make_golden.py --big)")
    pairs = z["cfg4/pairs"]
    # regenerate only what the pinned pairs need would still draw the full
    # stream; check the cheap per-core statistics of the first cores instead
    a = O.random_tt((64,) * 16, 16, seed=0, batch_size=4096, scale=0.25)
    _stats_match(a, z["cfg4/core_stats_a"])
    ta = O.make_chain([("tt", c) for c in a], 4096)
    na = np.array([O.norm(O.batch_element(ta, int(p))) for p in pairs])
    close(na, z["cfg4/norm"], 1e-10)
