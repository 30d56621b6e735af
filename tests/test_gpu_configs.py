"""Parity at the five BASELINE configurations (SURVEY §8(d) parity sampling).

Inputs come from the pinned generators (tests/test_oracle_golden.py checks
them against the real reference); the CPU oracle runs on subsets sized to
finish in seconds, and size-independent properties cover the full sizes.
"""

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests.helpers import assert_close, facade, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
tb = pytest.importorskip("paper_2206_11128_b200")
from paper_2206_11128_b200 import _native as N  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def tt(cores, batch=None):
    return facade([("tt", c, None) for c in cores], batch), O.make_chain([("tt", c) for c in cores], batch)


def test_cfg1_everything():
    cores = O.random_tt((16,) * 6, 8, seed=0, scale=8 ** -0.5)
    t, o = tt(cores)
    ref = O.full(o)
    assert_close(tb.full(t), ref, what="cfg1 full")
    idx = O.uniform_indices((16,) * 6, 1 << 20, 2)
    ref_e = ref[tuple(idx.T)]
    for algo in (N.ALGO_AUTO, N.ALGO_CHAIN, N.ALGO_LAYERED):
        assert_close(tb.entries(t, idx, algo=algo), ref_e, what=f"cfg1 entries {algo}")
    assert_close(np.asarray(tb.norm(t)), np.asarray(O.norm(o)), what="cfg1 norm")


@pytest.mark.parametrize("gsort", ["1", "0"])
def test_cfg2_subset(gsort, monkeypatch):
    # AUTO at the benchmarked size: the global-sort tcgen05 path (default) and
    # the bucketed state kernel (TNB_ENTRIES_GSORT=0)
    monkeypatch.setenv("TNB_ENTRIES_GSORT", gsort)
    cores = O.random_tt((32,) * 10, 32, seed=0, scale=32 ** -0.5)
    t, o = tt(cores)
    m = 1 << 24
    assert N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)["compute_kernel"] == (3 if gsort == "1" else 0)
    idx = torch.from_numpy(O.uniform_indices((32,) * 10, m, 2)).cuda()
    got = tb.entries(t, idx)
    assert tuple(got.shape) == (m,)
    # oracle on 2^20 samples spread over the whole batch (every shard)
    sel = np.linspace(0, m - 1, 1 << 20).astype(np.int64)
    sub = idx[torch.from_numpy(sel).cuda()].cpu().numpy()
    assert_close(to_np(got)[sel], O.entries(o, sub), what="cfg2")


def test_cfg5_subset():
    nodes = O.cfg5_nodes(seed=0)
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = 1 << 22
    idx = torch.from_numpy(O.uniform_indices((128,) * 8, m, 2)).cuda()
    got = to_np(tb.entries(t, idx))
    sel = np.linspace(0, m - 1, 1 << 18).astype(np.int64)
    assert_close(got[sel], O.entries(o, idx[torch.from_numpy(sel).cuda()].cpu().numpy()), what="cfg5")
    assert_close(np.asarray(tb.norm(t)), np.asarray(O.norm(o)), what="cfg5 norm")


def test_cfg3_slabs_and_norm():
    cores = O.random_tt((256,) * 4, 64, seed=0, scale=64 ** -0.5)
    t, o = tt(cores)
    for i0 in (0, 37, 128, 255):
        assert_close(tb.full(t, lead=(i0, i0 + 1)), O.full_slab(o, i0, i0 + 1), what=f"cfg3 slab {i0}")
    # a multi-slab shard (what one of 8 GPUs writes) against its slabs
    shard = tb.full(t, lead=(32, 64))
    for i in (0, 31):
        assert_close(shard[i:i + 1], O.full_slab(o, 32 + i, 33 + i), what="cfg3 shard")
    assert_close(np.asarray(tb.norm(t)), np.asarray(O.norm(o)), what="cfg3 norm")


@pytest.mark.slow
def test_cfg3_whole_tensor_checksum():
    # size-independent property at the full 17 GB size: sum of squares of
    # full(t) equals norm(t)^2 (core.py:387-391), accumulated in float64
    cores = O.random_tt((256,) * 4, 64, seed=0, scale=64 ** -0.5)
    t, o = tt(cores)
    f = tb.full(t)
    assert tuple(f.shape) == (256,) * 4
    acc = 0.0
    for i in range(0, 256, 16):
        acc += float((f[i:i + 16].double() ** 2).sum())
    ref = O.norm(o) ** 2
    assert abs(acc - ref) <= 1e-5 * ref
    del f


def test_cfg4_pairs():
    # all 4096 pairs, in 16 chunks of 256 through batch-sliced oracle chains
    # (SURVEY 8(d) parity sampling); dot and norm
    a = O.random_tt((64,) * 16, 16, seed=0, batch_size=4096, scale=0.25)
    b = O.random_tt((64,) * 16, 16, seed=1, batch_size=4096, scale=0.25)
    ta, oa = tt(a, 4096)
    tb_, ob = tt(b, 4096)
    dots = to_np(tb.dot(ta, tb_))
    norms = to_np(tb.norm(ta))
    assert dots.shape == (4096,) and norms.shape == (4096,)
    for lo in range(0, 4096, 256):
        hi = lo + 256
        sa, sb = O.batch_slice(oa, lo, hi), O.batch_slice(ob, lo, hi)
        ref_d = O.chain_dot(sa, sb)
        ref_n = O.norm(sa)
        assert_close(dots[lo:hi], ref_d, what=f"cfg4 dot [{lo}, {hi})")
        assert_close(norms[lo:hi], ref_n, what=f"cfg4 norm [{lo}, {hi})")


def test_cfg5_benchmarked_plan():
    # cfg5 at the size bench.py times (2^26 tuples): the planner's HBM prefix
    # table P012 (2^21 rows), the diagonal CP table and the stream kernel --
    # the exact plan behind the benchmark line, checked on 2^20 oracle rows
    # spread over the whole batch (core.py:394-444)
    nodes = O.cfg5_nodes(seed=0)
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = 1 << 26
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert (plan["n_virtual"], plan["prefix_rows"], plan["compute_kernel"]) == (4, 1 << 21, 1), plan
    idx = torch.from_numpy(O.uniform_indices((128,) * 8, m, 2)).cuda()
    got = tb.entries(t, idx)
    assert tuple(got.shape) == (m,)
    sel = torch.from_numpy(np.linspace(0, m - 1, 1 << 20).astype(np.int64)).cuda()
    sub = idx[sel].cpu().numpy()
    g = got[sel].double().cpu().numpy()
    del idx, got
    assert_close(g, O.entries(o, sub), what="cfg5 at 2^26")


def test_cfg2_benchmarked_plan(monkeypatch):
    # the plan behind the cfg2 headline: P0123 / S6789 HBM tables (2^20 rows
    # each), modes 4-5 merged into one sorted mode of 1024 slices, one global
    # sort, tcgen05 tiles (test_cfg2_subset checks its values at 2^24 tuples)
    monkeypatch.delenv("TNB_ENTRIES_GSORT", raising=False)
    cores = O.random_tt((32,) * 10, 32, seed=0, scale=32 ** -0.5)
    t, _ = tt(cores)
    plan = N.entries_plan(t._packed().chain, 1 << 24, N.ALGO_AUTO)
    assert (plan["algo"], plan["n_virtual"], plan["prefix_rows"], plan["suffix_rows"], plan["compute_kernel"]) == \
        (N.ALGO_GSORT, 3, 1 << 20, 1 << 20, 3), plan
    assert plan["tensor_flops"] == 3 * 2 * 32 * 32 * float(1 << 24)
    # without the global sort: two tensor-core sorted modes on the state kernel
    monkeypatch.setenv("TNB_ENTRIES_GSORT", "0")
    plan = N.entries_plan(t._packed().chain, 1 << 24, N.ALGO_AUTO)
    assert (plan["n_virtual"], plan["prefix_rows"], plan["suffix_rows"], plan["compute_kernel"]) == \
        (4, 1 << 20, 1 << 20, 0), plan
    assert plan["tensor_flops"] > 0
