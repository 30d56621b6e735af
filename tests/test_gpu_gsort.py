"""GPU parity of the global-sort tcgen05 entries path (TNB_ALGO_GSORT,
csrc/entries_gsort.cuh) against the oracle (core.py:394-444): merged interior
modes, diagonal tables, ragged bucket tails, empty buckets, skewed keys,
negative wrap and the lowest-bad-mode report, all through the C ABI."""

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests.helpers import assert_close, facade

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
tb = pytest.importorskip("paper_2206_11128_b200")
from paper_2206_11128_b200 import _native as N  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _plan(t, m, algo=N.ALGO_GSORT):
    return N.entries_plan(t._packed().chain, m, algo)


def _tt(shape, ranks, seed, scale):
    rng = np.random.default_rng(seed)
    rk = [1] + list(ranks) + [1]
    return [("tt", (rng.standard_normal((rk[k], shape[k], rk[k + 1])) * scale).astype(np.float32), None)
            for k in range(len(shape))]


def _no_tables(monkeypatch):
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "1")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "1")


@pytest.mark.parametrize("m", [1, 127, 129, 5000, 300001])
def test_gsort_tiles_and_tails(m, monkeypatch):
    # first . G1234 (4 merged modes, 4096 slices: ragged and empty buckets) . last
    _no_tables(monkeypatch)
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 6, 16, seed=7, scale=0.25)]
    t, o = facade(nodes), O.make_chain(nodes)
    idx = O.uniform_indices(t.shape, m, 3)
    idx[::3] -= np.asarray(t.shape)
    plan = _plan(t, m)
    assert (plan["algo"], plan["compute_kernel"], plan["n_virtual"]) == (N.ALGO_GSORT, 3, 3), plan
    assert_close(tb.entries(t, idx, algo=N.ALGO_GSORT), O.entries(o, idx), what=f"m={m}")


def test_gsort_tt_merged_interior(monkeypatch):
    # P012 . G3456 (4 merged modes, 4096 slices) . S789
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "512")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "512")
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 10, 16, seed=7, scale=0.25)]
    t, o = facade(nodes), O.make_chain(nodes)
    m = 300001
    idx = O.uniform_indices(t.shape, m, 3)
    idx[::3] -= np.asarray(t.shape)
    plan = _plan(t, m)
    assert (plan["compute_kernel"], plan["n_virtual"], plan["prefix_rows"], plan["suffix_rows"]) == (3, 3, 512, 512), plan
    assert_close(tb.entries(t, idx, algo=N.ALGO_GSORT), O.entries(o, idx))


@pytest.mark.parametrize("r", [8, 24, 32])
def test_gsort_rank_classes(r, monkeypatch):
    _no_tables(monkeypatch)
    # first . G1 G2 (merged, 30 * 20 slices) . last, original boundary modes
    nodes = _tt((50, 30, 20, 70), (r, r, r), seed=r, scale=r ** -0.5)
    t, o = facade(nodes), O.make_chain(nodes)
    m = 40000
    idx = O.uniform_indices(t.shape, m, r)
    plan = _plan(t, m)
    assert plan["compute_kernel"] == 3, plan
    assert_close(tb.entries(t, idx, algo=N.ALGO_GSORT), O.entries(o, idx))


def test_gsort_rectangular_slices(monkeypatch):
    _no_tables(monkeypatch)
    # r0 = 24 into r1 = 16 through a 12-wide interior rank: non-square levels
    nodes = _tt((40, 9, 11, 60), (24, 12, 16), seed=3, scale=0.3)
    t, o = facade(nodes), O.make_chain(nodes)
    idx = O.uniform_indices(t.shape, 30011, 4)
    assert _plan(t, 30011)["compute_kernel"] == 3
    assert_close(tb.entries(t, idx, algo=N.ALGO_GSORT), O.entries(o, idx))


def test_gsort_cfg5_structure_with_diag():
    # P01 . G2 G3 (16384 slices: the many-bucket histogram / scatter) . D45 . S67
    nodes = O.cfg5_nodes(seed=1)
    t, o = facade(nodes), O.make_chain(nodes)
    m = 1 << 18
    idx = O.uniform_indices((128,) * 8, m, 9)
    idx[1::5] -= 128
    plan = _plan(t, m)
    assert (plan["compute_kernel"], plan["n_virtual"], plan["diag_tables"]) == (3, 4, 1), plan
    got = tb.entries(t, idx, algo=N.ALGO_GSORT)
    sel = np.arange(0, m, 3)
    assert_close(got[torch.as_tensor(sel, device=got.device)], O.entries(o, idx[sel]))


@pytest.mark.parametrize("pattern", ["one_key", "two_keys", "slice_first", "fibers"])
def test_gsort_skewed_keys(pattern, monkeypatch):
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "512")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "512")
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 8, 16, seed=11, scale=0.25)]
    t, o = facade(nodes), O.make_chain(nodes)
    m = 50000
    idx = O.uniform_indices(t.shape, m, 5)
    if pattern == "one_key":
        idx[:, 3:5] = 5
    elif pattern == "two_keys":
        idx[:, 3] = 2
        idx[:, 4] = idx[:, 4] % 2 * 7
    elif pattern == "slice_first":
        idx[:, :4] = 1
    else:
        idx[:, :-1] = idx[0, :-1]
    assert_close(tb.entries(t, idx, algo=N.ALGO_GSORT), O.entries(o, idx), what=pattern)


def test_gsort_reports_lowest_bad_mode(monkeypatch):
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "512")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "512")
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 8, 8, seed=13, scale=0.35)]
    t = facade(nodes)
    idx = O.uniform_indices(t.shape, 20000, 6)
    for mode in (0, 2, 3, 4, 6, 7):
        bad = idx.copy()
        bad[777, mode] = 8
        bad[12000, 7] = -9
        with pytest.raises(tb.ContractViolationError, match=f"mode {mode}"):
            tb.entries(t, bad, algo=N.ALGO_GSORT)


def test_gsort_auto_at_cfg2_shape():
    # AUTO picks the global-sort path for large calls (here an 8-mode cfg2-style chain
    # at 2^20 tuples: P012 . G34 . S567) and the result matches the bucketed kernels' and the oracle
    c32 = O.random_tt((32,) * 8, 32, seed=7, scale=32 ** -0.5)
    nodes = [("tt", c, None) for c in c32]
    t, o = facade(nodes), O.make_chain(nodes)
    m = 1 << 20
    plan = _plan(t, m, N.ALGO_AUTO)
    assert (plan["algo"], plan["compute_kernel"]) == (N.ALGO_GSORT, 3), plan
    idx = O.uniform_indices(t.shape, m, 8)
    got = tb.entries(t, idx)
    sel = np.arange(0, m, 16)
    assert_close(got[torch.as_tensor(sel, device=got.device)], O.entries(o, idx[sel]))
    old = tb.entries(t, idx, algo=N.ALGO_BUCKETED)
    assert_close(got, old.double().cpu().numpy(), tol=2e-5)


def test_gsort_rejects_unsupported_chains():
    # odd ranks have no 16-byte row pieces: the explicit algorithm refuses, AUTO falls back
    nodes = _tt((20, 12, 13, 25), (5, 7, 6), seed=2, scale=0.4)
    t, o = facade(nodes), O.make_chain(nodes)
    idx = O.uniform_indices(t.shape, 70000, 1)
    with pytest.raises(tb.ContractViolationError):
        tb.entries(t, idx, algo=N.ALGO_GSORT)
    assert_close(tb.entries(t, idx), O.entries(o, idx))


def test_gsort_is_bitwise_reproducible(monkeypatch):
    # the scatter's order inside a bucket is not fixed, the values must not depend on it
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "512")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "512")
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 8, 32, seed=21, scale=32 ** -0.5)]
    t = facade(nodes)
    idx = torch.from_numpy(O.uniform_indices(t.shape, 400000, 7)).cuda()
    a = tb.entries(t, idx, algo=N.ALGO_GSORT)
    b = tb.entries(t, idx, algo=N.ALGO_GSORT)
    perm = torch.randperm(idx.shape[0], device="cuda")
    c = tb.entries(t, idx[perm], algo=N.ALGO_GSORT)
    assert torch.equal(a, b)
    assert torch.equal(a[perm], c)


def test_gsort_mid_size_uses_wider_tables():
    # cfg2 chain at 2^21 tuples (a rank's shard of the headline at 8 GPUs): the
    # usual merge (tables of up to m / 8 rows) leaves four interior modes, so
    # the planner retries with tables of up to m / 2 rows: P0123 . G45 . S6789
    cores = O.random_tt((32,) * 10, 32, seed=0, scale=32 ** -0.5)
    nodes = [("tt", c, None) for c in cores]
    t, o = facade(nodes), O.make_chain(nodes)
    m = 1 << 21
    plan = _plan(t, m, N.ALGO_AUTO)
    assert (plan["algo"], plan["n_virtual"], plan["prefix_rows"], plan["suffix_rows"]) == \
        (N.ALGO_GSORT, 3, 1 << 20, 1 << 20), plan
    idx = O.uniform_indices(t.shape, m, 5)
    idx[3::11] -= 32
    got = tb.entries(t, idx)
    sel = np.arange(0, m, 37)
    assert_close(got[torch.as_tensor(sel, device=got.device)], O.entries(o, idx[sel]))


def test_gsort_batched_chains():
    # batched chains (core.py:425-429, 447-460): the records are sorted once and
    # every element runs its own tables and compute launch; each column equals
    # the unbatched element bitwise
    B, m = 3, 1 << 20
    cores = O.random_tt((32,) * 8, 32, seed=31, batch_size=B, scale=32 ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in cores], B)
    plan = _plan(t, m, N.ALGO_AUTO)
    assert (plan["algo"], plan["compute_kernel"], plan["n_virtual"]) == (N.ALGO_GSORT, 3, 3), plan
    idx = O.uniform_indices((32,) * 8, m, 9)
    idx[5::13] -= 32
    got = tb.entries(t, idx)
    assert tuple(got.shape) == (m, B)
    sel = np.arange(0, m, 257)
    o = O.make_chain([("tt", c) for c in cores], B)
    assert_close(got[torch.as_tensor(sel, device=got.device)], O.entries(o, idx[sel]))
    for b in range(B):
        tb_b = t.batch_element(b)
        assert torch.equal(got[:, b], tb.entries(tb_b, idx))
    bad = idx.copy()
    bad[4242, 6] = 32
    with pytest.raises(tb.ContractViolationError, match="mode 6"):
        tb.entries(t, bad)


def test_gsort_batched_cfg2_shape_plan():
    # B cfg2-shape chains on 2^20 tuples (bench.py's batched line): tables of up
    # to m rows pay because the index passes are shared -- P0123 . G45 . S6789
    B, m = 2, 1 << 20
    cores = O.random_tt((32,) * 10, 32, seed=33, batch_size=B, scale=32 ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in cores], B)
    plan = _plan(t, m, N.ALGO_AUTO)
    assert (plan["algo"], plan["n_virtual"], plan["prefix_rows"], plan["suffix_rows"]) == \
        (N.ALGO_GSORT, 3, 1 << 20, 1 << 20), plan
    idx = O.uniform_indices((32,) * 10, m, 10)
    got = tb.entries(t, idx)
    sel = np.arange(0, m, 509)
    o = O.make_chain([("tt", c) for c in cores], B)
    assert_close(got[torch.as_tensor(sel, device=got.device)], O.entries(o, idx[sel]))


@pytest.mark.parametrize("log2", ["16", "18"])
def test_gsort_result_windows(log2, monkeypatch):
    # results too large for L2 are written one window of samples at a time
    # (the sample index's high bits lead the sort key, CTAs interleaved);
    # TNB_GS_CHUNK_LOG2 forces small windows here.  Per-sample values do not
    # depend on the sort order: bitwise equal to the unwindowed call.
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "512")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "512")
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 8, 16, seed=9, scale=0.25)]
    t, o = facade(nodes), O.make_chain(nodes)
    m = 700001  # ragged last window
    idx = O.uniform_indices(t.shape, m, 5)
    idx[::5] -= np.asarray(t.shape)
    monkeypatch.setenv("TNB_GS_CHUNK_LOG2", "0")
    ref = tb.entries(t, idx, algo=N.ALGO_GSORT)
    monkeypatch.setenv("TNB_GS_CHUNK_LOG2", log2)
    got = tb.entries(t, idx, algo=N.ALGO_GSORT)
    assert torch.equal(got, ref)
    sel = np.arange(0, m, 53)
    assert_close(got[torch.from_numpy(sel).cuda()], O.entries(o, idx[sel]))
    bad = idx.copy()
    bad[m - 3, 6] = 8
    with pytest.raises(tb.ContractViolationError, match="mode 6"):
        tb.entries(t, bad, algo=N.ALGO_GSORT)


@pytest.mark.slow
def test_gsort_result_windows_default_above_64mb(monkeypatch):
    # a result above 64 MB takes the windowed sort key by default; same bits as
    # the unwindowed call, values against the oracle on a subsample
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "512")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "512")
    nodes = [("tt", c, None) for c in O.random_tt((8,) * 8, 16, seed=13, scale=0.25)]
    t, o = facade(nodes), O.make_chain(nodes)
    m = (1 << 24) + (1 << 21) + 77
    g = torch.Generator(device="cuda")
    g.manual_seed(17)
    idx = torch.randint(0, 8, (m, 8), device="cuda", generator=g)
    monkeypatch.delenv("TNB_GS_CHUNK_LOG2", raising=False)
    got = tb.entries(t, idx, algo=N.ALGO_GSORT)
    monkeypatch.setenv("TNB_GS_CHUNK_LOG2", "0")
    ref = tb.entries(t, idx, algo=N.ALGO_GSORT)
    assert torch.equal(got, ref)
    sel = torch.arange(0, m, 4099, device="cuda")
    assert_close(got[sel], O.entries(o, idx[sel].cpu().numpy()))
