"""GPU parity: the CUDA path (through libtnb's C ABI via the façade) against
the reference's golden vectors and the pinned CPU oracle."""

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests import golden_cases as G
from tests.helpers import assert_close, assert_dot_close, facade, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
tb = pytest.importorskip("paper_2206_11128_b200")
from paper_2206_11128_b200 import _native as N  # noqa: E402

ALGOS = [N.ALGO_AUTO, N.ALGO_LAYERED, N.ALGO_CHAIN, N.ALGO_BUCKETED]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(autouse=True)
def _bucketed_auto(monkeypatch):
    # this module pins the bucketed / generic kernels: AUTO must not route
    # large calls to the global-sort path (tests/test_gpu_gsort.py covers it)
    monkeypatch.setenv("TNB_ENTRIES_GSORT", "0")


@pytest.mark.parametrize("name", G.CASE_NAMES)
def test_golden_full_norm(name):
    c = G.case(name)
    t = facade(c["nodes"], c["batch"])
    out = c["out"]
    if "full" in out:
        assert_close(tb.full(t), out["full"], what=f"{name} full")
    ref_norm = np.asarray(out["norm"], dtype=np.float64)
    got = tb.norm(t)
    if c["batch"] is None:
        assert isinstance(got, float)
    assert_close(np.asarray(to_np(got)), ref_norm, what=f"{name} norm")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("name", [n for n in G.CASE_NAMES if "entries" in G.case(n)["out"]])
def test_golden_entries(name, algo):
    c = G.case(name)
    t = facade(c["nodes"], c["batch"])
    # batched chains run the bucketed kernels per batch element too
    # (shared tile records, per-element tables, [m][B] transpose)
    got = tb.entries(t, c["out"]["idx"], algo=algo)
    assert_close(got, c["out"]["entries"], what=f"{name} entries algo={algo}")


@pytest.mark.parametrize("name", [n for n in G.CASE_NAMES if "dot" in G.case(n)["out"]])
def test_golden_dot(name):
    c = G.case(name)
    a = facade(c["nodes"], c["batch"])
    b = facade(*c["other"])
    oa, ob = O.make_chain(c["nodes"], c["batch"]), O.make_chain(*c["other"])
    scale = np.asarray(O.norm(oa)) * np.asarray(O.norm(ob))
    got = tb.dot(a, b)
    if c["batch"] is None:
        assert isinstance(got, float)
    assert_dot_close(got, c["out"]["dot"], scale, what=f"{name} dot")


@pytest.mark.parametrize("name", G.CASE_NAMES)
def test_node_tt_core_matches_oracle(name):
    c = G.case(name)
    t = facade(c["nodes"], c["batch"])
    oc = O.make_chain(c["nodes"], c["batch"])
    for k in range(t.ndim):
        assert_close(tb.node_tt_core(t, k), O.tt_core(oc, k), what=f"{name} mode {k}")


def test_promote_cp_node_layouts():
    # test_core.py:21-53 layouts
    n = tb.ModeNode("cp", np.eye(2))
    d = to_np(tb.promote_cp_node(n, tb.INTERIOR))
    exp = np.zeros((2, 2, 2))
    for a in range(2):
        exp[a, a, a] = 1.0
    assert np.array_equal(d, exp)
    d = to_np(tb.promote_cp_node(tb.ModeNode("cp", np.ones((3, 2))), tb.LEFT_BOUNDARY))
    assert d.shape == (1, 3, 2) and np.array_equal(d, np.ones((1, 3, 2)))
    u = np.arange(12.0).reshape(4, 3)
    d = to_np(tb.promote_cp_node(tb.ModeNode("cp", u), tb.RIGHT_BOUNDARY))
    assert d.shape == (3, 4, 1) and np.array_equal(d[:, :, 0], u.T)
    ub = np.random.default_rng(0).standard_normal((2, 4, 3)).astype(np.float32)
    d = to_np(tb.promote_cp_node(tb.ModeNode("cp", ub, batched=True), tb.INTERIOR))
    for b in range(2):
        assert np.array_equal(d[b], O.promote_cp(ub[b].astype(np.float64), 1, 3, False))
    with pytest.raises(tb.ContractViolationError):
        tb.promote_cp_node(tb.ModeNode("tt", np.ones((1, 3, 1))), tb.INTERIOR)


# -- index semantics (core.py:402-416, indexing.py:120-130) -----------------

def _small():
    cores = O.random_tt((4, 5, 3), [2, 3], seed=1)
    return facade([("tt", c, None) for c in cores]), O.make_chain([("tt", c) for c in cores])


@pytest.mark.parametrize("algo", ALGOS)
def test_index_semantics(algo):
    t, o = _small()
    f = O.full(o)
    v = to_np(tb.entries(t, np.array([[-1, -2, -3]]), algo=algo))
    assert v.shape == (1,) and abs(v[0] - f[3, 3, 0]) <= 1e-5 * np.abs(f).max()
    # -size wraps to 0
    v = to_np(tb.entries(t, np.array([[-4, -5, -3]]), algo=algo))
    assert abs(v[0] - f[0, 0, 0]) <= 1e-5 * np.abs(f).max()
    # out of bounds: lowest offending mode named, both directions
    with pytest.raises(tb.ContractViolationError, match="index out of bounds on mode 1"):
        tb.entries(t, np.array([[0, 5, 0], [0, 0, 7]]), algo=algo)
    with pytest.raises(tb.ContractViolationError, match="mode 0"):
        tb.entries(t, np.array([[0, 0, 0], [-5, 0, 9]]), algo=algo)
    with pytest.raises(tb.ContractViolationError, match="mode 2"):
        tb.entries(t, np.array([[0, 0, -4]]), algo=algo)
    # 1-D index -> one sample; int32 accepted; empty -> (0,)
    assert tuple(tb.entries(t, np.array([1, 2, 0])).shape) == (1,)
    i32 = np.array([[1, 2, 0], [3, 4, 2]], dtype=np.int32)
    assert_close(tb.entries(t, i32, algo=algo), O.entries(o, i32))
    assert tuple(tb.entries(t, np.zeros((0, 3), dtype=np.int64)).shape) == (0,)
    # torch index tensors, host and device
    ti = torch.tensor([[1, 2, 0]])
    assert_close(tb.entries(t, ti), O.entries(o, ti.numpy()))
    assert_close(tb.entries(t, ti.cuda()), O.entries(o, ti.numpy()))
    with pytest.raises(tb.ContractViolationError):
        tb.entries(t, np.zeros((2, 2), dtype=np.int64))


def test_float_indices_follow_reference_quirk():
    # entries() floors float indices after wrapping (SURVEY §8(a) probes);
    # getitem() rejects them (indexing.py:128-129)
    t, o = _small()
    fi = np.array([[1.5, 2.0, -0.5]])
    assert_close(tb.entries(t, fi), O.entries(o, fi))
    with pytest.raises(tb.ContractViolationError, match="mode 1"):
        tb.entries(t, np.array([[0.0, 5.0, 0.0]]))
    with pytest.raises(tb.ContractViolationError, match="integers"):
        t[np.array([[0.5, 1.0, 0.0]])]


def test_getitem_forms():
    t, o = _small()
    f = O.full(o)
    idx = np.array([[0, 1, 2], [3, 4, 0], [1, 0, 1]])
    vals = t[idx]
    assert tuple(vals.shape) == (3,)
    assert_close(vals, f[idx[:, 0], idx[:, 1], idx[:, 2]])
    with pytest.raises(tb.ContractViolationError, match="columns"):
        t[np.array([[0, 1]])]
    # all-integer tuple -> python float; bounds checked last mode first
    assert abs(t[1, 2, -1] - f[1, 2, 2]) <= 1e-5 * np.abs(f).max()
    with pytest.raises(tb.ContractViolationError, match="index 9 out of bounds for size 3"):
        t[7, 0, 9]
    with pytest.raises(NotImplementedError):
        t[0:2]


def test_batched_entries_and_getitem():
    c = G.case("batched_tt")
    t = facade(c["nodes"], c["batch"])
    got = t[c["out"]["idx"]]
    assert tuple(got.shape) == (c["out"]["idx"].shape[0], c["batch"])
    assert_close(got, c["out"]["entries"])


def test_full_slabs_match_reference_slicing():
    for name in ("tt_453", "tucker_675", "blended_3", "batched_hybrid", "hybrid_wide"):
        c = G.case(name)
        t = facade(c["nodes"], c["batch"])
        o = O.make_chain(c["nodes"], c["batch"])
        j0 = t.shape[0]
        for lo, hi in [(0, 1), (1, j0), (j0 - 1, j0), (0, j0)]:
            assert_close(tb.full(t, lead=(lo, hi)), O.full_slab(o, lo, hi), what=f"{name} [{lo},{hi})")
        assert tuple(tb.full(t, lead=(1, 1)).shape)[-t.ndim] == 0


def test_dot_contract_errors():
    a = facade([("tt", c, None) for c in O.random_tt((2, 3), 1, seed=0)])
    b = facade([("tt", c, None) for c in O.random_tt((3, 2), 1, seed=0)])
    with pytest.raises(tb.ContractViolationError, match="dot needs equal shapes"):
        tb.dot(a, b)
    bb = facade([("tt", c, None) for c in O.random_tt((2, 3), 1, seed=0, batch_size=2)], 2)
    with pytest.raises(tb.ContractViolationError, match="agree on batching"):
        tb.dot(a, bb)


def test_dot_zero_is_exact():
    # test_arithmetic.py:121-123
    a = facade([("tt", c, None) for c in O.random_tt((3, 4), 2, seed=16)])
    z = facade([("tt", c * 0, None) for c in O.random_tt((3, 4), 2, seed=16)])
    assert tb.dot(a, z) == 0.0
    assert tb.norm(z) == 0.0


def test_batched_dot_equals_loop():
    # test_arithmetic.py:346-387
    a = facade([("tt", c, None) for c in O.random_tt((3, 4, 5), 3, seed=45, batch_size=3)], 3)
    b = facade([("tt", c, None) for c in O.random_tt((3, 4, 5), 2, seed=46, batch_size=3)], 3)
    vec = to_np(tb.dot(a, b))
    for e in range(3):
        assert abs(vec[e] - tb.dot(a.batch_element(e), b.batch_element(e))) <= 1e-6 * max(abs(vec[e]), 1)


@pytest.mark.parametrize("m", [1, 31, 1000, 5000, 70001])
@pytest.mark.parametrize("algo", [N.ALGO_BUCKETED, N.ALGO_AUTO])
def test_bucketed_tiles_and_tails(m, algo):
    # ragged tile tails, ranks that are not multiples of 4, a rank-1 edge,
    # an interior CP (diagonal) mode and Tucker factors, uint8 compaction
    rng = np.random.default_rng(m)
    nodes = [
        ("tt", rng.standard_normal((1, 5, 3)).astype(np.float32), None),
        ("cp", rng.standard_normal((7, 3)).astype(np.float32), rng.standard_normal((11, 7)).astype(np.float32)),
        ("tt", rng.standard_normal((3, 4, 1)).astype(np.float32), None),
        ("tt", rng.standard_normal((1, 6, 7)).astype(np.float32), rng.standard_normal((9, 6)).astype(np.float32)),
        ("tt", rng.standard_normal((7, 13, 2)).astype(np.float32), None),
        ("tt", rng.standard_normal((2, 3, 1)).astype(np.float32), None),
    ]
    t = facade(nodes)
    o = O.make_chain(nodes)
    idx = O.uniform_indices(t.shape, m, 5)
    idx[::3] -= np.asarray(t.shape)
    assert_close(tb.entries(t, idx, algo=algo), O.entries(o, idx), what=f"m={m}")
    bad = idx.copy()
    bad[m // 2, 4] = 13
    with pytest.raises(tb.ContractViolationError, match="mode 4"):
        tb.entries(t, bad, algo=algo)


@pytest.mark.parametrize("lane_major", ["1", "0"])
@pytest.mark.parametrize("r,J", [(8, 300), (16, 40), (24, 128), (32, 32), (32, 1024)])
def test_bucketed_rank_classes(r, J, lane_major, monkeypatch):
    # every register geometry (R = 8/16/24/32), the uint16 index path, and
    # core slices read from lane-major copies or from the repacked cores
    monkeypatch.setenv("TNB_LANE_MAJOR", lane_major)
    cores = O.random_tt((J, J, 5, J), r, seed=r + J, scale=r ** -0.5)
    t = facade([("tt", c, None) for c in cores])
    o = O.make_chain([("tt", c) for c in cores])
    idx = O.uniform_indices(t.shape, 20000, 1)
    assert_close(tb.entries(t, idx, algo=N.ALGO_BUCKETED), O.entries(o, idx), what=f"r={r} J={J}")


@pytest.mark.parametrize("generic", ["0", "1"])
def test_dot_rank16_fast_and_generic(generic, monkeypatch):
    # the rank-16 streaming kernel (dot_fast.cu) and the generic one agree
    # with the oracle; J=20 exercises a partial slice chunk
    monkeypatch.setenv("TNB_DOT_GENERIC", generic)
    a = O.random_tt((20,) * 5, 16, seed=3, batch_size=7, scale=0.25)
    b = O.random_tt((20,) * 5, 16, seed=4, batch_size=7, scale=0.25)
    ta, oa = facade([("tt", c, None) for c in a], 7), O.make_chain([("tt", c) for c in a], 7)
    tb_, ob = facade([("tt", c, None) for c in b], 7), O.make_chain([("tt", c) for c in b], 7)
    assert_close(tb.dot(ta, tb_), O.chain_dot(oa, ob), what="dot")
    assert_close(tb.norm(ta), O.norm(oa), what="norm")
    # unbatched rank-16 chains take the same kernel with one CTA
    a1 = O.random_tt((16,) * 3, 16, seed=5, scale=0.25)
    t1, o1 = facade([("tt", c, None) for c in a1]), O.make_chain([("tt", c) for c in a1])
    assert abs(tb.norm(t1) - O.norm(o1)) <= 1e-5 * O.norm(o1)


@pytest.mark.parametrize("codec,raw_frac", [("1", None), ("1", "0.35"), ("1", "0"), ("0", "0.35")])
def test_pipelined_host_indices_match_device_path(codec, raw_frac, monkeypatch):
    # a large pinned int64 host matrix takes the chunked copy/compute pipeline
    # (with and without the int8 index transport codec, some chunks raw or all
    # narrowed); per-sample results do not depend on chunking, tiling or the
    # codec (bitwise equal); raw_frac None = the self-balancing chunk order
    from paper_2206_11128_b200 import core as C

    monkeypatch.setenv("TNB_E2E_CODEC", codec)
    if raw_frac is None:  # the self-balancing pipeline (the default)
        monkeypatch.delenv("TNB_E2E_RAW_FRAC", raising=False)
    else:
        monkeypatch.setenv("TNB_E2E_RAW_FRAC", raw_frac)
    cores = O.random_tt((32,) * 6, 16, seed=11, scale=0.25)
    t = facade([("tt", c, None) for c in cores])
    assert C._codec_width(t) == (1 if codec == "1" else 0)
    m = 2 * C._PIPELINE_ROWS + 12345
    idx = torch.from_numpy(O.uniform_indices((32,) * 6, m, 3))
    idx[::3] -= 32  # negative indices cross the codec as negatives and wrap on the device
    idx = idx.pin_memory()
    got = tb.entries(t, idx)
    ref = tb.entries(t, idx.cuda())
    assert torch.equal(got, ref)
    o = O.make_chain([("tt", c) for c in cores])
    sel = np.arange(0, m, 997)
    assert_close(to_np(got)[sel], O.entries(o, idx.numpy()[sel]))
    bad = idx.clone()
    bad[m - 5, 4] = 40
    with pytest.raises(tb.ContractViolationError, match="mode 4"):
        tb.entries(t, bad.pin_memory())
    # values outside int8: that chunk crosses PCIe as int64, the other chunks
    # narrowed; the lowest offending mode is still reported
    bad = idx.clone()
    bad[7, 5] = 1000
    bad[C._PIPELINE_ROWS + 3, 2] = -33
    bad[C._PIPELINE_ROWS + 4, 1] = -(1 << 40)
    with pytest.raises(tb.ContractViolationError, match="mode 1"):
        tb.entries(t, bad.pin_memory())
    ok = idx.clone()
    ok[C._PIPELINE_ROWS + 9, 3] = -32  # the most negative valid index
    assert torch.equal(tb.entries(t, ok.pin_memory()), tb.entries(t, ok.cuda()))


def test_bucketed_cfg5_structure():
    # the R=24 lane-group geometry on the cfg5 structure (J=128 buckets)
    nodes = O.cfg5_nodes(seed=1)
    t = facade(nodes)
    o = O.make_chain(nodes)
    idx = O.uniform_indices((128,) * 8, 70000, 9)
    assert_close(tb.entries(t, idx, algo=N.ALGO_BUCKETED), O.entries(o, idx))


MERGE_CASES = {
    # prefix 0-2 and suffix 7-9 tables (cfg2 shape, smaller J)
    "tt10": lambda rng: [("tt", c, None) for c in O.random_tt((8,) * 10, 16, seed=7, scale=0.25)],
    # every mode merged into two tables (virtual chain of 2 modes)
    "two_tables": lambda rng: [("tt", c, None) for c in O.random_tt((8,) * 6, 8, seed=8, scale=0.35)],
    # CP modes inside the merged ranges, Tucker factors, ragged extents
    "hybrid": lambda rng: [
        ("tt", rng.standard_normal((1, 5, 6)).astype(np.float32), None),
        ("cp", rng.standard_normal((7, 6)).astype(np.float32), rng.standard_normal((9, 7)).astype(np.float32)),
        ("tt", rng.standard_normal((6, 6, 6)).astype(np.float32) * 0.4, None),
        ("tt", rng.standard_normal((6, 11, 6)).astype(np.float32) * 0.4, None),
        ("tt", rng.standard_normal((6, 3, 6)).astype(np.float32) * 0.4, None),
        ("cp", rng.standard_normal((4, 6)).astype(np.float32), None),
        ("tt", rng.standard_normal((6, 5, 1)).astype(np.float32), None),
    ],
    # cfg5 structure: prefix 0-1, CP suffix 6-7, CP 4-5 as a diagonal product
    # table folded into the last mode
    "cfg5": lambda rng: O.cfg5_nodes(seed=2),
    # no prefix/suffix (large extents); the interior CP run 2-4 becomes one
    # diagonal product table between two sorted modes
    "cp_run": lambda rng: [
        ("tt", rng.standard_normal((1, 200, 5)).astype(np.float32), None),
        ("tt", rng.standard_normal((5, 150, 5)).astype(np.float32) * 0.45, None),
        ("cp", rng.standard_normal((10, 5)).astype(np.float32), None),
        ("cp", rng.standard_normal((12, 5)).astype(np.float32), None),
        ("cp", rng.standard_normal((9, 5)).astype(np.float32), None),
        ("tt", rng.standard_normal((5, 160, 5)).astype(np.float32) * 0.45, None),
        ("tt", rng.standard_normal((5, 170, 1)).astype(np.float32), None),
    ],
}


@pytest.mark.parametrize("case", sorted(MERGE_CASES))
@pytest.mark.parametrize("merge", ["1", "0"])
def test_bucketed_mode_merging(case, merge, monkeypatch):
    # prefix/suffix tables over merged modes give the oracle's values; the
    # index checks still run per ORIGINAL mode (lowest bad mode reported)
    monkeypatch.setenv("TNB_ENTRIES_MERGE", merge)
    rng = np.random.default_rng(5)
    nodes = MERGE_CASES[case](rng)
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = 1 << 20 if case == "cfg5" else 300000
    idx = O.uniform_indices(t.shape, m, 3)
    idx[::5] -= np.asarray(t.shape)
    got = tb.entries(t, idx, algo=N.ALGO_BUCKETED)
    sel = np.arange(0, m, 7)
    assert_close(to_np(got)[sel], O.entries(o, idx[sel]), what=case)
    for k in (0, 1, t.ndim - 1):
        bad = idx.copy()
        bad[m // 3, k] = t.shape[k]
        bad[m // 2, t.ndim - 1] = -t.shape[t.ndim - 1] - 1
        with pytest.raises(tb.ContractViolationError, match=f"mode {k}"):
            tb.entries(t, bad, algo=N.ALGO_BUCKETED)


def test_entries_out_argument():
    # out= on the device or in pinned host memory (pipelined and direct paths)
    from paper_2206_11128_b200 import core as C

    cores = O.random_tt((16,) * 5, 8, seed=21, scale=0.4)
    t = facade([("tt", c, None) for c in cores])
    m = 2 * C._PIPELINE_ROWS + 777
    idx = torch.from_numpy(O.uniform_indices((16,) * 5, m, 4)).pin_memory()
    ref = tb.entries(t, idx.cuda())
    host = torch.empty(m, dtype=torch.float32).pin_memory()
    assert tb.entries(t, idx, out=host) is host
    assert torch.equal(host, ref.cpu())
    dev = torch.empty(m, dtype=torch.float32, device="cuda")
    assert tb.entries(t, idx, out=dev) is dev and torch.equal(dev, ref)
    small = idx[:1000].clone()
    h2 = torch.empty(1000, dtype=torch.float32).pin_memory()
    assert torch.equal(tb.entries(t, small, out=h2), tb.entries(t, small.cuda()).cpu())
    with pytest.raises(tb.ContractViolationError, match="pinned"):
        tb.entries(t, small, out=torch.empty(1000, dtype=torch.float32))
    with pytest.raises(tb.ContractViolationError, match="shape"):
        tb.entries(t, small, out=torch.empty(999, dtype=torch.float32).pin_memory())
    with pytest.raises(tb.ContractViolationError, match="float32"):
        tb.entries(t, small, out=torch.empty(1000, dtype=torch.float64).pin_memory())
    bad = idx.clone()
    bad[m - 3, 2] = 16
    with pytest.raises(tb.ContractViolationError, match="mode 2"):
        tb.entries(t, bad.pin_memory(), out=host)


@pytest.mark.parametrize("wide", ["1", "0"])
def test_bucketed_wide_tables(wide, monkeypatch):
    # prefix 0-3 and suffix 5-8 grow past 65535 rows (uint32 indices, tables in
    # HBM) when m allows; both ends wide, a CP mode inside the prefix, ragged m
    monkeypatch.setenv("TNB_MERGE_WIDE", wide)
    rng = np.random.default_rng(11)
    r = 8
    nodes = [("tt", rng.standard_normal((1, 16, r)).astype(np.float32) * 0.5, None),
             ("cp", rng.standard_normal((16, r)).astype(np.float32) * 0.7, None)]
    nodes += [("tt", rng.standard_normal((r, 16, r)).astype(np.float32) * 0.35, None) for _ in range(6)]
    nodes += [("tt", rng.standard_normal((r, 16, 1)).astype(np.float32) * 0.5, None)]
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = (1 << 20) + 123
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    if wide == "1":
        assert plan["prefix_rows"] == 16 ** 4 and plan["suffix_rows"] == 16 ** 4 and plan["n_virtual"] == 3
    else:
        assert plan["prefix_rows"] < 65536 and plan["suffix_rows"] < 65536
    idx = O.uniform_indices(t.shape, m, 21)
    idx[::7] -= np.asarray(t.shape)
    got = to_np(tb.entries(t, idx))
    sel = np.concatenate([np.arange(0, 4096), np.arange(m - 4096, m), np.arange(5000, m - 5000, 101)])
    assert_close(got[sel], O.entries(o, idx[sel]), what=f"wide={wide}")
    for k in (0, 3, 5, 8):  # OOB on modes inside the wide prefix / suffix
        bad = idx.copy()
        bad[m // 2, k] = t.shape[k]
        bad[m - 1, 8] = -17
        with pytest.raises(tb.ContractViolationError, match=f"mode {k}"):
            tb.entries(t, bad)


def _stream_nodes(rng, r, jl=5000):
    # prefix 0-2 (4096 rows), ONE sorted mode (J=300), the CP run 4-5 as a
    # diagonal table, a last mode too large to merge: P012 . G3 . D45 . L6
    s = r ** -0.5
    return [
        ("tt", rng.standard_normal((1, 8, r)).astype(np.float32), None),
        ("tt", (rng.standard_normal((r, 8, r)) * s).astype(np.float32), None),
        ("tt", (rng.standard_normal((r, 64, r)) * s).astype(np.float32), None),
        ("tt", (rng.standard_normal((r, 300, r)) * s).astype(np.float32), None),
        ("cp", rng.standard_normal((9, r)).astype(np.float32), None),
        ("cp", rng.standard_normal((7, r)).astype(np.float32), rng.standard_normal((11, 7)).astype(np.float32)),
        ("tt", (rng.standard_normal((r, jl, 1)) * s).astype(np.float32), None),
    ]


@pytest.mark.parametrize("r", [8, 16, 24])
@pytest.mark.parametrize("m", [300000, 70001])
def test_bucketed_stream_kernel(r, m, monkeypatch):
    # virtual chains with one sorted mode run the stream kernel (no state
    # array): per-warp TMA row rings running ahead across tiles, ragged tiles
    rng = np.random.default_rng(r)
    nodes = _stream_nodes(rng, r)
    t = facade(nodes)
    o = O.make_chain(nodes)
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert plan["compute_kernel"] == 1 and plan["n_virtual"] == 4, plan
    idx = O.uniform_indices(t.shape, m, 4)
    idx[::3] -= np.asarray(t.shape)
    got = to_np(tb.entries(t, idx))
    sel = np.concatenate([np.arange(0, 5000), np.arange(m - 3000, m), np.arange(5000, m - 3000, 13)])
    assert_close(got[sel], O.entries(o, idx[sel]), what=f"stream r={r}")
    monkeypatch.setenv("TNB_ENTRIES_STREAM", "0")
    assert N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)["compute_kernel"] == 0
    ref = to_np(tb.entries(t, idx))
    assert_close(got, ref.astype(np.float64), what="stream vs state kernel")
    monkeypatch.delenv("TNB_ENTRIES_STREAM")
    for k in (0, 3, 5, 6):  # OOB inside the prefix, the sorted mode, the CP table, the last mode
        bad = idx.copy()
        bad[m // 2, k] = t.shape[k]
        bad[m - 1, 6] = -t.shape[6] - 1
        with pytest.raises(tb.ContractViolationError, match=f"mode {k}"):
            tb.entries(t, bad)


def test_bucketed_stream_no_diag():
    # P012 . G3 . L4: no diagonal modes between the sorted and the last mode
    rng = np.random.default_rng(3)
    nodes = _stream_nodes(rng, 24)
    nodes = nodes[:4] + [nodes[6]]
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = 200000
    assert N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)["compute_kernel"] == 1
    idx = O.uniform_indices(t.shape, m, 5)
    sel = np.arange(0, m, 11)
    assert_close(to_np(tb.entries(t, idx))[sel], O.entries(o, idx[sel]), what="stream no diag")


@pytest.mark.parametrize("lane_major", ["1", "0"])
def test_bucketed_r32_tensor_core_paths(lane_major, monkeypatch):
    # an r = 32 sorted mode on tensor cores that reads the rows of a
    # (non-wide) prefix table itself and is followed by a CP mode, so the
    # closing dot is NOT fused (the CP row folds into the last mode);
    # lane_major=0 runs the FFMA2 K-split path on the same chain
    monkeypatch.setenv("TNB_LANE_MAJOR", lane_major)
    rng = np.random.default_rng(32)
    s = 32 ** -0.5
    nodes = [("tt", rng.standard_normal((1, 40, 32)).astype(np.float32), None),
             ("tt", (rng.standard_normal((32, 40, 32)) * s).astype(np.float32), None),
             ("tt", (rng.standard_normal((32, 40, 32)) * s).astype(np.float32), None),
             ("cp", rng.standard_normal((40, 32)).astype(np.float32), None),
             ("tt", (rng.standard_normal((32, 40, 1)) * s).astype(np.float32), None)]
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = 20001
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_BUCKETED)
    assert (plan["n_virtual"], plan["prefix_rows"], plan["compute_kernel"]) == (4, 1600, 0), plan
    idx = O.uniform_indices(t.shape, m, 7)
    idx[::9] -= np.asarray(t.shape)
    assert_close(tb.entries(t, idx, algo=N.ALGO_BUCKETED), O.entries(o, idx), what=f"r32 lane_major={lane_major}")
    bad = idx.copy()
    bad[m // 2, 2] = 40
    with pytest.raises(tb.ContractViolationError, match="mode 2"):
        tb.entries(t, bad, algo=N.ALGO_BUCKETED)


@pytest.mark.parametrize("three", [True, False])
@pytest.mark.parametrize("m", [1, 17, 1000, 4099])
def test_bucketed_stream_kernel_small_m(m, three):
    # forced bucketed algorithm at tiny sizes: one ragged 256-row tile, warps
    # with empty ranges, the producer's look-ahead past the last tile (the
    # 3-mode chain runs the stream kernel at every m, the 4-mode one switches
    # from the state kernel to the stream kernel once merging starts)
    rng = np.random.default_rng(m)
    nodes = _stream_nodes(rng, 24, jl=50)
    mid = ("tt", (rng.standard_normal((24, 300, 24)) * 24 ** -0.5).astype(np.float32), None)
    nodes = [nodes[0], mid, nodes[6]] if three else nodes[:2] + [mid, nodes[6]]
    t = facade(nodes)
    o = O.make_chain(nodes)
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_BUCKETED)
    idx = O.uniform_indices(t.shape, m, 5)
    got = tb.entries(t, idx, algo=N.ALGO_BUCKETED)
    assert_close(got, O.entries(o, idx), what=f"stream m={m} plan={plan}")


def test_bucketed_stream_kernel_few_buckets():
    # one sorted mode with only 40 buckets: the separate sort kernel (no sort
    # in prep) and a record that keeps the sorted mode's compact row (no key
    # packing) feed the stream kernel
    rng = np.random.default_rng(40)
    r = 24
    s_ = r ** -0.5
    nodes = [("tt", rng.standard_normal((1, 20000, r)).astype(np.float32), None),
             ("tt", (rng.standard_normal((r, 40, r)) * s_).astype(np.float32), None),
             ("tt", (rng.standard_normal((r, 5000, 1)) * s_).astype(np.float32), None)]
    t = facade(nodes)
    o = O.make_chain(nodes)
    m = 300001
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert (plan["compute_kernel"], plan["n_virtual"]) == (1, 3), plan
    idx = O.uniform_indices(t.shape, m, 6)
    idx[::5] -= np.asarray(t.shape)
    got = to_np(tb.entries(t, idx))
    sel = np.concatenate([np.arange(0, 3000), np.arange(m - 3000, m), np.arange(3000, m - 3000, 17)])
    assert_close(got[sel], O.entries(o, idx[sel]), what="stream few buckets")


@pytest.mark.parametrize("rank,batch", [(8, None), (24, None), (64, None), (16, 2)])
def test_full_tensor_core_gemm_ragged(rank, batch):
    # the final L @ R of full() on the tcgen05 path (M * N >= 2^20, N >= 128,
    # K <= 64) with neither M nor N a multiple of the 128-row tile or of the
    # 384-column resident block: partial row tiles, a partial n-block and an
    # n-block wholly past N (core.py:345-351)
    shape = (40, 37, 53, 29)
    cores = O.random_tt(shape, rank, seed=rank, batch_size=batch, scale=rank ** -0.5)
    t = facade([("tt", c, None) for c in cores], batch)
    o = O.make_chain([("tt", c) for c in cores], batch)
    assert_close(tb.full(t), O.full(o), what=f"full r{rank} b{batch}")
    assert_close(tb.full(t, lead=(3, 17)), O.full_slab(o, 3, 17), what=f"full slab r{rank} b{batch}")


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("batch", [None, 3])
def test_full_right_step_gemm_ragged(dtype, batch, monkeypatch):
    # split pinned at p=1 so the whole chain but mode 0 is the right partial:
    # mode 2's step (cols = 29 < 64) runs the per-output step kernel, mode 1's
    # (r_r = 8, cols = 2030) the tiled GEMM with the (j, a) -> (a, j) row
    # remap; gm_rows = 37 * 8 = 296 and cols = 2030 are not multiples of the
    # 128 x 128 tile (core.py:345-351)
    monkeypatch.setenv("TNB_FULL_SPLIT", "1")
    shape = (9, 37, 70, 29)
    cores = O.random_tt(shape, 8, seed=11, batch_size=batch, scale=8 ** -0.5)
    o = O.make_chain([("tt", c) for c in cores], batch)
    dt = torch.float64 if dtype == "f64" else torch.float32
    t = tb.TnTensor([tb.ModeNode("tt", c, batched=batch is not None, dtype=dt) for c in cores], batch)
    ref = O.full(o)
    got = tb.full(t)
    if dtype == "f64":
        err = np.abs(to_np(got) - ref).max() / np.abs(ref).max()
        assert err <= 1e-12, err
    else:
        assert_close(got, ref, what=f"right-step gemm b{batch}")
    assert_close(tb.full(t, lead=(2, 7)), O.full_slab(o, 2, 7), what="right-step gemm slab")


def test_full_tall_thin_generic_gemm(monkeypatch):
    # an fp32 chain of shape (2^24, 2) split at p=1 has 2^24 rows
    # of L and N=2 columns (no tensor-core GEMM), i.e. 131072 row tiles: more
    # than the 65535 a grid's y axis holds
    monkeypatch.setenv("TNB_FULL_SPLIT", "1")
    rng = np.random.default_rng(5)
    nodes = [("tt", rng.standard_normal((1, 1 << 24, 3)).astype(np.float32), None),
             ("tt", rng.standard_normal((3, 2, 1)).astype(np.float32), None)]
    t = facade(nodes)
    got = to_np(tb.full(t))
    a, b = nodes[0][1][0].astype(np.float64), nodes[1][1][:, :, 0].astype(np.float64)
    sel = np.r_[0:4096, (1 << 24) - 4096:(1 << 24)]
    assert_close(got[sel], a[sel] @ b, what="tall thin full")


@pytest.mark.parametrize("batch,shape,rank,m", [
    (3, (32,) * 6, 32, (1 << 16) + 5),      # state kernel, r=32 tensor-core modes, merged tables
    (5, (16,) * 7, 16, 70001),              # state kernel, R=16
    (2, (2048, 40, 2048), 24, 1 << 17),     # stream kernel
    (4, (32,) * 10, 32, 1 << 18),           # the cfg2 chain shape
])
def test_batched_bucketed_entries(batch, shape, rank, m):
    # _step_entries_batched (core.py:447-460) on the bucketed path: output
    # [m, B]; every element's column equals the unbatched chain of that
    # element, bitwise (same kernels, same plan)
    cores = O.random_tt(shape, rank, seed=rank + batch, batch_size=batch, scale=rank ** -0.5)
    t = facade([("tt", c, None) for c in cores], batch)
    o = O.make_chain([("tt", c) for c in cores], batch)
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert plan["algo"] == N.ALGO_BUCKETED, plan
    idx = O.uniform_indices(shape, m, 21)
    idx[::9] -= np.asarray(shape)
    got = tb.entries(t, idx)
    assert tuple(got.shape) == (m, batch)
    sel = np.arange(0, m, max(1, m // 4000))
    assert_close(to_np(got)[sel], O.entries(o, idx[sel]), what=f"batched bucketed B={batch}")
    dev_idx = torch.from_numpy(idx).cuda()
    for b in (0, batch - 1):
        tb1 = facade([("tt", c[b], None) for c in cores])
        assert torch.equal(got[:, b], tb.entries(tb1, dev_idx)), b
    bad = idx.copy()
    bad[m // 2, 1] = shape[1]
    with pytest.raises(tb.ContractViolationError, match="mode 1"):
        tb.entries(t, bad)


@pytest.mark.parametrize("rank", [5, 8, 24, 32, 40])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_dot_norm_rank_general(rank, dtype):
    # chains of ranks other than 16 (the mma.sync kernel's) on the chunked
    # kernel (16-byte staged slices; rank 5 takes the scalar rows, 40 the
    # one-slice chunks); core.py:362-391
    batch = 37
    a = O.random_tt((24, 17, 33, 9, 20), rank, seed=rank, batch_size=batch, scale=rank ** -0.5)
    b = O.random_tt((24, 17, 33, 9, 20), rank + 1, seed=rank + 1, batch_size=batch, scale=(rank + 1) ** -0.5)
    dt = torch.float64 if dtype == "f64" else torch.float32
    ta = tb.TnTensor([tb.ModeNode("tt", c, batched=True, dtype=dt) for c in a], batch)
    tb_ = tb.TnTensor([tb.ModeNode("tt", c, batched=True, dtype=dt) for c in b], batch)
    oa, ob = O.make_chain([("tt", c) for c in a], batch), O.make_chain([("tt", c) for c in b], batch)
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert_dot_close(tb.dot(ta, tb_), O.chain_dot(oa, ob), O.norm(oa) * O.norm(ob), tol=tol, what=f"dot r{rank}")
    assert_close(tb.norm(ta), O.norm(oa), tol=tol, what=f"norm r{rank}")
    u = tb.TnTensor([tb.ModeNode("tt", c[3], dtype=dt) for c in a])
    ou = O.make_chain([("tt", c[3]) for c in a])
    assert abs(tb.norm(u) - O.norm(ou)) <= tol * O.norm(ou)


@pytest.mark.parametrize("case", ["cfg3_r64", "two_modes", "cp_ends", "odd_rank", "negatives"])
def test_two_table_entries(case):
    # chains whose mode merging leaves a prefix and a suffix table: the fused
    # two-table kernel, any rank (core.py:394-444)
    rng = np.random.default_rng(31)
    if case == "cfg3_r64":
        cores = O.random_tt((256,) * 4, 64, seed=0, scale=64 ** -0.5)
        nodes = [("tt", c, None) for c in cores]
        m = 1 << 20
    elif case == "two_modes":
        nodes = [("tt", rng.standard_normal((1, 3000, 48)).astype(np.float32), None),
                 ("tt", rng.standard_normal((48, 2500, 1)).astype(np.float32), None)]
        m = 1 << 16
    elif case == "cp_ends":
        nodes = [("cp", rng.standard_normal((40, 12)).astype(np.float32), rng.standard_normal((70, 40)).astype(np.float32)),
                 ("tt", (rng.standard_normal((12, 30, 12)) * 0.3).astype(np.float32), None),
                 ("cp", rng.standard_normal((50, 12)).astype(np.float32), None)]
        m = 100003
    elif case == "odd_rank":
        cores = O.random_tt((64, 30, 64), 37, seed=3, scale=37 ** -0.5)
        nodes = [("tt", c, None) for c in cores]
        m = 70001
    else:
        cores = O.random_tt((16,) * 6, 8, seed=4, scale=8 ** -0.5)
        nodes = [("tt", c, None) for c in cores]
        m = 1 << 17
    t = facade(nodes)
    o = O.make_chain(nodes)
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert (plan["compute_kernel"], plan["n_virtual"]) == (2, 2), plan
    idx = O.uniform_indices(t.shape, m, 7)
    idx[::3] -= np.asarray(t.shape)
    got = to_np(tb.entries(t, idx))
    sel = np.arange(0, m, max(1, m // 5000))
    assert_close(got[sel], O.entries(o, idx[sel]), what=case)
    for k in range(t.ndim):
        bad = idx.copy()
        bad[m // 2, k] = t.shape[k]
        bad[m // 3, t.ndim - 1] = -t.shape[-1] - 1
        with pytest.raises(tb.ContractViolationError, match=f"mode {min(k, t.ndim - 1)}"):
            tb.entries(t, bad)


@pytest.mark.parametrize("case", ["state_r32", "stream_cfg5"])
@pytest.mark.parametrize("pattern", ["prefix_fixed", "all_same", "half_same"])
def test_bucketed_repeated_first_rows(case, pattern):
    # slice queries: every sample shares its first-mode (prefix-table) row --
    # detect_hot_kernel flags the call and the compute kernels' rings copy
    # through L1; results identical in value to the oracle (core.py:394-444)
    if case == "state_r32":
        cores = O.random_tt((32,) * 6, 32, seed=2, scale=32 ** -0.5)
        nodes = [("tt", c, None) for c in cores]
        m = (1 << 17) + 3
    else:
        nodes = O.cfg5_nodes(seed=4)
        m = 1 << 18
    t = facade(nodes)
    o = O.make_chain(nodes)
    idx = O.uniform_indices(t.shape, m, 12)
    if pattern == "prefix_fixed":
        idx[:, : t.ndim // 2] = idx[0, : t.ndim // 2]
    elif pattern == "all_same":
        idx[:] = idx[5]
    else:
        idx[::2, :3] = idx[0, :3]
    got = to_np(tb.entries(t, idx))
    sel = np.arange(0, m, 61)
    assert_close(got[sel], O.entries(o, idx[sel]), what=f"{case} {pattern}")


@pytest.mark.parametrize("case", ["cfg2_like", "cfg5_structure"])
def test_table_levels_on_tcgen05(case, monkeypatch):
    # TNB_TABLE_TCGEN05=1: large dense prefix table levels as one tcgen05
    # 3xTF32 GEMM against a transposed core (off by default: SM contention
    # with the overlapped prep); values within the fp32 bar of the oracle
    monkeypatch.setenv("TNB_TABLE_TCGEN05", "1")
    if case == "cfg2_like":
        cores = O.random_tt((32,) * 8, 32, seed=9, scale=32 ** -0.5)
        nodes = [("tt", c, None) for c in cores]
        m = 1 << 21
    else:
        nodes = O.cfg5_nodes(seed=6)
        m = 1 << 24  # the 2^21-row P012 table (its second level is a tcgen05 GEMM)
    t = facade(nodes)
    o = O.make_chain(nodes)
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert plan["prefix_rows"] >= 1 << 15, plan
    idx = O.uniform_indices(t.shape, m, 14)
    got = to_np(tb.entries(t, torch.from_numpy(idx).cuda()))
    sel = np.arange(0, m, m // 20000)
    assert_close(got[sel], O.entries(o, idx[sel]), what=case)


@pytest.mark.parametrize("rank", [8, 24, 32, 48])
@pytest.mark.parametrize("batch", [1, 37, 300])
def test_dot_norm_tensor_core_ranks(rank, batch):
    # uniform-rank TT chains of ranks 8 / 32 / 48 on the mma.sync (24: chunked)
    # split-TF32 kernel (dot_mma.cu): staged chunks, padded split rows, Y and
    # A^T Y products on tensor cores (core.py:362-391)
    shape = (24, 17, 33, 9, 20, 5)
    a = O.random_tt(shape, rank, seed=rank, batch_size=batch, scale=rank ** -0.5)
    b = O.random_tt(shape, rank, seed=rank + 100, batch_size=batch, scale=rank ** -0.5)
    ta = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in a], batch)
    tb_ = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in b], batch)
    oa, ob = O.make_chain([("tt", c) for c in a], batch), O.make_chain([("tt", c) for c in b], batch)
    assert_dot_close(tb.dot(ta, tb_), O.chain_dot(oa, ob), O.norm(oa) * O.norm(ob), what=f"dot r{rank}")
    assert_close(tb.norm(ta), O.norm(oa), what=f"norm r{rank}")
    # self-dot = norm^2 on the same kernel
    d = to_np(tb.dot(ta, ta))
    n = to_np(tb.norm(ta))
    assert np.all(np.abs(d - n * n) <= 1e-5 * n * n)
