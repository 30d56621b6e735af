"""Out-of-bounds write checks for every fast kernel (compute-sanitizer is
closed on this GPU pool: profiles/r02_sanitizer_closed.txt).  Each kernel
runs through the C ABI on buffers embedded in larger allocations whose
margins hold a sentinel pattern -- output, workspace and index buffers --
and the margins must come back untouched, on shapes that exercise ragged
tiles, short last tiles and partial warps.  Results are checked against the
oracle as usual."""

import ctypes

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests.helpers import assert_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
tb = pytest.importorskip("paper_2206_11128_b200")
from paper_2206_11128_b200 import _native as N  # noqa: E402

PAD = 4096  # bytes of margin on each side
SENT = 0x5A


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(autouse=True)
def _bucketed_auto(monkeypatch):
    # this module pins the bucketed / generic kernels: AUTO must not route
    # large calls to the global-sort path (tests/test_gpu_gsort.py covers it)
    monkeypatch.setenv("TNB_ENTRIES_GSORT", "0")


class Guarded:
    """nbytes usable device bytes at a 256-byte aligned offset inside a
    buffer whose PAD-byte margins hold SENT."""

    def __init__(self, nbytes):
        self.n = max(int(nbytes), 1)
        self.raw = torch.full((self.n + 2 * PAD,), SENT, dtype=torch.uint8, device="cuda")
        self.ptr = self.raw.data_ptr() + PAD

    def view(self, dtype, count):
        return self.raw[PAD:PAD + count * torch.tensor([], dtype=dtype).element_size()].view(dtype)

    def check(self, what):
        torch.cuda.synchronize()
        lo, hi = self.raw[:PAD], self.raw[PAD + self.n:]
        assert bool((lo == SENT).all()), f"{what}: write before the buffer"
        assert bool((hi == SENT).all()), f"{what}: write past the buffer"


def _entries_guarded(t, idx_np, algo=N.ALGO_AUTO):
    p = t._packed()
    lib = N.load()
    m = idx_np.shape[0]
    gi = Guarded(idx_np.nbytes)
    gi.view(torch.int64, idx_np.size).copy_(torch.from_numpy(idx_np.reshape(-1)))
    go = Guarded(4 * m)
    ge = Guarded(4)
    wsb = lib.tnb_entries_workspace_bytes(ctypes.byref(p.chain), m, algo)
    gw = Guarded(wsb)
    N.check(lib.tnb_entries_f32(ctypes.byref(p.chain), gi.ptr, m, go.ptr, ge.ptr, algo,
                                gw.ptr if wsb > 0 else None, wsb, N.stream_ptr(p.device)), "entries")
    for g, w in ((gi, "idx"), (go, "out"), (ge, "err"), (gw, "workspace")):
        g.check(f"entries {w}")
    assert int(ge.view(torch.int32, 1).item()) >= t.ndim
    return go.view(torch.float32, m).clone()


@pytest.mark.parametrize("m", [1, 31, 1000, (1 << 16) + 17])
def test_guard_state_kernel(m):
    cores = O.random_tt((32,) * 6, 32, seed=7, scale=32 ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    idx = O.uniform_indices(t.shape, m, 8)
    got = _entries_guarded(t, idx)
    sel = np.arange(0, m, max(1, m // 3000))
    assert_close(got.cpu().numpy()[sel], O.entries(O.make_chain([("tt", c) for c in cores]), idx[sel]))


@pytest.mark.parametrize("m", [7, 5000, (1 << 17) + 3])
def test_guard_stream_kernel(m):
    rng = np.random.default_rng(9)
    cores = [rng.standard_normal(s).astype(np.float32) * 24 ** -0.5
             for s in ((1, 2048, 24), (24, 40, 24), (24, 2048, 1))]
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    idx = O.uniform_indices(t.shape, m, 10)
    got = _entries_guarded(t, idx)
    sel = np.arange(0, m, max(1, m // 3000))
    assert_close(got.cpu().numpy()[sel], O.entries(O.make_chain([("tt", c) for c in cores]), idx[sel]))


@pytest.mark.parametrize("m", [1, 129, 70001, (1 << 18) + 5])
def test_guard_gsort_kernels(m, monkeypatch):
    # global-sort path: prep / scan / scatter / tcgen05 compute with ragged
    # bucket tails and empty buckets (P01 . G23 . S45 of an 8^6 chain, r = 16)
    monkeypatch.setenv("TNB_PREFIX_MAX_ROWS", "64")
    monkeypatch.setenv("TNB_SUFFIX_MAX_ROWS", "64")
    cores = O.random_tt((8,) * 6, 16, seed=17, scale=0.25)
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    idx = O.uniform_indices(t.shape, m, 4)
    idx[::5] -= 8
    assert N.entries_plan(t._packed().chain, m, N.ALGO_GSORT)["compute_kernel"] == 3
    got = _entries_guarded(t, idx, N.ALGO_GSORT)
    sel = np.arange(0, m, max(1, m // 3000))
    assert_close(got.cpu().numpy()[sel], O.entries(O.make_chain([("tt", c) for c in cores]), idx[sel]))


@pytest.mark.parametrize("t5", ["1", "0"])
def test_guard_table_levels(t5, monkeypatch):
    # table levels with 4913 input rows (ragged against the 128-row tiles), 17
    # slices (groups of 8, 8, 1) and rank 12 (zero-padded k-steps): the tcgen05
    # level kernel (TNB_TABLE_T5=1) and the mma.sync / SIMT kernels it replaces
    monkeypatch.delenv("TNB_ENTRIES_GSORT", raising=False)
    monkeypatch.setenv("TNB_TABLE_T5", t5)
    cores = O.random_tt((17,) * 9, 12, seed=23, scale=12 ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    m = 1 << 20
    plan = N.entries_plan(t._packed().chain, m, N.ALGO_AUTO)
    assert (plan["prefix_rows"], plan["suffix_rows"]) == (17 ** 4, 17 ** 4), plan
    idx = O.uniform_indices(t.shape, m, 6)
    idx[::9] -= 17
    got = _entries_guarded(t, idx)
    sel = np.arange(0, m, 331)
    assert_close(got.cpu().numpy()[sel], O.entries(O.make_chain([("tt", c) for c in cores]), idx[sel]))


def test_guard_cfg5_structure():
    nodes = O.cfg5_nodes(seed=2)
    t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in nodes])
    idx = O.uniform_indices(t.shape, 200003, 3)
    got = _entries_guarded(t, idx)
    sel = np.arange(0, 200003, 67)
    assert_close(got.cpu().numpy()[sel], O.entries(O.make_chain(nodes), idx[sel]))


@pytest.mark.parametrize("shape,rank,lead", [((40, 37, 53, 29), 16, None), ((128, 96, 130), 16, None),
                                             ((9, 37, 70, 29), 8, (2, 7)), ((256, 64, 256), 64, (3, 200))])
def test_guard_full(shape, rank, lead):
    cores = O.random_tt(shape, rank, seed=4, scale=rank ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    p = t._packed()
    lib = N.load()
    lo, hi = lead or (0, shape[0])
    n_out = (hi - lo) * int(np.prod(shape[1:]))
    go = Guarded(4 * n_out)
    wsb = lib.tnb_full_workspace_bytes(ctypes.byref(p.chain), lo, hi)
    gw = Guarded(wsb)
    N.check(lib.tnb_full_f32(ctypes.byref(p.chain), lo, hi, go.ptr, gw.ptr, wsb, N.stream_ptr(p.device)), "full")
    go.check("full out")
    gw.check("full workspace")
    ref = O.full_slab(O.make_chain([("tt", c) for c in cores]), lo, hi)
    assert_close(go.view(torch.float32, n_out).reshape(ref.shape), ref, what=f"full {shape}")


@pytest.mark.parametrize("batch", [1, 5, 37])
def test_guard_dot_norm(batch):
    a = O.random_tt((16,) * 5, 16, seed=13, batch_size=batch, scale=0.25)
    b = O.random_tt((16,) * 5, 16, seed=14, batch_size=batch, scale=0.25)
    ta = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in a], batch)
    tb_ = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in b], batch)
    pa, pb = ta._packed(), tb_._packed()
    lib = N.load()
    gd, gn = Guarded(4 * batch), Guarded(4 * batch)
    N.check(lib.tnb_dot_f32(ctypes.byref(pa.chain), ctypes.byref(pb.chain), gd.ptr, N.stream_ptr(pa.device)), "dot")
    N.check(lib.tnb_norm_f32(ctypes.byref(pa.chain), gn.ptr, N.stream_ptr(pa.device)), "norm")
    gd.check("dot out")
    gn.check("norm out")
    oa, ob = O.make_chain([("tt", c) for c in a], batch), O.make_chain([("tt", c) for c in b], batch)
    scale = O.norm(oa) * O.norm(ob)
    d = gd.view(torch.float32, batch).double().cpu().numpy()
    assert np.all(np.abs(d - O.chain_dot(oa, ob)) <= 1e-5 * scale)
    assert_close(gn.view(torch.float32, batch), O.norm(oa), what="norm")


def test_guard_widen():
    lib = N.load()
    for count in (1, 2, 17, 1000003):
        src = torch.randint(-128, 128, (count,), dtype=torch.int8)
        gi, go = Guarded(count), Guarded(8 * count)
        gi.view(torch.int8, count).copy_(src)
        N.check(lib.tnb_widen_indices(gi.ptr, 1, count, go.ptr, N.stream_ptr(torch.device("cuda", 0))), "widen")
        gi.check("widen in")
        go.check("widen out")
        assert torch.equal(go.view(torch.int64, count).cpu(), src.long())
