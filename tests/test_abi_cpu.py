"""CPU-side checks of the boundary: libtnb.so loads, exports exactly the
symbols include/tnb.h declares, and the host-side contract (validation,
planning, error mapping) behaves like the reference without a GPU."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2206_11128_b200 import _build, _native

    if not _native.LIB_PATH.exists():
        _build.build(verbose=False)
    return _native.load()


def declared_symbols():
    text = (ROOT / "include" / "tnb.h").read_text()
    return sorted(set(re.findall(r"\b(tnb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("tnb_entries_f32", "tnb_full_f32", "tnb_dot_f32", "tnb_norm_f32", "tnb_repack_f32"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2206_11128_b200 import _native

    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} lacks a ctypes signature"
    assert set(_native.SIGNATURES) == set(declared_symbols())
    assert lib.tnb_version().startswith(b"tnb")


def test_struct_layouts_match_header():
    from paper_2206_11128_b200 import _native as N

    assert ctypes.sizeof(N.TnbNode) == 40
    assert ctypes.sizeof(N.TnbMode) == 24
    assert ctypes.sizeof(N.TnbChain) == 24


def _plan(lib, specs):
    from paper_2206_11128_b200 import _native as N

    n = len(specs)
    nodes = (N.TnbNode * n)()
    for k, (kind, I, J, rl, rr) in enumerate(specs):
        nodes[k].kind, nodes[k].internal, nodes[k].phys = kind, I, J
        nodes[k].r_left, nodes[k].r_right = rl, rr
        nodes[k].core = 1  # never dereferenced by planning
        nodes[k].factor = 1 if I != J else None
    modes = (N.TnbMode * n)()
    rc = lib.tnb_plan_modes(nodes, n, modes)
    return rc, modes


def test_plan_promotes_cp_by_position(lib):
    from paper_2206_11128_b200 import _native as N

    rc, modes = _plan(lib, [(N.KIND_CP, 4, 4, 3, 3), (N.KIND_CP, 5, 7, 3, 3), (N.KIND_TT, 6, 6, 3, 2),
                            (N.KIND_CP, 2, 2, 2, 2)])
    assert rc == 0
    got = [(m.layout, m.phys, m.r_left, m.r_right) for m in modes]
    assert got == [(N.LAYOUT_DENSE, 4, 1, 3), (N.LAYOUT_DIAG, 7, 3, 3),
                   (N.LAYOUT_DENSE, 6, 3, 2), (N.LAYOUT_DENSE, 2, 2, 1)]
    assert lib.tnb_mode_floats(ctypes.byref(modes[1]), 0) == 7 * 3
    assert lib.tnb_mode_floats(ctypes.byref(modes[2]), 5) == 5 * 6 * 3 * 2
    rc, modes = _plan(lib, [(N.KIND_CP, 5, 5, 3, 3)])
    assert rc == 0 and (modes[0].r_left, modes[0].r_right) == (1, 1)


def test_plan_rejects_bad_chains(lib):
    from paper_2206_11128_b200 import _native as N

    rc, _ = _plan(lib, [(N.KIND_TT, 3, 3, 1, 2), (N.KIND_TT, 4, 4, 3, 1)])
    assert rc == N.TNB_EINVAL and b"rank mismatch between modes 0 and 1" in lib.tnb_last_error()
    rc, _ = _plan(lib, [(N.KIND_TT, 3, 3, 2, 1)])
    assert rc == N.TNB_EINVAL and b"boundary ranks must be 1" in lib.tnb_last_error()


def test_workspace_queries(lib):
    from paper_2206_11128_b200 import _native as N

    _, modes = _plan(lib, [(N.KIND_TT, 16, 16, 1, 8), (N.KIND_TT, 16, 16, 8, 8), (N.KIND_TT, 16, 16, 8, 1)])
    ch = N.TnbChain(3, 0, 0, ctypes.cast(modes, ctypes.POINTER(N.TnbMode)))
    assert lib.tnb_entries_workspace_bytes(ctypes.byref(ch), 1000, N.ALGO_CHAIN) == 0
    assert lib.tnb_entries_workspace_bytes(ctypes.byref(ch), 1000, N.ALGO_LAYERED) == 2 * 1000 * 8 * 4
    assert lib.tnb_full_workspace_bytes(ctypes.byref(ch), 0, 16) >= 0
    assert lib.tnb_full_workspace_bytes(ctypes.byref(ch), 0, 17) == -1


# -- façade validation mirrors the reference (no GPU needed) ---------------

def test_facade_validation_messages():
    import paper_2206_11128_b200 as tb

    with pytest.raises(tb.ContractViolationError):
        tb.ModeNode("xx", np.ones((1, 2, 1)))
    with pytest.raises(tb.StructuralError, match="3 axes"):
        tb.ModeNode("tt", np.ones((2, 2)))
    with pytest.raises(tb.StructuralError, match="internal size"):
        tb.ModeNode("tt", np.ones((1, 3, 1)), factor=np.ones((5, 2)))
    with pytest.raises(tb.StructuralError, match="rank mismatch between modes 0 and 1"):
        tb.TnTensor([tb.ModeNode("tt", np.ones((1, 3, 2))), tb.ModeNode("tt", np.ones((3, 4, 1)))])
    with pytest.raises(tb.StructuralError, match="boundary ranks"):
        tb.TnTensor([tb.ModeNode("tt", np.ones((2, 3, 1)))])
    with pytest.raises(tb.StructuralError):
        tb.TnTensor([tb.ModeNode("cp", np.ones((3, 2))), tb.ModeNode("tt", np.ones((3, 4, 1)))])
    with pytest.raises(tb.ContractViolationError):
        tb.TnTensor([])
    good = tb.ModeNode("tt", np.ones((2, 1, 3, 1)), batched=True)
    with pytest.raises(tb.StructuralError):
        tb.TnTensor([good], batch_size=3)
    with pytest.raises(tb.StructuralError):
        tb.TnTensor([tb.ModeNode("tt", np.ones((1, 3, 1)))], batch_size=2)
    assert issubclass(tb.ContractViolationError, ValueError)
    assert issubclass(tb.StructuralError, ValueError)


def test_facade_metadata():
    import paper_2206_11128_b200 as tb

    t = tb.TnTensor([tb.ModeNode("cp", np.ones((3, 5))), tb.ModeNode("cp", np.ones((4, 5)), np.ones((6, 4))),
                     tb.ModeNode("tt", np.ones((5, 2, 1)))])
    assert t.shape == (3, 6, 2) and t.ranks == [1, 5, 5, 1] and t.ndim == 3
    assert t.numel() == 36 and t.dof() == 15 + 20 + 24 + 10
    assert "kinds=CCT" in repr(t)


def test_no_cpu_fallback():
    import torch

    import paper_2206_11128_b200 as tb

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = tb.TnTensor([tb.ModeNode("tt", np.ones((1, 3, 1)))])
    with pytest.raises(tb.NativeError):
        tb.full(t)
    with pytest.raises(tb.NativeError):
        t[np.zeros((1, 1), dtype=np.int64)]


def _chain(specs):
    """tnb_chain over (layout, J, r_l, r_r) specs with dummy slice pointers
    (plan queries never touch device memory)."""
    from paper_2206_11128_b200 import _native as N

    modes = (N.TnbMode * len(specs))()
    for k, (lay, J, rl, rr) in enumerate(specs):
        modes[k].layout, modes[k].phys, modes[k].r_left, modes[k].r_right = lay, J, rl, rr
        modes[k].slices = 0x1000
    ch = N.TnbChain()
    ch.n_modes, ch.batch, ch.modes = len(specs), 0, modes
    ch._keep = modes
    return ch


def test_entries_plan_merges_cfg2_and_cfg5(lib, monkeypatch):
    from paper_2206_11128_b200 import _native as N

    monkeypatch.delenv("TNB_ENTRIES_MERGE", raising=False)
    monkeypatch.delenv("TNB_ENTRIES_GSORT", raising=False)
    r = 32
    specs = [(0, 32, 1, r)] + [(0, 32, r, r)] * 8 + [(0, 32, r, 1)]
    # cfg2 at 2^24 tuples, AUTO: the global-sort tcgen05 path -- prefix 0-3
    # and suffix 6-9 tables, modes 4-5 merged into ONE sorted mode of 1024
    # slices: one r x r product (3 tf32 MMAs) + the closing dot per entry
    g = N.entries_plan(_chain(specs), 1 << 24)
    assert (g["algo"], g["compute_kernel"], g["tile"], g["n_virtual"]) == (N.ALGO_GSORT, 3, 128, 3), g
    assert (g["prefix_modes"], g["suffix_modes"]) == (4, 4) and g["prefix_rows"] == g["suffix_rows"] == 32 ** 4
    assert g["kernel_flops"] == (2 * r * r + 2 * r) * float(1 << 24)
    assert g["tensor_flops"] == 3 * 2 * r * r * float(1 << 24)
    # tables P0123, S6789 and the merged level G4 G5 (32 * 32 rows of G4 against the 32 slices of G5)
    assert g["table_flops"] == 2 * (32 ** 2 + 32 ** 3 + 32 ** 4) * r * 2 * r + (32 * r) * 32 * r * 2 * r
    # below 2^20 tuples the tables stop at 2^15 rows and four interior modes
    # (2^20 slices) do not merge: the bucketed kernels
    assert N.entries_plan(_chain(specs), 1 << 19)["algo"] == N.ALGO_BUCKETED
    # from 2^20 tuples the merge may use tables of up to m rows so that one sort suffices
    for lg in (20, 21):
        gm = N.entries_plan(_chain(specs), 1 << lg)
        assert (gm["algo"], gm["prefix_rows"], gm["suffix_rows"]) == (N.ALGO_GSORT, 32 ** 4, 32 ** 4), gm
    # the explicit algorithm needs a supported chain (rank multiples of 4)
    odd = [(0, 32, 1, 5), (0, 32, 5, 5), (0, 32, 5, 5), (0, 32, 5, 1)]
    with pytest.raises(Exception):
        N.entries_plan(_chain(odd), 1 << 20, N.ALGO_GSORT)
    # TNB_ENTRIES_GSORT=0: the bucketed kernels, as before the global sort
    monkeypatch.setenv("TNB_ENTRIES_GSORT", "0")
    # cfg2: 10 x TT, J=32, r=32, m=2^24 -> wide (HBM) prefix 0-3 and suffix
    # 6-9 tables of 2^20 rows: two sorted modes remain
    info = N.entries_plan(_chain(specs), 1 << 24)
    assert info["algo"] == N.ALGO_BUCKETED
    assert (info["prefix_modes"], info["suffix_modes"], info["n_virtual"]) == (4, 4, 4)
    assert info["prefix_rows"] == info["suffix_rows"] == 32 ** 4
    # virtual chain: 2 dense r x r steps + closing dot
    assert info["kernel_flops"] == (2 * 2 * r * r + 2 * r) * float(1 << 24)
    # without wide tables: 16-bit indexed L2 tables over modes 0-2 and 7-9
    monkeypatch.setenv("TNB_MERGE_WIDE", "0")
    info = N.entries_plan(_chain(specs), 1 << 24)
    assert (info["prefix_modes"], info["suffix_modes"], info["n_virtual"]) == (3, 3, 6)
    assert info["prefix_rows"] == info["suffix_rows"] == 32 ** 3
    assert info["kernel_flops"] == (4 * 2 * r * r + 2 * r) * float(1 << 24)
    assert info["table_flops"] == 2 * (32 ** 2 * r * 2 * r + 32 ** 3 * r * 2 * r)
    monkeypatch.delenv("TNB_MERGE_WIDE")
    # cfg5: TT 0-3 (r=24), CP 4-7 (diag interior, dense right end), J=128;
    # a single interior mode is left after merging, so AUTO keeps the stream
    # kernel with or without the global-sort path
    specs5 = [(0, 128, 1, 24)] + [(0, 128, 24, 24)] * 3 + [(1, 128, 24, 24)] * 3 + [(0, 128, 24, 1)]
    monkeypatch.delenv("TNB_ENTRIES_GSORT")
    assert N.entries_plan(_chain(specs5), 1 << 26)["compute_kernel"] == 1
    g5 = N.entries_plan(_chain(specs5), 1 << 26, N.ALGO_GSORT)
    assert (g5["compute_kernel"], g5["n_virtual"], g5["diag_tables"], g5["prefix_rows"]) == (3, 4, 1, 128 ** 3), g5
    monkeypatch.setenv("TNB_ENTRIES_GSORT", "0")
    info5 = N.entries_plan(_chain(specs5), 1 << 26)
    # wide prefix 0-2 (2^21 rows), CP suffix 6-7 (16384 rows), CP 4-5 as one
    # diagonal product table: virtual chain P012, G3, D45, S67
    assert (info5["prefix_modes"], info5["suffix_modes"], info5["n_virtual"]) == (3, 2, 4)
    assert info5["prefix_rows"] == 128 ** 3 and info5["diag_tables"] == 1
    assert info5["kernel_flops"] == (2 * 24 * 24 + 24 + 2 * 24) * float(1 << 26)
    # one sorted mode left: the stream kernel (4096-sample tiles); cfg2 keeps
    # the state kernel (two sorted modes)
    assert (info5["compute_kernel"], info5["tile"]) == (1, 6144)
    assert N.entries_plan(_chain(specs), 1 << 24)["compute_kernel"] == 0
    monkeypatch.setenv("TNB_ENTRIES_STREAM", "0")
    assert N.entries_plan(_chain(specs5), 1 << 26)["compute_kernel"] == 0
    monkeypatch.delenv("TNB_ENTRIES_STREAM")
    # the GPU stream tests' chain (tests/test_gpu_parity.py::_stream_nodes)
    for rr in (8, 16, 24):
        st = [(0, 8, 1, rr), (0, 8, rr, rr), (0, 64, rr, rr), (0, 300, rr, rr), (1, 9, rr, rr), (1, 11, rr, rr),
              (0, 5000, rr, 1)]
        for mm in (300000, 70001):
            i = N.entries_plan(_chain(st), mm)
            assert (i["compute_kernel"], i["n_virtual"], i["prefix_rows"]) == (1, 4, 4096), (rr, mm, i)
        i = N.entries_plan(_chain(st[:4] + st[6:]), 200000)
        assert (i["compute_kernel"], i["n_virtual"]) == (1, 3), i
    # smaller m: tables limited to m / 16 rows (2^16 -> 32*32 rows per side);
    # the chain kernel below 2^16 samples
    small = N.entries_plan(_chain(specs), 1 << 16)
    assert small["algo"] == N.ALGO_BUCKETED and small["prefix_modes"] == small["suffix_modes"] == 2
    assert small["prefix_rows"] == 1024 and small["n_virtual"] == 8
    assert N.entries_plan(_chain(specs), 1000)["algo"] == N.ALGO_CHAIN
    monkeypatch.setenv("TNB_ENTRIES_MERGE", "0")
    off = N.entries_plan(_chain(specs), 1 << 24)
    assert off["n_virtual"] == 10 and off["kernel_flops"] == (8 * 2 * r * r + 2 * r) * float(1 << 24)


def test_timing_is_opt_in(lib):
    from paper_2206_11128_b200 import _native as N

    N.timing_enable(True)
    assert N.timing_read("entries_compute") == (0.0, 0)
    N.timing_enable(False)


@pytest.mark.parametrize("width", [1, 2])
@pytest.mark.parametrize("nthreads", [1, 0])
def test_host_narrow_codec(width, nthreads, lib):
    # the host half of the index transport codec runs without a GPU
    import torch

    from paper_2206_11128_b200 import _native

    lo, hi = (-128, 127) if width == 1 else (-32768, 32767)
    nt = torch.int8 if width == 1 else torch.int16
    rng = np.random.default_rng(width)
    for n in (0, 1, 17, 1000, (3 << 20) + 5):
        src = torch.from_numpy(rng.integers(lo, hi + 1, size=n, dtype=np.int64))
        if n:
            src[0], src[-1] = lo, hi
        dst = torch.empty(n, dtype=nt)
        assert _native.narrow_indices(src, dst, width, nthreads)
        assert torch.equal(dst.to(torch.int64), src)
        if n:
            for bad in (hi + 1, lo - 1, 1 << 40, -(1 << 62)):
                s2 = src.clone()
                s2[n // 2] = bad
                assert not _native.narrow_indices(s2, dst, width, nthreads)


def test_host_narrow_codec_rejects_bad_width(lib):
    import torch

    from paper_2206_11128_b200 import _native
    from paper_2206_11128_b200.errors import ContractViolationError

    with pytest.raises(ContractViolationError):
        _native.narrow_indices(torch.zeros(4, dtype=torch.int64), torch.zeros(4, dtype=torch.int32), 4)


def test_tntorch_attribute_aliases():
    # tntorch.Tensor spellings over the tntz data model (no device work)
    import paper_2206_11128_b200 as tb

    rng = np.random.default_rng(0)
    g0 = rng.standard_normal((1, 4, 3)).astype(np.float32)
    u1 = rng.standard_normal((5, 3)).astype(np.float32)
    f1 = rng.standard_normal((7, 5)).astype(np.float32)
    t = tb.Tensor([tb.ModeNode("tt", g0), tb.ModeNode("cp", u1, f1)])
    assert t.shape == (4, 7)
    assert [tuple(c.shape) for c in t.cores] == [(1, 4, 3), (5, 3)]
    assert t.Us[0] is None and tuple(t.Us[1].shape) == (7, 5)
    assert np.array_equal(t.cores[1].cpu().numpy(), u1)
