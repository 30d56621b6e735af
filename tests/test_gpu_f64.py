"""The float64 instantiation against the reference's own
float64 outputs -- the golden vectors and the golden containers written by
the real tntz -- at a float64 tolerance instead of the fp32 bar."""

from pathlib import Path

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests import golden_cases as G
from tests.helpers import to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
tb = pytest.importorskip("paper_2206_11128_b200")
from paper_2206_11128_b200 import _native as N  # noqa: E402

TOL64 = 1e-12
GOLD = Path(__file__).resolve().parent / "golden" / "containers"


def close64(got, ref, what, tol=TOL64):
    got, ref = to_np(got), np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, what
    if not ref.size:
        return
    scale = max(np.abs(ref).max(), 1e-300)
    err = np.abs(got - ref).max() / scale
    assert err <= tol, f"{what}: max|d|/max|ref| = {err:.3e}"


def f64(nodes, batch=None):
    return tb.TnTensor([tb.ModeNode(k, c, f, batched=batch is not None, dtype=torch.float64)
                        for k, c, f in nodes], batch)


@pytest.mark.parametrize("name", G.CASE_NAMES)
def test_golden_f64(name):
    c = G.case(name)
    t = f64(c["nodes"], c["batch"])
    assert t.dtype == torch.float64
    out = c["out"]
    if "full" in out:
        close64(tb.full(t), out["full"], f"{name} full")
    got = tb.norm(t)
    close64(np.asarray(to_np(got)), np.asarray(out["norm"]), f"{name} norm")
    if "entries" in out:
        for algo in (N.ALGO_AUTO, N.ALGO_CHAIN, N.ALGO_LAYERED):
            r = tb.entries(t, out["idx"], algo=algo)
            assert r.dtype == torch.float64
            close64(r, out["entries"], f"{name} entries algo={algo}")
    if "dot" in out:
        b = f64(*c["other"])
        oa, ob = O.make_chain(c["nodes"], c["batch"]), O.make_chain(*c["other"])
        scale = np.asarray(O.norm(oa)) * np.asarray(O.norm(ob))
        d = np.asarray(to_np(tb.dot(t, b)))
        assert np.all(np.abs(d - np.asarray(out["dot"])) <= TOL64 * np.maximum(scale, 1e-300)), name
    oc = O.make_chain(c["nodes"], c["batch"])
    for k in range(t.ndim):
        close64(tb.node_tt_core(t, k), O.tt_core(oc, k), f"{name} mode {k}")


@pytest.mark.parametrize("name", ["tt", "cp", "tucker", "blended", "tt_batched", "cp_batched", "hybrid"])
def test_containers_f64(name):
    # the payload floats arrive bit for bit; contractions agree at 1e-12
    exp = np.load(GOLD / "expected.npz")
    t = tb.load(GOLD / f"{name}.tntz", dtype=torch.float64)
    for k, n in enumerate(t.nodes):
        assert np.array_equal(to_np(n.core), exp[f"{name}/core{k}"])
    if f"{name}/full" in exp:
        close64(tb.full(t), exp[f"{name}/full"], f"{name} full")
    close64(tb.entries(t, exp[f"{name}/idx"]), exp[f"{name}/entries"], f"{name} entries")
    close64(np.asarray(to_np(tb.norm(t))), np.asarray(exp[f"{name}/norm"]), f"{name} norm")


def test_f64_contracts():
    rng = np.random.default_rng(3)
    nodes = [("tt", rng.standard_normal((1, 5, 3)), None), ("cp", rng.standard_normal((4, 3)), None),
             ("tt", rng.standard_normal((3, 6, 1)), None)]
    t64 = f64(nodes)
    t32 = t64.float()
    assert t32.dtype == torch.float32 and t64.double() is t64
    idx = O.uniform_indices(t64.shape, 5000, 1)
    bad = idx.copy()
    bad[17, 1] = 4
    with pytest.raises(tb.ContractViolationError, match="mode 1"):
        tb.entries(t64, bad)
    with pytest.raises(tb.ContractViolationError, match="bucketed"):
        tb.entries(t64, idx, algo=N.ALGO_BUCKETED)
    with pytest.raises(tb.ContractViolationError, match="dtype"):
        tb.dot(t64, t32)
    with pytest.raises(tb.ContractViolationError, match="one dtype"):
        tb.TnTensor([t64.nodes[0], t32.nodes[1], t64.nodes[2]])
    ref = O.entries(O.make_chain([(k, c) if f is None else (k, c, f) for k, c, f in nodes]), idx)
    close64(tb.entries(t64, idx), ref, "entries")
    close64(tb.full(t64, lead=(1, 3)), O.full_slab(O.make_chain([(k, c) for k, c, f in nodes]), 1, 3), "slab")
    # a large f64 batch of pairs through the generic dot kernel
    a = O.random_tt((8,) * 5, 4, seed=2, batch_size=64, scale=0.5)
    b = O.random_tt((8,) * 5, 3, seed=4, batch_size=64, scale=0.5)
    ta, tb_ = f64([("tt", x, None) for x in a], 64), f64([("tt", x, None) for x in b], 64)
    ref = O.chain_dot(O.make_chain([("tt", x) for x in a], 64), O.make_chain([("tt", x) for x in b], 64))
    close64(tb.dot(ta, tb_), ref, "batched dot", tol=1e-11)


@pytest.mark.parametrize("batch", [None, 3])
def test_f64_entries_layered_auto(batch):
    # float64 AUTO picks the layered kernels from 2^12 rows up
    cores = O.random_tt((32,) * 7, 16, seed=8, batch_size=batch, scale=0.25)
    nodes = [("tt", c, None) for c in cores]
    t, o = f64(nodes, batch), O.make_chain([("tt", c) for c in cores], batch)
    idx = O.uniform_indices((32,) * 7, 9001, 4)
    idx[::4] -= 32
    close64(tb.entries(t, idx), O.entries(o, idx), "f64 layered entries")
    bad = idx.copy()
    bad[77, 3] = 32
    with pytest.raises(tb.ContractViolationError, match="mode 3"):
        tb.entries(t, bad)
