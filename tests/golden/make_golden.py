"""Generate golden vectors from the REAL reference (tntz) -- run in the build
container only (needs /root/reference; the GPU box never runs this).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Writes ``tests/golden/golden.npz`` (small cases, inputs + reference outputs)
and ``tests/golden/configs.npz`` (pins of the five BASELINE configs: core
checksums of the seeded generators and reference outputs on small index
subsets).  Every input is fp32-valued (the GPU path's dtype) and handed to
tntz, which upcasts it exactly to float64 (core.py:37-38, 54); the stored
outputs are the reference's float64 results.

Cases cite the reference tests they mirror (pkg/tests/...).  ``--big`` also
regenerates the config-4 pin, which needs ~18 GB of RAM (4096-pair batch).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tntz  # noqa: E402
from tntz.core import entries as t_entries, chain_dot as t_chain_dot  # noqa: E402

HERE = Path(__file__).resolve().parent
F32 = np.float32


def f32_chain(t):
    """Round every core/factor to fp32 and rebuild the TnTensor."""
    nodes = []
    for n in t.nodes:
        fac = None if n.factor is None else n.factor.astype(F32)
        nodes.append(tntz.ModeNode(n.kind, n.core.astype(F32), fac, n.batched))
    return tntz.TnTensor(nodes, t.batch_size)


class Store:
    def __init__(self):
        self.arrays = {}
        self.meta = {}

    def chain(self, name, t, role="t"):
        kinds = []
        for k, n in enumerate(t.nodes):
            kinds.append(n.kind)
            self.arrays[f"{name}/{role}/core{k}"] = n.core.astype(F32)
            if n.factor is not None:
                self.arrays[f"{name}/{role}/factor{k}"] = n.factor.astype(F32)
        m = self.meta.setdefault(name, {})
        m[role] = {"kinds": kinds, "batch": t.batch_size,
                   "factors": [n.factor is not None for n in t.nodes],
                   "shape": list(t.shape)}

    def put(self, name, key, arr):
        self.arrays[f"{name}/{key}"] = np.asarray(arr)
        self.meta.setdefault(name, {}).setdefault("outputs", []).append(key)


def add_case(st, name, t, *, idx=None, other=None, do_full=True, cite=""):
    t = f32_chain(t)
    st.chain(name, t)
    st.meta[name]["cite"] = cite
    if do_full:
        st.put(name, "full", tntz.full(t))
    st.put(name, "norm", np.asarray(tntz.norm(t)))
    if idx is not None:
        st.put(name, "idx", idx)
        st.put(name, "entries", t_entries(t, idx))
    if other is not None:
        o = f32_chain(other)
        st.chain(name, o, role="b")
        st.put(name, "dot", np.asarray(tntz.dot(t, o)))


def rand_idx(shape, m, seed, neg=True):
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, s, m) for s in shape], axis=1).astype(np.int64)
    if neg:  # exercise the negative wrap of core.py:411-413
        flip = rng.random(idx.shape) < 0.3
        idx = np.where(flip, idx - np.asarray(shape)[None, :], idx)
    return idx


def small_cases(st):
    # known answers (test_core.py:62-72, 127-136)
    ones_cp = tntz.TnTensor([tntz.ModeNode("cp", np.ones((2, 3))),
                             tntz.ModeNode("cp", np.ones((2, 3)))])
    add_case(st, "kat_ones_cp", ones_cp, idx=np.array([[0, 0], [1, 1], [-1, 0]]),
             cite="test_core.py:62-64")
    u, v = np.array([1.0, 2.0, 3.0]), np.array([4.0, 5.0])
    outer = tntz.TnTensor([tntz.ModeNode("tt", u.reshape(1, 3, 1)),
                           tntz.ModeNode("tt", v.reshape(1, 2, 1))])
    add_case(st, "kat_outer", outer, idx=np.array([[0, 0], [2, 1], [1, -1]]),
             cite="test_core.py:66-72")
    w = np.array([0.6, 0.8])
    unit = tntz.TnTensor([tntz.ModeNode("tt", w.reshape(1, 2, 1)),
                          tntz.ModeNode("tt", w.reshape(1, 2, 1))])
    add_case(st, "kat_unit", unit, other=unit, cite="test_core.py:132-136")
    zero = tntz.TnTensor([tntz.ModeNode("tt", np.zeros((1, 3, 2))),
                          tntz.ModeNode("tt", np.zeros((2, 4, 1)))])
    add_case(st, "kat_zero", zero, idx=rand_idx((3, 4), 5, 0),
             other=tntz.random_tt((3, 4), 2, seed=16), cite="test_core.py:127-130")
    # single-mode chains: CP sums over R (core.py:316-320), TT is a vector
    add_case(st, "single_cp", tntz.TnTensor([tntz.ModeNode("cp", np.arange(15.0).reshape(5, 3) / 7)]),
             idx=np.array([[0], [4], [-2]]), other=tntz.random_cp((5,), 2, seed=4),
             cite="core.py:316-320")
    add_case(st, "single_tucker_cp",
             tntz.TnTensor([tntz.ModeNode("cp", np.arange(6.0).reshape(3, 2) / 5,
                                          np.linspace(-1, 1, 12).reshape(4, 3))]),
             idx=np.array([[0], [3], [-1]]), cite="core.py:316-326")
    # random TT / CP / Tucker / blended (test_core.py:74-102, 178-190)
    add_case(st, "tt_453", tntz.random_tt((4, 5, 3), [2, 3], seed=1),
             idx=rand_idx((4, 5, 3), 64, 1), other=tntz.random_tt((4, 5, 3), 2, seed=2),
             cite="test_core.py:178-190")
    add_case(st, "cp_345", tntz.random_cp((3, 4, 5), 3, seed=9),
             idx=rand_idx((3, 4, 5), 64, 2), other=tntz.random_cp((3, 4, 5), 2, seed=10),
             cite="random.py:43-53")
    add_case(st, "tucker_675", tntz.random_tucker((6, 7, 5), (3, 4, 2), [2, 3], seed=3),
             idx=rand_idx((6, 7, 5), 64, 3),
             other=tntz.random_tucker((6, 7, 5), (2, 5, 3), [3, 2], seed=4),
             cite="random.py:56-65")
    shapes = [(3, 4, 5), (3, 2, 4, 3), (4, 3, 5, 2), (2, 3), (5, 4, 3, 2, 3), (7,), (4, 5)]
    for s in range(14):
        shp = shapes[s % len(shapes)]
        t = tntz.random_blended(shp, seed=s)
        o = tntz.random_blended(shp, seed=100 + s)
        add_case(st, f"blended_{s}", t, idx=rand_idx(shp, 64, 10 + s), other=o,
                 cite="test_core.py:74-89, test_acceptance.py:87-96")
    # rank-5 wider chain with CP interior runs of larger rank
    t = tntz.TnTensor([
        tntz.ModeNode("cp", np.random.default_rng(5).standard_normal((6, 5))),
        tntz.ModeNode("cp", np.random.default_rng(6).standard_normal((4, 5)),
                      np.random.default_rng(7).standard_normal((9, 4))),
        tntz.ModeNode("tt", np.random.default_rng(8).standard_normal((5, 3, 4))),
        tntz.ModeNode("cp", np.random.default_rng(9).standard_normal((7, 4))),
        tntz.ModeNode("tt", np.random.default_rng(10).standard_normal((4, 5, 1)),
                      np.random.default_rng(11).standard_normal((8, 5))),
    ])
    add_case(st, "hybrid_wide", t, idx=rand_idx(t.shape, 128, 12), cite="core.py:266-334")
    # batched chains (test_core.py:98-102, test_arithmetic.py:346-387,
    # test_indexing.py:315-321)
    tb = tntz.random_tt((3, 4, 2), 3, seed=7, batch_size=5)
    ob = tntz.random_tt((3, 4, 2), 2, seed=8, batch_size=5)
    add_case(st, "batched_tt", tb, idx=rand_idx((3, 4, 2), 32, 20), other=ob,
             cite="test_core.py:98-102")
    rng = np.random.default_rng(21)
    bsz = 3
    nb = [
        tntz.ModeNode("cp", rng.standard_normal((bsz, 4, 3)), rng.standard_normal((bsz, 5, 4)), True),
        tntz.ModeNode("tt", rng.standard_normal((bsz, 3, 6, 2)), None, True),
        tntz.ModeNode("cp", rng.standard_normal((bsz, 3, 2)), None, True),
        tntz.ModeNode("tt", rng.standard_normal((bsz, 2, 4, 1)), rng.standard_normal((bsz, 6, 4)), True),
    ]
    hb = tntz.TnTensor(nb, bsz)
    nb2 = [
        tntz.ModeNode("tt", rng.standard_normal((bsz, 1, 5, 2)), None, True),
        tntz.ModeNode("tt", rng.standard_normal((bsz, 2, 6, 3)), None, True),
        tntz.ModeNode("cp", rng.standard_normal((bsz, 3, 3)), None, True),
        tntz.ModeNode("cp", rng.standard_normal((bsz, 6, 3)), None, True),
    ]
    add_case(st, "batched_hybrid", hb, idx=rand_idx(hb.shape, 32, 22),
             other=tntz.TnTensor(nb2, bsz), cite="core.py:280-288, 352-359, 379-384, 425-460")


def core_stats(cores):
    """Checksums pinning a generator: per core sum, sum of squares, head."""
    out = []
    for c in cores:
        c64 = np.asarray(c, dtype=np.float64)
        out.append(np.concatenate([[c64.sum(), (c64 ** 2).sum()], c64.ravel()[:16]]))
    return np.stack(out)


def config_pins(st, big):
    # cfg1: TT N=6, I=16, r=8 -- small enough to pin everything but full()
    t1 = f32_chain(tntz.random_tt((16,) * 6, 8, seed=0, scale=8 ** -0.5))
    i1 = np.random.default_rng(2).integers(0, 16, size=(4096, 6), dtype=np.int64)
    st.put("cfg1", "core_stats", core_stats([n.core for n in t1.nodes]))
    st.put("cfg1", "idx_head", i1[:64])
    st.put("cfg1", "entries", t_entries(t1, i1))
    st.put("cfg1", "norm", np.asarray(tntz.norm(t1)))
    slab = tntz.full(t1[0:1])
    st.put("cfg1", "slab0_sum", np.asarray([slab.sum(), (slab ** 2).sum()]))
    st.put("cfg1", "slab0_head", slab.ravel()[:256])
    # cfg2: TT N=10, I=32, r=32
    t2 = f32_chain(tntz.random_tt((32,) * 10, 32, seed=0, scale=32 ** -0.5))
    i2 = np.random.default_rng(2).integers(0, 32, size=(2048, 10), dtype=np.int64)
    st.put("cfg2", "core_stats", core_stats([n.core for n in t2.nodes]))
    st.put("cfg2", "idx_head", i2[:64])
    st.put("cfg2", "entries", t_entries(t2, i2))
    st.put("cfg2", "norm", np.asarray(tntz.norm(t2)))
    # cfg3: TT N=4, I=256, r=64 -- norm and one mode-0 slab, sampled
    t3 = f32_chain(tntz.random_tt((256,) * 4, 64, seed=0, scale=64 ** -0.5))
    st.put("cfg3", "core_stats", core_stats([n.core for n in t3.nodes]))
    st.put("cfg3", "norm", np.asarray(tntz.norm(t3)))
    for i0 in (0, 255):
        slab = tntz.full(t3[i0:i0 + 1])
        st.put("cfg3", f"slab{i0}_sum", np.asarray([slab.sum(), (slab ** 2).sum()]))
        rng = np.random.default_rng(i0)
        pos = rng.integers(0, slab.size, 512)
        st.put("cfg3", f"slab{i0}_pos", pos)
        st.put("cfg3", f"slab{i0}_val", slab.ravel()[pos])
    # cfg5: hybrid CP-TT-Tucker (explicit ModeNodes)
    rng = np.random.default_rng(0)
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
        nodes.append(tntz.ModeNode(kind, core.astype(F32), fac.astype(F32)))
    t5 = tntz.TnTensor(nodes)
    i5 = np.random.default_rng(2).integers(0, 128, size=(2048, 8), dtype=np.int64)
    st.put("cfg5", "core_stats", core_stats([n.core for n in t5.nodes] + [n.factor for n in t5.nodes]))
    st.put("cfg5", "idx_head", i5[:64])
    st.put("cfg5", "entries", t_entries(t5, i5))
    st.put("cfg5", "norm", np.asarray(tntz.norm(t5)))
    if big:
        # cfg4: 4096 TT pairs, N=16, I=64, r=16 (seed s and s+1)
        ta = f32_chain(tntz.random_tt((64,) * 16, 16, seed=0, batch_size=4096, scale=0.25))
        st.put("cfg4", "core_stats_a", core_stats([n.core for n in ta.nodes]))
        pairs = np.array([0, 1, 2, 1000, 4095])
        st.put("cfg4", "pairs", pairs)
        ea = [ta.batch_element(int(p)) for p in pairs]
        st.put("cfg4", "norm", np.array([tntz.norm(e) for e in ea]))
        del ta
        tb = f32_chain(tntz.random_tt((64,) * 16, 16, seed=1, batch_size=4096, scale=0.25))
        st.put("cfg4", "core_stats_b", core_stats([n.core for n in tb.nodes]))
        eb = [tb.batch_element(int(p)) for p in pairs]
        st.put("cfg4", "dot", np.array([t_chain_dot(x, y) for x, y in zip(ea, eb)]))
        # batched vs loop on the first 4 pairs (test_arithmetic.py:346-387)
        del tb


def main():
    big = "--big" in sys.argv
    st = Store()
    small_cases(st)
    np.savez_compressed(HERE / "golden.npz", **st.arrays)
    (HERE / "golden.json").write_text(json.dumps(st.meta, indent=1, sort_keys=True))
    cf = Store()
    old = {}
    if not big and (HERE / "configs.npz").exists():
        with np.load(HERE / "configs.npz") as z:
            old = {k: z[k] for k in z.files if k.startswith("cfg4/")}
    config_pins(cf, big)
    cf.arrays.update(old)
    np.savez_compressed(HERE / "configs.npz", **cf.arrays)
    print("wrote", len(st.arrays), "golden arrays,", len(cf.arrays), "config arrays")


if __name__ == "__main__":
    main()
