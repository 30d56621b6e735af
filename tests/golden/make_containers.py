"""Golden TNTZ1 containers written by the REAL reference's save() -- run in
the build container only (needs /root/reference):

    python tests/golden/make_containers.py

For each fixture (the shapes of pkg/tests/test_serialization.py's FIXTURES,
plus a cfg5-structured hybrid) the reference's own generator draws the chain;
every array is rounded to fp32-representable values (the GPU path's dtype, so
the device copy is exact), rebuilt as tntz ModeNodes and saved with
tntz.save.  ``expected.npz`` holds the reference's float64 full(), entries at
seeded indices and norm of each, plus one raw dense file written by
tntz.serialization.write_dense.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tntz  # noqa: E402
from tntz.core import ModeNode, TnTensor, entries  # noqa: E402
from tntz.serialization import write_dense  # noqa: E402

OUT = Path(__file__).resolve().parent / "containers"


def fp32_valued(t):
    nodes = []
    for n in t.nodes:
        core = n.core.astype(np.float32).astype(np.float64)
        fac = None if n.factor is None else n.factor.astype(np.float32).astype(np.float64)
        nodes.append(ModeNode(n.kind, core, fac, batched=t.batch_size is not None))
    return TnTensor(nodes, t.batch_size)


def cfg5_like(seed):
    rng = np.random.default_rng(seed)
    nodes = []
    for k in range(6):
        if k < 3:
            rl, rr = (1 if k == 0 else 6), 6
            core = rng.standard_normal((rl, 5, rr)) * 6 ** -0.5
            kind = "tt"
        else:
            core = rng.standard_normal((5, 6)) * 6 ** -0.5
            kind = "cp"
        fac = rng.standard_normal((9, 5)) * 6 ** -0.5
        nodes.append(ModeNode(kind, core, fac))
    return TnTensor(nodes)


FIXTURES = {
    "tt": lambda: tntz.random_tt((3, 4, 5), (2, 3), seed=0),
    "cp": lambda: tntz.random_cp((4, 4), 3, seed=1),
    "tucker": lambda: tntz.random_tucker((5, 4, 6), (2, 3, 2), (2, 2), seed=2),
    "blended": lambda: tntz.random_blended((3, 4, 3, 2), seed=3),
    "tt_batched": lambda: tntz.random_tt((3, 4), 2, seed=4, batch_size=6),
    "cp_batched": lambda: tntz.random_cp((3, 5), 2, seed=5, batch_size=2),
    "hybrid": lambda: cfg5_like(6),
}


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    exp = {}
    for name, make in FIXTURES.items():
        t = fp32_valued(make())
        tntz.save(t, OUT / f"{name}.tntz")
        if int(np.prod(t.shape)) * (t.batch_size or 1) <= 10_000:
            exp[f"{name}/full"] = tntz.full(t)
        idx = np.random.default_rng(7).integers(0, t.shape, size=(64, t.ndim), dtype=np.int64)
        exp[f"{name}/idx"] = idx
        exp[f"{name}/entries"] = entries(t, idx)
        exp[f"{name}/norm"] = np.asarray(tntz.norm(t), dtype=np.float64)
        for k, n in enumerate(t.nodes):
            exp[f"{name}/core{k}"] = n.core
            if n.factor is not None:
                exp[f"{name}/factor{k}"] = n.factor
    write_dense(exp["tucker/full"], OUT / "tucker_full.raw")
    np.savez_compressed(OUT / "expected.npz", **exp)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
