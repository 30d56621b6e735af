"""Loader for the committed golden vectors (tests/golden/*.npz).

The vectors were produced by the real reference (tntz) through
tests/golden/make_golden.py; this loader rebuilds each case's chain as
``(kind, core, factor)`` triples so both the oracle and the GPU façade can
consume it.  No import of /root/reference happens here.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def _load():
    z = np.load(GOLDEN / "golden.npz")
    meta = json.loads((GOLDEN / "golden.json").read_text())
    return z, meta


_Z, _META = _load()
CASE_NAMES = sorted(_META)


def case(name):
    """Returns dict: nodes (list of triples), batch, other (or None), outputs."""
    m = _META[name]

    def triples(role):
        spec = m[role]
        out = []
        for k, kind in enumerate(spec["kinds"]):
            core = _Z[f"{name}/{role}/core{k}"]
            fac = _Z[f"{name}/{role}/factor{k}"] if spec["factors"][k] else None
            out.append((kind, core, fac))
        return out, spec["batch"]

    nodes, batch = triples("t")
    other = triples("b") if "b" in m else None
    outs = {key: _Z[f"{name}/{key}"] for key in m.get("outputs", [])}
    return {"name": name, "nodes": nodes, "batch": batch, "other": other,
            "out": outs, "cite": m.get("cite", "")}


def configs():
    return np.load(GOLDEN / "configs.npz")
