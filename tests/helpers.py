"""Shared helpers for the GPU parity tests (oracle = oracle/tntz_oracle.py)."""

from __future__ import annotations

import numpy as np

from oracle import tntz_oracle as O

# Acceptance bar of BASELINE north_star / SURVEY §8(c): relative Frobenius
# error AND max|diff| / max|ref|, both <= 1e-5, against the float64 oracle on
# identical fp32 inputs.
TOL = 1e-5


def to_np(x):
    import torch

    if isinstance(x, torch.Tensor):
        return x.detach().cpu().double().numpy()
    return np.asarray(x, dtype=np.float64)


def assert_close(got, ref, tol=TOL, what=""):
    got, ref = to_np(got), np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    if not ref.size:
        return
    if not np.any(ref):
        assert np.abs(got).max() <= tol, f"{what}: expected zeros"
        return
    e = O.rel_errors(got, ref)
    assert e["rel_fro"] <= tol and e["max_rel"] <= tol, f"{what}: {e}"


def assert_dot_close(got, ref, scale, tol=TOL, what=""):
    """Scalar inner products can cancel: accept |diff| <= tol*|ref| plus a
    floor of 1e-6 * ||a|| ||b|| (fp32 accumulation of the transfer matrix)."""
    got, ref, scale = to_np(got), np.asarray(ref, dtype=np.float64), np.asarray(scale, dtype=np.float64)
    assert got.shape == ref.shape, what
    assert np.all(np.abs(got - ref) <= tol * np.abs(ref) + 1e-6 * scale), \
        f"{what}: got {got} ref {ref}"


def facade(nodes, batch=None):
    import paper_2206_11128_b200 as tb

    return tb.TnTensor([tb.ModeNode(k, c, f, batched=batch is not None) for k, c, f in nodes],
                       batch)
