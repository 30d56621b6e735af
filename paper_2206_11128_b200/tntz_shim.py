"""Run the reference package itself on the GPU: ``install()`` re-points
tntz's hot-path functions at this package's CUDA path.

The reference (``tntz``, /root/reference/pkg/src/tntz) computes in float64
with numpy.  After ``install(tntz)``:

==========================  ===========================================
tntz symbol                 now runs
==========================  ===========================================
core.full (core.py:337)     K2 ``tnb_full_f64`` (or f32)
core.entries (core.py:394)  K1 ``tnb_entries_f64`` (or f32)
core.chain_dot (core.py:362)  K3 ``tnb_dot_f64`` (or f32)
core.norm (core.py:387)     K3 ``tnb_norm_f64`` (or f32)
==========================  ===========================================

and every module that imported those names (``tntz``, ``tntz.arithmetic``
for ``dot``, ``tntz.indexing`` for the array form of ``t[idx]``) sees the
GPU versions; ``TnTensor.full`` / ``.norm`` look the names up in
``tntz.core`` and follow.  Results come back as the reference returns them
(fresh float64 ndarrays, Python floats for unbatched dot / norm) and errors
as the reference's own exception classes with this package's (identical)
messages.  ``dtype=torch.float64`` (the default) runs the float64
instantiation, so the reference's own tests pass at their native 1e-12 ..
1e-14 tolerances (tests/test_tntz_shim.py); float32 is the fast path.

This module is the integration a tntz user would switch on; it imports
nothing from the oracle and has no CPU fallback -- without a GPU every
patched call raises like the rest of the package.
"""

from __future__ import annotations

import functools

import numpy as np
import torch

from . import core as C
from . import errors as E

_PATCHED = ("full", "entries", "chain_dot", "norm")


def _convert(t, dtype):
    """A reference TnTensor (float64 numpy nodes) as this package's chain."""
    nodes = [C.ModeNode(n.kind, n.core, n.factor, n.batched, dtype=dtype) for n in t.nodes]
    return C.TnTensor(nodes, t.batch_size)


def _translate(tz, fn):
    """Re-raise this package's errors as the reference's classes."""
    mapping = {E.ContractViolationError: tz.ContractViolationError, E.StructuralError: tz.StructuralError}

    @functools.wraps(fn)
    def wrapped(*a, **k):
        try:
            return fn(*a, **k)
        except (E.ContractViolationError, E.StructuralError) as e:
            raise mapping[type(e)](str(e)) from None

    return wrapped


def _to_np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy().astype(np.float64, copy=False)
    return x


def install(tz, dtype=torch.float64):
    """Patch the reference package ``tz`` (the imported ``tntz`` module);
    returns a function that restores the originals."""
    saved = {}

    def full(t):
        return _to_np(C.full(_convert(t, dtype)))

    def entries(t, indices):
        idx = indices
        if not isinstance(idx, (np.ndarray, torch.Tensor)):
            idx = np.asarray(idx)
        return _to_np(C.entries(_convert(t, dtype), idx))

    def chain_dot(a, b):
        if a.shape != b.shape:  # the reference's message (core.py:368-369)
            raise E.ContractViolationError(f"shape mismatch: {a.shape} vs {b.shape}")
        return _to_np(C.chain_dot(_convert(a, dtype), _convert(b, dtype)))

    def norm(t):
        return _to_np(C.norm(_convert(t, dtype)))

    impl = {"full": full, "entries": entries, "chain_dot": chain_dot, "norm": norm}
    impl = {k: _translate(tz, v) for k, v in impl.items()}
    mods = [tz.core, tz, tz.arithmetic, tz.indexing]
    for mod in mods:
        for name in _PATCHED:
            if hasattr(mod, name):
                saved[(mod, name)] = getattr(mod, name)
                setattr(mod, name, impl[name])

    def restore():
        for (mod, name), fn in saved.items():
            setattr(mod, name, fn)

    return restore
