"""GPU-backed callers of entry evaluation.

The reference's cross-approximation drives entry evaluation through two
hooks: ``elementwise`` approximates g(t) by sampling f(idx) = g(entries(t,
idx)) (cross.py:348-363), and every sweep scores the current approximation
on a validation set (cross.py:277-282).  Both are entry evaluation plus an
elementwise map or a reduction, so here they stay on the device: indices go
through K1, g is applied to the device tensor, the validation norms are
reduced on the device in float64.  The cross-approximation algorithm itself
(index-set selection, maxvol) is outside this package's scope.
"""

from __future__ import annotations

from typing import Callable, Optional

import torch

from .core import TnTensor, entries
from .errors import ContractViolationError


def sampler(t: TnTensor, g: Optional[Callable[[torch.Tensor], torch.Tensor]] = None):
    """f(idx) = g(entries(t, idx)) on the device (the sampling function of
    cross.elementwise, cross.py:358-360).  ``g`` must be an elementwise torch
    function (identity when omitted); indices are anything ``entries``
    accepts, including pinned host int64 matrices."""
    if t.batch_size is not None:
        raise ContractViolationError("elementwise does not support batched tensors")

    def f(idx):
        v = entries(t, idx)
        return v if g is None else g(v)

    return f


def validation_error(t: TnTensor, x_val, y_val) -> float:
    """max over the batch columns of ||y - t[x]|| / ||y|| (||t[x]|| where
    ||y|| = 0), as cross.py:277-282 scores an approximation."""
    approx = entries(t, x_val)
    stack = 1 if t.batch_size is None else t.batch_size
    approx = approx.reshape(-1, stack).to(torch.float64)
    y = torch.as_tensor(y_val, dtype=torch.float64, device=approx.device).reshape(-1, stack)
    if y.shape != approx.shape:
        raise ContractViolationError(f"y_val has shape {tuple(y.shape)}, the samples give {tuple(approx.shape)}")
    diff = torch.linalg.vector_norm(y - approx, dim=0)
    ynorm = torch.linalg.vector_norm(y, dim=0)
    rel = torch.where(ynorm > 0, diff / torch.clamp(ynorm, min=1e-300), torch.linalg.vector_norm(approx, dim=0))
    return float(rel.max().item())
