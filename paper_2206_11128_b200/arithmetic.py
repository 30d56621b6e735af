"""``dot`` of the hot path (reference: arithmetic.dot, arithmetic.py:189-193)."""

from __future__ import annotations

from .core import TnTensor, chain_dot
from .errors import ContractViolationError


def dot(a: TnTensor, b: TnTensor):
    """Inner product of equal-shaped chains; a vector of dots when batched."""
    if a.shape != b.shape:
        raise ContractViolationError(f"dot needs equal shapes, got {a.shape} vs {b.shape}")
    return chain_dot(a, b)
