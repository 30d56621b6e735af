"""``t[idx]`` for the hot path (reference: indexing.getitem, indexing.py:120-151).

Supported keys:

* a 2-D integer array (numpy or torch): the array form of indexing.py:123-130,
  evaluated by the K1 entries kernel;
* a tuple of ``ndim`` integers (or one integer for a one-mode tensor): the
  all-integer form, whose value the reference obtains through repeated
  ``ttv`` (indexing.py:138-147) -- here it is one K1 sample.

Compressed slicing (slices, lists, ``None``, ``Ellipsis``; indexing.py:52-88,
131-151) builds new chains rather than contracting one and is outside the
GPU hot path; it raises ``NotImplementedError``.
"""

from __future__ import annotations

import numbers

import numpy as np
import torch

from .core import TnTensor, entries
from .errors import ContractViolationError


def _is_int(x) -> bool:
    return isinstance(x, numbers.Integral) and not isinstance(x, bool)


def getitem(t: TnTensor, key):
    if isinstance(key, (np.ndarray, torch.Tensor)) and key.ndim == 2:
        if key.shape[1] != t.ndim:
            raise ContractViolationError(
                f"index matrix must have {t.ndim} columns, got {key.shape[1]}")
        is_int = (not key.dtype.is_floating_point and not key.dtype.is_complex
                  and key.dtype != torch.bool) if isinstance(key, torch.Tensor) \
            else np.issubdtype(key.dtype, np.integer)
        if key.numel() if isinstance(key, torch.Tensor) else key.size:
            if not is_int:
                raise ContractViolationError("index matrix must hold integers")
        return entries(t, key)
    if _is_int(key) and t.ndim == 1:
        key = (key,)
    if isinstance(key, tuple) and len(key) == t.ndim and all(_is_int(i) for i in key):
        # bounds are checked from the last mode backwards (indexing.py:142-146)
        for k in reversed(range(t.ndim)):
            i, size = int(key[k]), t.shape[k]
            i_norm = i + size if i < 0 else i
            if not 0 <= i_norm < size:
                raise ContractViolationError(f"index {i} out of bounds for size {size}")
        val = entries(t, np.asarray([key], dtype=np.int64))
        if t.batch_size is None:
            return float(val[0].item())
        return val[0]
    raise NotImplementedError(
        "compressed slicing (indexing.py:131-151) is outside the GPU contraction hot path; "
        "index with a 2-D integer array or a full tuple of integers")
