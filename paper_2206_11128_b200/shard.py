"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed).

All three operations shard without any data exchange:

* entries  -- contiguous row blocks of the index matrix; cores replicated;
* full     -- contiguous slabs of the leading mode (the reference's own
              ``full(t[lo:hi])``, indexing.py:132-137), output stays sharded;
* dot/norm -- contiguous blocks of the batch (pairs).

The only collective is the OPTIONAL gather of results to every rank (NCCL
all-gather over NVLink on GPUs, gloo in the CPU tests).  ``compute`` hooks
let the CPU tests drive the same planning/gather code with the oracle.
"""

from __future__ import annotations

from typing import Callable, Optional

import torch

from .core import TnTensor, chain_dot, entries, full, norm
from .errors import ContractViolationError


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced [lo, hi) of n units for ``rank`` of ``world``
    (the first n % world ranks get one extra unit)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist(group):
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return None, 1, 0
    return dist, dist.get_world_size(group), dist.get_rank(group)


def gather_rows(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather variable-size row blocks (rank order == row order).  NCCL
    gathers device tensors in place; under gloo (the CPU test backend, or
    ranks sharing one GPU) a device block is gathered through host memory
    and the result moved back to the block's device."""
    dist, world, rank = _dist(group)
    if dist is None or world == 1:
        return local
    if local.device.type == "cuda" and dist.get_backend(group) == "gloo":
        return gather_rows(local.cpu(), n_total, group).to(local.device)
    base = n_total // world + (1 if n_total % world else 0)
    pad = torch.zeros((base,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * base,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = []
    for r in range(world):
        lo, hi = shard_bounds(n_total, world, r)
        parts.append(out[r * base: r * base + (hi - lo)])
    return torch.cat(parts, 0)


def entries_sharded(t: TnTensor, indices, *, group=None, gather: bool = True,
                    compute: Optional[Callable] = None):
    """Rank r evaluates rows shard_bounds(M, world, r) of ``indices``."""
    _, world, rank = _dist(group)
    m = int(indices.shape[0])
    lo, hi = shard_bounds(m, world, rank)
    fn = compute or entries
    local = fn(t, indices[lo:hi])
    if not gather:
        return local, (lo, hi)
    return gather_rows(local, m, group)


def batch_slice(t: TnTensor, lo: int, hi: int) -> TnTensor:
    """Batch elements [lo, hi) of a batched chain (views, no copies)."""
    from .core import ModeNode

    nodes = [ModeNode(n.kind, n.core[lo:hi], None if n.factor is None else n.factor[lo:hi], True, dtype=n.dtype)
             for n in t.nodes]
    return TnTensor(nodes, hi - lo)


def _batch_of(t, op: str) -> int:
    nb = getattr(t, "batch_size", None)
    if nb is None:
        raise ContractViolationError(f"{op} shards the batch axis: the tensor is not batched")
    return int(nb)


def _empty_result(t) -> torch.Tensor:
    """The (0,) result of a rank whose pair shard is empty (batch < world):
    it still joins the gather, so the other ranks do not wait forever."""
    if isinstance(t, TnTensor):
        return torch.empty(0, dtype=t.dtype, device=t.device)
    return torch.empty(0, dtype=torch.float64)


def dot_sharded(a: TnTensor, b: TnTensor, *, group=None, gather: bool = True,
                compute: Optional[Callable] = None, slicer: Optional[Callable] = None):
    """Batched dot with the pairs split across ranks."""
    _, world, rank = _dist(group)
    nb = _batch_of(a, "dot_sharded")
    if _batch_of(b, "dot_sharded") != nb:
        raise ContractViolationError("operands must agree on batching")
    lo, hi = shard_bounds(nb, world, rank)
    sl = slicer or batch_slice
    local = (compute or chain_dot)(sl(a, lo, hi), sl(b, lo, hi)) if hi > lo else _empty_result(a)
    if not gather:
        return local, (lo, hi)
    return gather_rows(local, nb, group)


def norm_sharded(t: TnTensor, *, group=None, gather: bool = True,
                 compute: Optional[Callable] = None, slicer: Optional[Callable] = None):
    _, world, rank = _dist(group)
    nb = _batch_of(t, "norm_sharded")
    lo, hi = shard_bounds(nb, world, rank)
    local = (compute or norm)((slicer or batch_slice)(t, lo, hi)) if hi > lo else _empty_result(t)
    if not gather:
        return local, (lo, hi)
    return gather_rows(local, nb, group)


def full_sharded(t: TnTensor, *, group=None, compute: Optional[Callable] = None):
    """Rank r writes the leading-mode slab shard_bounds(J_0, world, r) of
    full(t); returns (slab, (lo, hi)).  No gather: 256^4 fp32 is 17 GB."""
    _, world, rank = _dist(group)
    lo, hi = shard_bounds(t.shape[0], world, rank)
    fn = compute or (lambda tt, l, h: full(tt, lead=(l, h)))
    return fn(t, lo, hi), (lo, hi)
