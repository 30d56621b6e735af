"""CPU oracle for the contraction hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(``tntz``, /root/reference/pkg/src/tntz/core.py) for the three hot-path
operations: entry evaluation, dense decompression and the chain inner
product / norm.  It exists so that

* ``tests/`` can check the CUDA path against it,
* ``__graft_entry__.smoke()`` can check one small launch against it, and
* ``bench.py`` can time it as the CPU baseline (``cpu_baseline`` and the
  ``--impl reference`` arm, ``kind: "port"``).

Nothing in the product package (``paper_2206_11128_b200``) may import it:
the product path fails loudly when its CUDA library is missing instead of
falling back here.

Parity pinning: ``tests/golden/*.npz`` hold outputs of the real reference
(generated in the build container by ``tests/golden/make_golden.py``, which
imports ``tntz`` from /root/reference); ``tests/test_oracle_golden.py``
checks this restatement against every one of them.  The generators
(``random_tt``, ``cfg5_chain``) are pinned the same way, so the bench's
synthetic inputs are the same numbers the reference would produce for the
same seed.

A chain is represented by :class:`Chain` -- a tuple of :class:`Node` plus
an optional batch size -- duck-compatible with tntz's ``TnTensor``
(``nodes``/``batch_size``, nodes with ``kind``/``core``/``factor``).
All arithmetic is float64, as in the reference (core.py:37-38, 54).
"""

from __future__ import annotations

import os
from typing import NamedTuple, Optional, Sequence

import numpy as np

TT = "tt"
CP = "cp"


class OracleError(ValueError):
    """Raised where the reference raises ContractViolationError/StructuralError."""


class Node(NamedTuple):
    kind: str
    core: np.ndarray
    factor: Optional[np.ndarray] = None


class Chain(NamedTuple):
    nodes: tuple
    batch_size: Optional[int] = None

    @property
    def ndim(self) -> int:
        return len(self.nodes)

    @property
    def shape(self) -> tuple:
        # physical size: factor rows if present, else core's internal size
        # (core.py:81-86, 151-154)
        return tuple(
            (n.factor.shape[-2] if n.factor is not None else n.core.shape[-2])
            for n in self.nodes
        )


def make_chain(nodes, batch_size=None) -> Chain:
    """Build a float64 chain from (kind, core, factor) triples."""
    out = []
    for n in nodes:
        kind, core = n[0], np.asarray(n[1], dtype=np.float64)
        fac = n[2] if len(n) > 2 else None
        fac = None if fac is None else np.asarray(fac, dtype=np.float64)
        out.append(Node(kind, core, fac))
    ch = Chain(tuple(out), batch_size)
    rank_chain(ch)
    return ch


def from_tntz(t) -> Chain:
    """Duck-typed conversion of a tntz TnTensor (used only by fixture scripts)."""
    return Chain(tuple(Node(n.kind, np.asarray(n.core), n.factor) for n in t.nodes),
                 t.batch_size)


# --------------------------------------------------------------------------
# rank bookkeeping -- core.py:244-263
# --------------------------------------------------------------------------

def node_ranks(node: Node, k: int, n: int) -> tuple:
    """(left, right) rank a node exposes; CP collapses to 1 at chain ends."""
    if node.kind == TT:
        return node.core.shape[-3], node.core.shape[-1]
    r = node.core.shape[-1]
    return (1 if k == 0 else r), (1 if k == n - 1 else r)


def rank_chain(ch: Chain) -> list:
    n = ch.ndim
    pairs = [node_ranks(nd, k, n) for k, nd in enumerate(ch.nodes)]
    for k in range(n - 1):
        if pairs[k][1] != pairs[k + 1][0]:
            raise OracleError(f"rank mismatch between modes {k} and {k + 1}")
    ranks = [pairs[0][0]] + [p[1] for p in pairs]
    if ranks[0] != 1 or ranks[-1] != 1:
        raise OracleError("boundary ranks must be 1")
    return ranks


# --------------------------------------------------------------------------
# per-node preparation -- core.py:266-334
# --------------------------------------------------------------------------

def promote_cp(u: np.ndarray, k: int, n: int, batched: bool) -> np.ndarray:
    """TT core equivalent of a CP node (core.py:266-296, 315-322).

    Interior: D[a, i, b] = U[i, a] * delta(a, b); left end (1, I, R) = U;
    right end (R, I, 1) = U^T; a single-mode CP chain sums over R.
    """
    if not batched:
        u = u[None]
    bsz, isz, r = u.shape
    if n == 1:
        d = u.sum(axis=-1)[:, None, :, None]
    elif k == 0:
        d = u[:, None, :, :]
    elif k == n - 1:
        d = np.transpose(u, (0, 2, 1))[..., None]
    else:
        d = np.zeros((bsz, r, isz, r))
        for a in range(r):
            d[:, a, :, a] = u[:, :, a]
    d = np.ascontiguousarray(d)
    return d if batched else d[0]


def tt_core(ch: Chain, k: int) -> np.ndarray:
    """Effective (batched: 4-D) TT core of mode k, factor absorbed
    (core.py:307-334: node_tt_core + apply_factor)."""
    node = ch.nodes[k]
    batched = ch.batch_size is not None
    if node.kind == CP:
        g = promote_cp(node.core, k, ch.ndim, batched)
    else:
        g = node.core
    if node.factor is not None:
        # einsum "ji,rik->rjk" (core.py:334); batched "bji,brik->brjk" (333)
        if batched:
            g = np.einsum("bji,brik->brjk", node.factor, g)
        else:
            g = np.einsum("ji,rik->rjk", node.factor, g)
    return g


# --------------------------------------------------------------------------
# dense decompression -- core.py:337-359
# --------------------------------------------------------------------------

def full(ch: Chain) -> np.ndarray:
    """Left-to-right unfolding GEMM chain; C order, last index fastest."""
    shape = ch.shape
    if ch.batch_size is None:
        m = np.ones((1, 1))
        for k in range(ch.ndim):
            g = tt_core(ch, k)
            rl, j, rr = g.shape
            m = (m @ g.reshape(rl, j * rr)).reshape(-1, rr)
        return m.reshape(shape)
    b = ch.batch_size
    m = np.ones((b, 1, 1))
    for k in range(ch.ndim):
        g = tt_core(ch, k)
        _, rl, j, rr = g.shape
        m = np.matmul(m, g.reshape(b, rl, j * rr)).reshape(b, -1, rr)
    return m.reshape((b,) + shape)


def full_slab(ch: Chain, lo: int, hi: int) -> np.ndarray:
    """full() restricted to leading-mode rows [lo, hi) -- the reference's own
    ``full(t[lo:hi])`` (indexing.py:132-137 -> _subset_node 106-111)."""
    nodes = list(ch.nodes)
    n0 = nodes[0]
    if n0.factor is not None:
        nodes[0] = Node(n0.kind, n0.core, n0.factor[..., lo:hi, :])
    else:
        nodes[0] = Node(n0.kind, np.take(n0.core, np.arange(lo, hi), axis=-2), None)
    return full(Chain(tuple(nodes), ch.batch_size))


# --------------------------------------------------------------------------
# inner product and norm -- core.py:362-391, arithmetic.py:189-193
# --------------------------------------------------------------------------

def chain_dot(a: Chain, b: Chain):
    if a.shape != b.shape:
        raise OracleError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.batch_size != b.batch_size:
        raise OracleError("operands must agree on batching")
    if a.batch_size is None:
        m = np.ones((1, 1))
        for k in range(a.ndim):
            m = np.einsum("ab,aic,bid->cd", m, tt_core(a, k), tt_core(b, k),
                          optimize=True)
        return float(m[0, 0])
    m = np.ones((a.batch_size, 1, 1))
    for k in range(a.ndim):
        m = np.einsum("xab,xaic,xbid->xcd", m, tt_core(a, k), tt_core(b, k),
                      optimize=True)
    return m[:, 0, 0].copy()


def chain_dot_loop(a: Chain, b: Chain) -> np.ndarray:
    """Batched dot as a loop of unbatched dots (the faster CPU form, §3.3)."""
    out = np.empty(a.batch_size)
    for e in range(a.batch_size):
        out[e] = chain_dot(batch_element(a, e), batch_element(b, e))
    return out


def norm(ch: Chain):
    sq = chain_dot(ch, ch)
    if ch.batch_size is not None:
        return np.sqrt(np.maximum(sq, 0.0))
    return float(np.sqrt(max(sq, 0.0)))


def batch_element(ch: Chain, e: int) -> Chain:
    return Chain(tuple(Node(n.kind, n.core[e], None if n.factor is None else n.factor[e])
                       for n in ch.nodes), None)


def batch_slice(ch: Chain, lo: int, hi: int) -> Chain:
    return Chain(tuple(Node(n.kind, n.core[lo:hi],
                            None if n.factor is None else n.factor[lo:hi])
                       for n in ch.nodes), hi - lo)


# --------------------------------------------------------------------------
# entry evaluation -- core.py:394-460
# --------------------------------------------------------------------------

def normalize_indices(ch: Chain, indices) -> np.ndarray:
    """Shape check, negative wrap and per-mode bound check in mode order
    (core.py:402-416).  Raises for the lowest mode holding a bad index."""
    idx = np.asarray(indices)
    if idx.ndim == 1:
        idx = idx[None, :]
    if idx.ndim != 2 or idx.shape[1] != ch.ndim:
        raise OracleError(f"index array must be (M, {ch.ndim}), got {idx.shape}")
    out = idx.copy()
    for k, size in enumerate(ch.shape):
        col = out[:, k]
        col = np.where(col < 0, col + size, col)
        if col.size and (col.min() < 0 or col.max() >= size):
            raise OracleError(f"index out of bounds on mode {k}")
        out[:, k] = col
    return out


def _bucket_step(v: np.ndarray, g: np.ndarray, col: np.ndarray, batched: bool):
    """One mode step: group samples by index value so each group is a real
    matrix product (core.py:432-460)."""
    jsz = g.shape[-2]
    order = np.argsort(col, kind="stable")
    edges = np.searchsorted(col[order], np.arange(jsz + 1))
    if batched:
        out = np.empty((v.shape[0], v.shape[1], g.shape[-1]))
    else:
        out = np.empty((v.shape[0], g.shape[-1]))
    for j in range(jsz):
        lo, hi = edges[j], edges[j + 1]
        if lo == hi:
            continue
        rows = order[lo:hi]
        if batched:
            out[rows] = np.einsum("mbr,brs->mbs", v[rows], g[:, :, j, :])
        else:
            out[rows] = v[rows] @ g[:, j, :]
    return out


def entries(ch: Chain, indices) -> np.ndarray:
    idx = normalize_indices(ch, indices)
    m = idx.shape[0]
    if ch.batch_size is None:
        v = np.ones((m, 1))
        for k in range(ch.ndim):
            v = _bucket_step(v, tt_core(ch, k), idx[:, k], False)
        return v[:, 0].copy()
    v = np.ones((m, ch.batch_size, 1))
    for k in range(ch.ndim):
        v = _bucket_step(v, tt_core(ch, k), idx[:, k], True)
    return v[:, :, 0].copy()


# --------------------------------------------------------------------------
# independent brute force for tiny shapes (restates the idea of the
# reference test oracle, pkg/tests/oracles.py:18-73: explicit summation over
# every tuple of edge-rank values, no unfolding GEMMs)
# --------------------------------------------------------------------------

def dense_bruteforce(ch: Chain) -> np.ndarray:
    if ch.batch_size is not None:
        return np.stack([dense_bruteforce(batch_element(ch, e))
                         for e in range(ch.batch_size)])
    if int(np.prod(ch.shape)) > 10**6:
        raise OracleError("brute-force oracle limited to 1e6 entries")
    n = ch.ndim
    ranks = rank_chain(ch)
    out = np.zeros(ch.shape)

    def vec(k, a, b):
        node = ch.nodes[k]
        if node.kind == TT:
            v = node.core[a, :, b]
        elif n == 1:
            v = node.core.sum(axis=1)
        elif k == 0:
            v = node.core[:, b]
        elif k == n - 1:
            v = node.core[:, a]
        else:
            v = node.core[:, a] if a == b else np.zeros(node.core.shape[0])
        return v if node.factor is None else node.factor @ v

    import itertools
    for inner in itertools.product(*[range(r) for r in ranks[1:-1]]):
        edge = (0,) + inner + (0,)
        acc = vec(0, edge[0], edge[1])
        for k in range(1, n):
            acc = np.multiply.outer(acc, vec(k, edge[k], edge[k + 1]))
        out += acc
    return out


# --------------------------------------------------------------------------
# seeded generators (restating random.py:14-40 and SURVEY §8(d))
# --------------------------------------------------------------------------

def default_seed() -> int:
    """TNTZ_SEED convention (config.py:5-18)."""
    return int(os.environ.get("TNTZ_SEED", "0"))


def random_tt(shape: Sequence[int], ranks, seed=None, batch_size=None,
              scale: float = 1.0, dtype=np.float32) -> list:
    """Cores of random.py:28-40 (``scale * standard_normal`` per mode, one
    default_rng stream), cast to ``dtype``.  Returns a list of TT cores."""
    rng = np.random.default_rng(default_seed() if seed is None else int(seed))
    n = len(shape)
    if np.isscalar(ranks):
        ranks = [int(ranks)] * (n - 1)
    ranks = [1] + [int(r) for r in ranks] + [1]
    cores = []
    for k, isz in enumerate(shape):
        dims = (ranks[k], isz, ranks[k + 1])
        if batch_size is not None:
            dims = (batch_size,) + dims
        cores.append((scale * rng.standard_normal(dims)).astype(dtype))
    return cores


def cfg5_nodes(seed=None, dtype=np.float32) -> list:
    """Hybrid CP-TT-Tucker config 5: for k=0..7 draw the core
    then the factor, each standard_normal * 24**-0.5; modes 0-3 TT rank 24,
    modes 4-7 CP rank 24, factor (128, 16) everywhere."""
    rng = np.random.default_rng(default_seed() if seed is None else int(seed))
    s = 24 ** -0.5
    nodes = []
    for k in range(8):
        if k < 4:
            dims = (1 if k == 0 else 24, 16, 24)
            core = (rng.standard_normal(dims) * s).astype(dtype)
            kind = TT
        else:
            core = (rng.standard_normal((16, 24)) * s).astype(dtype)
            kind = CP
        fac = (rng.standard_normal((128, 16)) * s).astype(dtype)
        nodes.append((kind, core, fac))
    return nodes


def uniform_indices(shape: Sequence[int], m: int, seed: int) -> np.ndarray:
    """int64 [m, N] uniform per mode."""
    rng = np.random.default_rng(seed)
    if len(set(shape)) == 1:
        return rng.integers(0, shape[0], size=(m, len(shape)), dtype=np.int64)
    return np.stack([rng.integers(0, s, size=m, dtype=np.int64) for s in shape], axis=1)


def rel_errors(got, ref) -> dict:
    """Acceptance metrics of SURVEY §8(c): relative Frobenius error and
    max|diff| / max|ref| (plus elementwise stats for information)."""
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    d = got - ref
    nref = np.linalg.norm(ref)
    mref = np.abs(ref).max() if ref.size else 0.0
    return {
        "rel_fro": float(np.linalg.norm(d) / nref) if nref > 0 else float(np.linalg.norm(d)),
        "max_rel": float(np.abs(d).max() / mref) if mref > 0 else float(np.abs(d).max() if d.size else 0.0),
    }
