"""Blended CP / TT / Tucker chains held on a B200, contracted by libtnb.

Drop-in for the reference's core model and hot path
(/root/reference/pkg/src/tntz/core.py):

============================  ==========================================
reference                     here
============================  ==========================================
ModeNode      core.py:41-99   :class:`ModeNode` (same kinds, shapes, checks)
TnTensor      core.py:102-241 :class:`TnTensor` (same validation/messages)
promote_cp_node core.py:266   :func:`promote_cp_node` (K0 kernel)
node_tt_core  core.py:307     :func:`node_tt_core` (K0 kernel)
full          core.py:337     :func:`full` (K2: step kernels + one GEMM)
chain_dot     core.py:362     :func:`chain_dot` (K3)
norm          core.py:387     :func:`norm` (K3)
entries       core.py:394     :func:`entries` (K1)
============================  ==========================================

Intended deviations (BASELINE north_star): values are fp32 (the reference
upcasts to float64, core.py:37-38) and results are CUDA ``torch.Tensor``s
(unbatched ``dot``/``norm`` still return a Python ``float``).  Cores are
repacked once per tensor into the kernels' layout (K0) and cached; values
are immutable, exactly as the reference requires, so the
cache never goes stale.
"""

from __future__ import annotations

import ctypes
import os
import time
from typing import Iterable, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import ContractViolationError, StructuralError

TT = "tt"
CP = "cp"

INTERIOR = "interior"
LEFT_BOUNDARY = "left_boundary"
RIGHT_BOUNDARY = "right_boundary"

_POS = {INTERIOR: N.POS_INTERIOR, LEFT_BOUNDARY: N.POS_LEFT, RIGHT_BOUNDARY: N.POS_RIGHT}


def _default_device() -> torch.device:
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


_DTYPES = (torch.float32, torch.float64)


def _as_f32(a, dtype=torch.float32) -> torch.Tensor:
    """``dtype`` (fp32 by default, float64 for the reference-precision
    instantiation), contiguous, on the current CUDA device when one exists."""
    if dtype not in _DTYPES:
        raise ContractViolationError(f"dtype must be torch.float32 or torch.float64, got {dtype}")
    if isinstance(a, torch.Tensor):
        t = a.detach()
        dev = t.device if t.device.type == "cuda" else _default_device()
    else:
        np_dt = np.float64 if dtype == torch.float64 else np.float32
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np_dt)))
        dev = _default_device()
    return t.to(device=dev, dtype=dtype).contiguous()


class ModeNode:
    """One node of the chain: a core plus an optional basis factor
    (core.py:41-99).  ``kind`` is ``"tt"`` (``r_left x I x r_right``) or
    ``"cp"`` (``I x R``); batched nodes carry one extra leading axis."""

    __slots__ = ("kind", "core", "factor", "batched")

    def __init__(self, kind: str, core, factor=None, batched: bool = False, dtype=torch.float32):
        if kind not in (TT, CP):
            raise ContractViolationError(f"unknown node kind {kind!r}")
        core = _as_f32(core, dtype)
        expected = (3 if kind == TT else 2) + (1 if batched else 0)
        if core.dim() != expected:
            raise StructuralError(
                f"{kind} core must have {expected} axes, got shape {tuple(core.shape)}")
        if factor is not None:
            factor = _as_f32(factor, dtype)
            if factor.dim() != 2 + (1 if batched else 0):
                raise StructuralError(
                    f"factor must have {2 + batched} axes, got shape {tuple(factor.shape)}")
            if factor.shape[-1] != core.shape[-2]:
                raise StructuralError(
                    f"factor maps onto internal size {factor.shape[-1]}, "
                    f"core has internal size {core.shape[-2]}")
            if factor.device != core.device:
                factor = factor.to(core.device)
        self.kind = kind
        self.core = core
        self.factor = factor
        self.batched = bool(batched)

    @property
    def internal_size(self) -> int:
        return int(self.core.shape[-2])

    @property
    def physical_size(self) -> int:
        if self.factor is not None:
            return int(self.factor.shape[-2])
        return self.internal_size

    @property
    def cp_rank(self) -> int:
        if self.kind != CP:
            raise ContractViolationError("cp_rank is only defined for CP nodes")
        return int(self.core.shape[-1])

    @property
    def dtype(self) -> torch.dtype:
        return self.core.dtype

    def copy(self) -> "ModeNode":
        return ModeNode(self.kind, self.core, self.factor, self.batched, dtype=self.core.dtype)

    def _native(self) -> N.TnbNode:
        nd = N.TnbNode()
        nd.kind = N.KIND_TT if self.kind == TT else N.KIND_CP
        nd.internal = self.internal_size
        nd.phys = self.physical_size
        if self.kind == TT:
            nd.r_left, nd.r_right = int(self.core.shape[-3]), int(self.core.shape[-1])
        else:
            nd.r_left = nd.r_right = self.cp_rank
        nd.core = self.core.data_ptr()
        nd.factor = self.factor.data_ptr() if self.factor is not None else None
        return nd

    def __repr__(self):
        f = "" if self.factor is None else f", factor{tuple(self.factor.shape)}"
        return f"ModeNode({self.kind}, core{tuple(self.core.shape)}{f})"


class _Packed:
    """Device-resident repacked chain (K0 output) plus its C descriptor."""

    __slots__ = ("chain", "modes", "buffers", "device", "n")

    def __init__(self, chain, modes, buffers, device, n):
        self.chain, self.modes, self.buffers, self.device, self.n = chain, modes, buffers, device, n


class TnTensor:
    """An N-mode tensor stored as a chain of TT/CP nodes (core.py:102-241)."""

    __slots__ = ("_nodes", "_batch_size", "_pack")

    def __init__(self, nodes: Iterable[ModeNode], batch_size: Optional[int] = None):
        nodes = tuple(n.copy() for n in nodes)
        if len(nodes) == 0:
            raise ContractViolationError("a tensor needs at least one mode")
        if batch_size is not None and batch_size < 1:
            raise ContractViolationError("batch size must be >= 1")
        for k, node in enumerate(nodes):
            if batch_size is None:
                if node.batched:
                    raise StructuralError(f"node {k} is batched but the tensor is not")
            else:
                if not node.batched:
                    raise StructuralError(f"node {k} lacks the batch axis")
                if node.core.shape[0] != batch_size:
                    raise StructuralError(
                        f"node {k} has batch {node.core.shape[0]}, expected {batch_size}")
                if node.factor is not None and node.factor.shape[0] != batch_size:
                    raise StructuralError(f"node {k} factor has a mismatched batch")
        ranks = _rank_chain(nodes)
        if ranks[0] != 1 or ranks[-1] != 1:
            raise StructuralError(f"boundary ranks must be 1, got {ranks[0]}, {ranks[-1]}")
        dt = nodes[0].dtype
        if any(n.dtype != dt for n in nodes):
            raise ContractViolationError("all nodes must share one dtype (float32 or float64)")
        dev = nodes[0].core.device
        if any(n.core.device != dev for n in nodes):
            nodes = tuple(ModeNode(n.kind, n.core.to(dev),
                                   None if n.factor is None else n.factor.to(dev), n.batched, dtype=dt)
                          for n in nodes)
        self._nodes = nodes
        self._batch_size = batch_size
        self._pack = None

    # -- metadata (core.py:139-172) ---------------------------------------
    @property
    def nodes(self) -> tuple:
        return self._nodes

    @property
    def batch_size(self) -> Optional[int]:
        return self._batch_size

    @property
    def dtype(self) -> torch.dtype:
        """torch.float32 (the hot path) or torch.float64 (the reference's
        precision, generic kernels)."""
        return self._nodes[0].dtype

    def to(self, dtype) -> "TnTensor":
        """The same chain with values in ``dtype`` (float32 / float64)."""
        if dtype == self.dtype:
            return self
        return TnTensor([ModeNode(n.kind, n.core, n.factor, n.batched, dtype=dtype) for n in self._nodes],
                        self._batch_size)

    def double(self) -> "TnTensor":
        return self.to(torch.float64)

    def float(self) -> "TnTensor":
        return self.to(torch.float32)

    # tntorch spellings (tntorch.Tensor): the per-mode cores and the Tucker
    # factors (None where a mode has none); views of the nodes' tensors
    @property
    def cores(self) -> list:
        return [n.core for n in self._nodes]

    @property
    def Us(self) -> list:
        return [n.factor for n in self._nodes]

    def numpy(self):
        """The dense tensor as a float64 ndarray (tntorch ``Tensor.numpy``)."""
        return full(self).cpu().double().numpy()

    @property
    def ndim(self) -> int:
        return len(self._nodes)

    @property
    def shape(self) -> tuple:
        return tuple(n.physical_size for n in self._nodes)

    @property
    def ranks(self) -> list:
        return _rank_chain(self._nodes)

    @property
    def device(self) -> torch.device:
        return self._nodes[0].core.device

    def numel(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.ndim else 0

    def dof(self) -> int:
        b = self._batch_size or 1
        total = 0
        for n in self._nodes:
            total += n.core.numel() // b
            if n.factor is not None:
                total += n.factor.numel() // b
        return total

    # -- conversions --------------------------------------------------------
    def full(self, *, lead: Optional[tuple] = None) -> torch.Tensor:
        return full(self, lead=lead)

    def norm(self):
        return norm(self)

    def batch_element(self, b: int) -> "TnTensor":
        if self._batch_size is None:
            raise ContractViolationError("tensor is not batched")
        nodes = [ModeNode(n.kind, n.core[b], None if n.factor is None else n.factor[b], dtype=n.dtype)
                 for n in self._nodes]
        return TnTensor(nodes)

    def __repr__(self):
        kinds = "".join("T" if n.kind == TT else "C" for n in self._nodes)
        b = "" if self._batch_size is None else f", batch={self._batch_size}"
        return f"TnTensor(shape={self.shape}, ranks={self.ranks}, kinds={kinds}{b})"

    def __getitem__(self, key):
        from . import indexing

        return indexing.getitem(self, key)

    # -- K0: repack once, cache (values are immutable) ------------------------
    def _packed(self) -> _Packed:
        if self._pack is not None:
            return self._pack
        dev = self.device
        N.require_device(dev)
        lib = N.load()
        n = self.ndim
        nodes = (N.TnbNode * n)(*[nd._native() for nd in self._nodes])
        modes = (N.TnbMode * n)()
        N.check(lib.tnb_plan_modes(nodes, n, modes), "plan")
        batch = self._batch_size or 0
        bufs = []
        for k in range(n):
            cnt = lib.tnb_mode_floats(ctypes.byref(modes[k]), batch)
            buf = torch.empty(max(cnt, 1), dtype=self.dtype, device=dev)
            modes[k].slices = buf.data_ptr()
            bufs.append(buf)
        repack = lib.tnb_repack_f64 if self.dtype == torch.float64 else lib.tnb_repack_f32
        with torch.cuda.device(dev):
            N.check(repack(nodes, n, batch, modes, N.stream_ptr(dev)), "repack")
        chain = N.TnbChain(n, 0, batch, ctypes.cast(modes, ctypes.POINTER(N.TnbMode)))
        self._pack = _Packed(chain, modes, bufs, dev, n)
        return self._pack


TnTensor.torch = TnTensor.full  # tntorch spelling of full()


# ---------------------------------------------------------------------------
# rank bookkeeping (core.py:244-263)

def _node_ranks(node: ModeNode, k: int, n_modes: int) -> tuple:
    if node.kind == TT:
        return int(node.core.shape[-3]), int(node.core.shape[-1])
    r = node.cp_rank
    return (1 if k == 0 else r), (1 if k == n_modes - 1 else r)


def _rank_chain(nodes: Sequence[ModeNode]) -> list:
    n = len(nodes)
    pairs = [_node_ranks(node, k, n) for k, node in enumerate(nodes)]
    for k in range(n - 1):
        if pairs[k][1] != pairs[k + 1][0]:
            raise StructuralError(
                f"rank mismatch between modes {k} and {k + 1}: "
                f"{pairs[k][1]} vs {pairs[k + 1][0]}")
    return [pairs[0][0]] + [p[1] for p in pairs]


# ---------------------------------------------------------------------------
# per-node preparation (core.py:266-334), on the device

def promote_cp_node(node: ModeNode, position: str) -> torch.Tensor:
    """TT core equivalent of a CP node at a chain position (core.py:266-296)."""
    if node.kind != CP:
        raise ContractViolationError("promote_cp_node expects a CP node")
    if position not in _POS:
        raise ContractViolationError(f"unknown position {position!r}")
    dev = node.core.device
    N.require_device(dev)
    r, i = node.cp_rank, node.internal_size
    b = int(node.core.shape[0]) if node.batched else 0
    shape = {INTERIOR: (r, i, r), LEFT_BOUNDARY: (1, i, r), RIGHT_BOUNDARY: (r, i, 1)}[position]
    out = torch.empty(((b,) if b else ()) + shape, dtype=node.dtype, device=dev)
    nd = ModeNode(CP, node.core, None, node.batched, dtype=node.dtype)._native()
    fn = N.load().tnb_promote_cp_f64 if node.dtype == torch.float64 else N.load().tnb_promote_cp_f32
    with torch.cuda.device(dev):
        N.check(fn(ctypes.byref(nd), _POS[position], b, out.data_ptr(), N.stream_ptr(dev)), "promote_cp_node")
    return out


def node_tt_core(t: TnTensor, k: int) -> torch.Tensor:
    """Effective TT core of mode k, CP promoted and factor absorbed
    (core.py:307-327), in the reference layout (r_l, J, r_r)."""
    if not 0 <= k < t.ndim:
        raise ContractViolationError(f"mode {k} out of range")
    p = t._packed()
    m = p.modes[k]
    b = t.batch_size
    shape = (m.r_left, m.phys, m.r_right)
    out = torch.empty(((b,) if b else ()) + shape, dtype=t.dtype, device=p.device)
    fn = N.load().tnb_tt_core_f64 if t.dtype == torch.float64 else N.load().tnb_tt_core_f32
    with torch.cuda.device(p.device):
        N.check(fn(ctypes.byref(p.chain), k, out.data_ptr(), N.stream_ptr(p.device)), "node_tt_core")
    return out


# ---------------------------------------------------------------------------
# K2: dense decompression (core.py:337-359)

def full(t: TnTensor, *, lead: Optional[tuple] = None) -> torch.Tensor:
    """Dense C-order tensor (leading batch axis if batched).

    ``lead=(lo, hi)`` (extension) returns only the slab whose leading index
    lies in [lo, hi), i.e. the reference's ``full(t[lo:hi])``."""
    p = t._packed()
    shape = t.shape
    lo, hi = (0, shape[0]) if lead is None else (int(lead[0]), int(lead[1]))
    if not (0 <= lo <= hi <= shape[0]):
        raise ContractViolationError(f"slab [{lo}, {hi}) outside mode 0 of size {shape[0]}")
    oshape = (hi - lo,) + tuple(shape[1:])
    if t.batch_size is not None:
        oshape = (t.batch_size,) + oshape
    out = torch.empty(oshape, dtype=t.dtype, device=p.device)
    lib = N.load()
    f64 = t.dtype == torch.float64
    wsb = (lib.tnb_full_workspace_bytes_f64 if f64 else lib.tnb_full_workspace_bytes)(ctypes.byref(p.chain), lo, hi)
    if wsb < 0:
        N.check(N.TNB_EINVAL, "full")
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=p.device)
    with torch.cuda.device(p.device):
        N.check((lib.tnb_full_f64 if f64 else lib.tnb_full_f32)(
            ctypes.byref(p.chain), lo, hi, out.data_ptr(), ws.data_ptr(), wsb, N.stream_ptr(p.device)), "full")
    return out


# ---------------------------------------------------------------------------
# K3: inner product and norm (core.py:362-391)

def chain_dot(a: TnTensor, b: TnTensor):
    if a.shape != b.shape:
        raise ContractViolationError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.batch_size != b.batch_size:
        raise ContractViolationError("operands must agree on batching")
    if a.dtype != b.dtype:
        raise ContractViolationError(f"operands must share a dtype: {a.dtype} vs {b.dtype}")
    pa, pb = a._packed(), b._packed()
    if pa.device != pb.device:
        raise ContractViolationError("operands live on different devices")
    out = torch.empty(a.batch_size or 1, dtype=a.dtype, device=pa.device)
    fn = N.load().tnb_dot_f64 if a.dtype == torch.float64 else N.load().tnb_dot_f32
    with torch.cuda.device(pa.device):
        N.check(fn(ctypes.byref(pa.chain), ctypes.byref(pb.chain), out.data_ptr(), N.stream_ptr(pa.device)),
                "chain_dot")
    if a.batch_size is None:
        return float(out[0].item())
    return out


def norm(t: TnTensor):
    p = t._packed()
    out = torch.empty(t.batch_size or 1, dtype=t.dtype, device=p.device)
    fn = N.load().tnb_norm_f64 if t.dtype == torch.float64 else N.load().tnb_norm_f32
    with torch.cuda.device(p.device):
        N.check(fn(ctypes.byref(p.chain), out.data_ptr(), N.stream_ptr(p.device)), "norm")
    if t.batch_size is None:
        return float(out[0].item())
    return out


# ---------------------------------------------------------------------------
# K1: entry evaluation (core.py:394-460)

def _index_tensor(t: TnTensor, indices, device) -> torch.Tensor:
    """Shape/dtype normalisation of core.py:402-408; returns a 2-D tensor."""
    if isinstance(indices, torch.Tensor):
        idx = indices.detach()
    else:
        idx = torch.from_numpy(np.ascontiguousarray(np.asarray(indices)))
    if idx.dim() == 1:
        idx = idx[None, :]
    if idx.dim() != 2 or idx.shape[1] != t.ndim:
        raise ContractViolationError(
            f"index array must be (M, {t.ndim}), got {tuple(idx.shape)}")
    if idx.dtype.is_floating_point:
        # the reference lets float indices through entries(): negatives wrap,
        # bounds are checked on the float values, and the searchsorted
        # bucketing floors them (core.py:409-416, 435-437)
        idx = idx.to(device=device, dtype=torch.float64)
        size = torch.tensor(t.shape, dtype=torch.float64, device=device)
        idx = torch.where(idx < 0, idx + size, idx)
        if idx.numel():
            bad = ((idx < 0) | (idx >= size)).any(dim=0).nonzero()
            if bad.numel():
                raise ContractViolationError(f"index out of bounds on mode {int(bad[0, 0])}")
        idx = torch.floor(idx)
    return idx.to(device=device, dtype=torch.int64).contiguous()


# host index matrices at least 2 * _PIPELINE_ROWS long are streamed in
# chunks of _CHUNK_ROWS (H2D of chunk i+1 overlaps the kernels of chunk i);
# 2^21 rows and up: an 8-way shard of the 2^24 cfg2 tuples still pipelines
_PIPELINE_ROWS = 1 << 20
_CHUNK_ROWS = 1 << 20

# what the last pipelined entries() call moved over PCIe (bench.py's e2e
# byte counts): {"h2d_bytes", "d2h_bytes", "codec"}
last_transfer: dict = {}


def _codec_width(t: TnTensor) -> int:
    """Width of the index transport codec for this chain (include/tnb.h):
    1 (int8) when every mode has <= 128 entries, 2 (int16) up to 32768, else
    0 (no codec).  Valid indices lie in [-J, J); anything else either fails
    the host range check (the chunk is then sent as int64) or is reported by
    the device prep kernel exactly as without the codec."""
    if os.environ.get("TNB_E2E_CODEC", "1") == "0":
        return 0
    jmax = max(t.shape)
    return 1 if jmax <= 128 else (2 if jmax <= 32768 else 0)


class _Narrower:
    """Background host thread of the index transport codec: narrows the
    chunks the pipeline sends narrowed, in order, into a ring of pinned
    staging buffers, while the calling thread enqueues copies and launches
    (ctypes releases the GIL during tnb_narrow_indices_host).  A staging
    buffer is refilled only after the H2D that read it has completed."""

    def __init__(self, idx_host, spans, stage, width, nthreads):
        import threading

        self.idx, self.spans, self.stage, self.width, self.nt = idx_host, spans, stage, width, nthreads
        k = len(spans)
        self.ready = [threading.Event() for _ in range(k)]
        self.recorded = [threading.Event() for _ in range(k)]
        self.landed = [None] * k
        self.fits = [False] * k
        self.stop = False
        self.error = None
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        nst = len(self.stage)
        try:
            for k, (lo, hi) in enumerate(self.spans):
                if k >= nst:
                    self.recorded[k - nst].wait()
                    if self.landed[k - nst] is not None:
                        self.landed[k - nst].synchronize()
                if self.stop:
                    return
                cnt = (hi - lo) * self.idx.shape[1]
                self.fits[k] = N.narrow_indices(self.idx[lo:hi].view(-1), self.stage[k % nst][:cnt], self.width,
                                                self.nt)
                self.ready[k].set()
        except BaseException as e:  # noqa: BLE001  (re-raised by the caller)
            self.error = e
            for r in self.ready:
                r.set()

    def get(self, k):
        """(staging buffer, fits) of narrowed chunk k, once narrowed."""
        self.ready[k].wait()
        if self.error is not None:
            raise self.error
        return self.stage[k % len(self.stage)], self.fits[k]

    def released(self, k, event):
        """The H2D of chunk k's staging buffer was enqueued; ``event`` marks
        its completion (None: the buffer was not read)."""
        self.landed[k] = event
        self.recorded[k].set()

    def close(self):
        self.stop = True
        for r in self.recorded:
            r.set()
        self.th.join()


def _entries_pipelined_dyn(t: TnTensor, p: _Packed, idx_host: torch.Tensor, algo: int,
                           out_host: Optional[torch.Tensor], width: int, chunk: int) -> torch.Tensor:
    """The self-balancing form of the pipelined host path (default when the
    index codec applies).  The two host resources that feed the GPU -- the DMA
    engine reading pinned int64 chunks and the host cores narrowing chunks to
    int8/int16 -- each take the next chunk they can: the calling thread sends
    RAW chunks from the front of the matrix whenever fewer than two raw copies
    are queued, the narrowing thread works from the BACK, and finished
    narrowed chunks are sent as they appear, until the two meet.  No chunk
    waits for the slower resource and the split adapts to the machine (a
    fixed raw fraction, TNB_E2E_DYNAMIC=0, has to be tuned per host: 0.35
    here, 0.5 on a box with slower cores).  Chunks are independent, so their
    order on the GPU does not matter; every launch sees `chunk` rows."""
    import queue
    import threading

    dev = p.device
    m = int(idx_host.shape[0])
    n = t.ndim
    nch = (m + chunk - 1) // chunk
    out = torch.empty(nch * chunk, dtype=torch.float32, device=dev)
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    back = torch.cuda.Stream(dev) if out_host is not None else None
    errs = torch.empty(nch, dtype=torch.int32, device=dev)
    bufs = [torch.empty((chunk, n), dtype=torch.int64, device=dev) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]  # compute finished with buffer b
    ndt = torch.int8 if width == 1 else torch.int16
    nstage = 4
    stage = [torch.empty(chunk * n, dtype=ndt, pin_memory=True) for _ in range(nstage)]
    dnar = [torch.empty(chunk * n, dtype=ndt, device=dev) for _ in range(2)]
    lib = N.load()
    # the enqueueing thread polls here and the CUDA driver has its own: leaving
    # them a few hardware threads measured steadier than using all but one
    nthreads = int(os.environ.get("TNB_E2E_THREADS", "0")) or max(1, lib.tnb_host_threads() * 3 // 4)
    spans = [(c * chunk, min(m, (c + 1) * chunk)) for c in range(nch)]

    lock = threading.Lock()
    ends = [0, nch - 1]  # next raw chunk (front), next chunk to narrow (back)
    ready: "queue.Queue" = queue.Queue()
    free = [threading.Event() for _ in range(nstage)]  # staging buffer may be refilled ...
    landed = [None] * nstage                              # ... once this H2D event has completed
    for f in free:
        f.set()
    state = {"stop": False, "error": None, "wait_ms": 0.0, "narrow_ms": 0.0}

    def claim(front: bool):
        with lock:
            if ends[0] > ends[1]:
                return None
            if front:
                ends[0] += 1
                return ends[0] - 1
            ends[1] -= 1
            return ends[1] + 1

    def narrower():
        k = 0
        try:
            while not state["stop"]:
                sb = k % nstage
                t0 = time.perf_counter()
                free[sb].wait()
                if state["stop"]:
                    return
                if landed[sb] is not None:
                    landed[sb].synchronize()
                c = claim(False)
                if c is None:
                    return
                free[sb].clear()
                lo, hi = spans[c]
                cnt = (hi - lo) * n
                t1 = time.perf_counter()
                fits = N.narrow_indices(idx_host[lo:hi].view(-1), stage[sb][:cnt], width, nthreads)
                t2 = time.perf_counter()
                state["wait_ms"] += (t1 - t0) * 1e3
                state["narrow_ms"] += (t2 - t1) * 1e3
                ready.put((c, sb, fits))
                k += 1
        except BaseException as e:  # noqa: BLE001  (re-raised by the caller)
            state["error"] = e
        finally:
            ready.put(None)  # the narrower is done

    th = threading.Thread(target=narrower, daemon=True)
    th.start()
    ws = None
    copy.wait_stream(comp)
    h2d = 0
    codecs = set()
    raw_events: list = []
    sent = 0
    narrower_done = False

    def dispatch(c, sb, narrow):
        nonlocal ws, h2d, sent
        lo, hi = spans[c]
        b = sent & 1
        buf = bufs[b]
        cnt = (hi - lo) * n
        with torch.cuda.stream(copy):
            if sent >= 2:
                copy.wait_event(done[b])
            if narrow:
                dnar[b][:cnt].copy_(stage[sb][:cnt], non_blocking=True)
                h2d += cnt * width
                codecs.add(f"int{8 * width}")
            else:
                buf[: hi - lo].copy_(idx_host[lo:hi], non_blocking=True)
                h2d += cnt * 8
                codecs.add("int64")
            ev = torch.cuda.Event()
            ev.record(copy)
            if hi - lo < chunk:
                buf[hi - lo:].zero_()
            ready_ev = torch.cuda.Event()
            ready_ev.record(copy)
        if sb is not None:  # the staging buffer is free once this copy (if any) has read it
            landed[sb] = ev if narrow else None
            free[sb].set()
        if not narrow:
            raw_events.append(ev)
        comp.wait_event(ready_ev)
        buf.record_stream(comp)
        if narrow:
            dnar[b].record_stream(comp)
            N.check(lib.tnb_widen_indices(dnar[b].data_ptr(), width, cnt, buf.data_ptr(), N.stream_ptr(dev)),
                    "widen indices")
        ws = launch_entries(p, buf, out[lo:lo + chunk], errs[c:c + 1], algo, ws)
        done[b].record(comp)
        if back is not None:
            back.wait_event(done[b])
            with torch.cuda.stream(back):
                out_host[lo:hi].copy_(out[lo:hi], non_blocking=True)
        sent += 1

    try:
        while sent < nch:
            item = None
            if not narrower_done:
                try:
                    item = ready.get_nowait()
                except queue.Empty:
                    item = False
                if item is None:
                    narrower_done = True
                    if state["error"] is not None:
                        raise state["error"]
                    continue
            if item:
                c, sb, fits = item
                dispatch(c, sb, fits)  # a chunk with a value outside the narrow range crosses as int64
                continue
            raw_events[:] = [e for e in raw_events if not e.query()]
            if len(raw_events) < 2:
                c = claim(True)
                if c is not None:
                    dispatch(c, None, False)
                    continue
                if narrower_done:
                    break  # nothing left to claim: every chunk was dispatched
            if not narrower_done:
                try:
                    item = ready.get(timeout=0.0002)
                except queue.Empty:
                    continue
                if item is None:
                    narrower_done = True
                    if state["error"] is not None:
                        raise state["error"]
                else:
                    dispatch(*item)
            else:
                time.sleep(0.0001)
    finally:
        state["stop"] = True
        for f in free:
            f.set()
        th.join()
    code = int(errs.min().item())
    if back is not None:
        back.synchronize()
    last_transfer.clear()
    last_transfer.update(h2d_bytes=h2d, d2h_bytes=m * 4 if back is not None else 0,
                         codec="+".join(sorted(codecs)), narrow_ms=round(state["narrow_ms"], 2),
                         narrow_wait_ms=round(state["wait_ms"], 2))
    if code < t.ndim:
        raise ContractViolationError(f"index out of bounds on mode {code}")
    return out_host if out_host is not None else out[:m]


def _entries_pipelined(t: TnTensor, p: _Packed, idx_host: torch.Tensor, algo: int,
                       out_host: Optional[torch.Tensor] = None) -> torch.Tensor:
    """entries() for a large PINNED int64 host index matrix: chunked
    copy-stream H2D overlapped with the K1 launches on the compute stream;
    with a pinned host ``out_host`` each chunk's values are copied back on a
    second copy stream (PCIe is full duplex) behind the next chunk's work.

    PCIe is the bound of this path, so most chunks cross it narrowed by the
    index transport codec (int64 -> int8/int16 on host threads, a pure range
    check; ``tnb_narrow_indices_host``, run ahead by a background thread) and
    are widened back on the device (``tnb_widen_indices``) before the
    unchanged K1 launch.  Two host resources feed the GPU -- the DMA engine
    reading pinned memory (~56 GB/s of int64) and the host cores narrowing
    (~86 GB/s of int64 read on 16 threads) -- so a fraction of the chunks
    (TNB_E2E_RAW_FRAC, default 0.35) crosses raw with no host work, spread
    evenly and starting with chunk 0 so the copy engine starts at once.  A
    chunk with a value outside the narrow range crosses as int64."""
    dev = p.device
    m = int(idx_host.shape[0])
    n = t.ndim
    chunk = 1 << int(os.environ.get("TNB_E2E_CHUNK_LOG2", "0")) if os.environ.get("TNB_E2E_CHUNK_LOG2") \
        else _CHUNK_ROWS
    width = _codec_width(t)
    if width and os.environ.get("TNB_E2E_DYNAMIC", "1") != "0" and "TNB_E2E_RAW_FRAC" not in os.environ:
        return _entries_pipelined_dyn(t, p, idx_host, algo, out_host, width, chunk)
    nch = (m + chunk - 1) // chunk
    # every launch sees exactly `chunk` rows (the short last chunk is padded
    # with index 0), so all chunks run the same plan
    out = torch.empty(nch * chunk, dtype=torch.float32, device=dev)
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    errs = torch.empty(nch, dtype=torch.int32, device=dev)
    bufs = [torch.empty((chunk, n), dtype=torch.int64, device=dev) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]  # compute finished with buffer b
    back = torch.cuda.Stream(dev) if out_host is not None else None
    raw_frac = float(os.environ.get("TNB_E2E_RAW_FRAC", "0.35")) if width else 1.0

    def raw_chunk(c):
        x = raw_frac
        return int((c + 1) * x + 1 - x + 1e-9) > int(c * x + 1 - x + 1e-9)

    spans = [(c * chunk, min(m, (c + 1) * chunk)) for c in range(nch)]
    narrow_k = {}  # chunk -> index among the narrowed chunks
    nar = None
    if width:
        for c in range(nch):
            if not raw_chunk(c):
                narrow_k[c] = len(narrow_k)
    if narrow_k:
        ndt = torch.int8 if width == 1 else torch.int16
        # 4 pinned staging buffers: the narrowing thread never waits for a
        # chunk's H2D queued behind a raw chunk's (the copy stream is FIFO)
        stage = [torch.empty(chunk * n, dtype=ndt, pin_memory=True) for _ in range(4)]
        dnar = [torch.empty(chunk * n, dtype=ndt, device=dev) for _ in range(2)]
        lib = N.load()
        # one hardware thread stays with this (enqueueing) thread
        nthreads = int(os.environ.get("TNB_E2E_THREADS", "0")) or max(1, lib.tnb_host_threads() - 1)
        nar = _Narrower(idx_host, [spans[c] for c in narrow_k], stage, width, nthreads)
    ws = None  # every launch has exactly `chunk` rows: AUTO resolves to one plan for all chunks
    copy.wait_stream(comp)
    h2d = 0
    codecs = set()
    try:
        for c in range(nch):
            lo, hi = spans[c]
            b = c & 1
            buf = bufs[b]
            narrow = False
            if c in narrow_k:
                k = narrow_k[c]
                sbuf, narrow = nar.get(k)
                cnt = (hi - lo) * n
            with torch.cuda.stream(copy):
                if c >= 2:
                    copy.wait_event(done[b])
                if narrow:
                    dnar[b][:cnt].copy_(sbuf[:cnt], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                    nar.released(k, ev)
                    h2d += cnt * width
                    codecs.add(f"int{8 * width}")
                else:
                    if c in narrow_k:
                        nar.released(narrow_k[c], None)  # did not fit: its staging buffer was not read
                    buf[: hi - lo].copy_(idx_host[lo:hi], non_blocking=True)
                    h2d += (hi - lo) * n * 8
                    codecs.add("int64")
                if hi - lo < chunk:
                    buf[hi - lo:].zero_()
                ready = torch.cuda.Event()
                ready.record(copy)
            comp.wait_event(ready)
            buf.record_stream(comp)
            if narrow:
                dnar[b].record_stream(comp)
                N.check(lib.tnb_widen_indices(dnar[b].data_ptr(), width, cnt, buf.data_ptr(),
                                              N.stream_ptr(dev)), "widen indices")
            ws = launch_entries(p, buf, out[lo:lo + chunk], errs[c:c + 1], algo, ws)
            done[b].record(comp)
            if back is not None:
                back.wait_event(done[b])
                with torch.cuda.stream(back):
                    out_host[lo:hi].copy_(out[lo:hi], non_blocking=True)
    finally:
        if nar is not None:
            nar.close()
    code = int(errs.min().item())
    if back is not None:
        back.synchronize()
    last_transfer.clear()
    last_transfer.update(h2d_bytes=h2d, d2h_bytes=m * 4 if back is not None else 0,
                         codec="+".join(sorted(codecs)))
    if code < t.ndim:
        raise ContractViolationError(f"index out of bounds on mode {code}")
    return out_host if out_host is not None else out[:m]


def _check_out(t: TnTensor, p: _Packed, out: torch.Tensor, m: int) -> None:
    b = t.batch_size
    shape = (m, b) if b else (m,)
    if (not isinstance(out, torch.Tensor) or out.dtype != t.dtype or tuple(out.shape) != shape
            or not out.is_contiguous()):
        name = "float64" if t.dtype == torch.float64 else "float32"
        raise ContractViolationError(f"out must be a contiguous {name} tensor of shape {shape}")
    if out.device.type == "cpu":
        if not out.is_pinned():
            raise ContractViolationError("a host out tensor must be in pinned memory")
    elif out.device != p.device:
        raise ContractViolationError(f"out is on {out.device}, the tensor on {p.device}")


def entries(t: TnTensor, indices, *, algo: int = N.ALGO_AUTO,
            out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Values at explicit multi-indices: shape (M,), or (M, B) if batched.

    ``out`` (optional): a contiguous float32 tensor of that shape, either on
    the tensor's device or in PINNED host memory; the values are written
    there and ``out`` is returned (a host ``out`` is complete on return).
    """
    p = t._packed()
    host_out = out is not None and out.device.type == "cpu"
    if (isinstance(indices, torch.Tensor) and indices.device.type == "cpu" and indices.is_pinned()
            and indices.dtype == torch.int64 and indices.dim() == 2 and indices.shape[1] == t.ndim
            and indices.is_contiguous() and indices.shape[0] >= 2 * _PIPELINE_ROWS
            and t.batch_size is None and t.dtype == torch.float32):
        if out is not None:
            _check_out(t, p, out, int(indices.shape[0]))
        res = _entries_pipelined(t, p, indices, algo, out if host_out else None)
        if out is not None and not host_out:
            out.copy_(res)
            return out
        return res
    host_in = isinstance(indices, torch.Tensor) and indices.device.type == "cpu" or \
        not isinstance(indices, torch.Tensor)
    idx = _index_tensor(t, indices, p.device)
    m = int(idx.shape[0])
    b = t.batch_size
    if host_in:
        last_transfer.clear()
        last_transfer.update(h2d_bytes=idx.numel() * 8, d2h_bytes=0, codec="int64")
    if out is not None:
        _check_out(t, p, out, m)
    dev_out = out if (out is not None and not host_out) else \
        torch.empty((m, b) if b else (m,), dtype=t.dtype, device=p.device)
    if m == 0:
        return out if out is not None else dev_out
    err = torch.empty(1, dtype=torch.int32, device=p.device)
    launch_entries(p, idx, dev_out, err, algo)
    if host_out:
        out.copy_(dev_out, non_blocking=True)
    code = int(err.item())
    if host_out:
        torch.cuda.current_stream(p.device).synchronize()
    if code < t.ndim:
        raise ContractViolationError(f"index out of bounds on mode {code}")
    return out if out is not None else dev_out


def launch_entries(p: _Packed, idx: torch.Tensor, out: torch.Tensor, err: torch.Tensor,
                   algo: int = N.ALGO_AUTO, ws: Optional[torch.Tensor] = None):
    """Asynchronous K1 launch on the current stream (no host sync); the
    caller reads ``err`` (>= n_modes means every index was valid)."""
    lib = N.load()
    m = int(idx.shape[0])
    f64 = out.dtype == torch.float64  # the reference-precision instantiation
    wsb = (lib.tnb_entries_workspace_bytes_f64 if f64 else lib.tnb_entries_workspace_bytes)(
        ctypes.byref(p.chain), m, algo)
    if wsb < 0:
        N.check(N.TNB_EINVAL, "entries")
    if wsb > 0 and (ws is None or ws.numel() < wsb):
        ws = torch.empty(wsb, dtype=torch.uint8, device=p.device)
    with torch.cuda.device(p.device):
        N.check((lib.tnb_entries_f64 if f64 else lib.tnb_entries_f32)(
            ctypes.byref(p.chain), idx.data_ptr(), m, out.data_ptr(), err.data_ptr(), algo,
            ws.data_ptr() if wsb > 0 else None, wsb, N.stream_ptr(p.device)), "entries")
    return ws
