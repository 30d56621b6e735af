"""paper_2206_11128_b200 -- B200-native contraction hot path of tntorch
(arXiv 2206.11128): batched entry evaluation ``t[idx]``, dense
decompression ``full()`` and ``dot``/``norm`` between tensor networks in the
blended CP / TT / Tucker format.

The public names mirror the reference package's (tntz/__init__.py:9-36) for
the hot path; compute runs in libtnb.so (hand-written sm_100a CUDA behind the
C ABI of include/tnb.h).  There is no CPU fallback.
"""

from . import arithmetic, callers, indexing, serialization
from .arithmetic import dot
from .core import (
    CP,
    INTERIOR,
    LEFT_BOUNDARY,
    RIGHT_BOUNDARY,
    TT,
    ModeNode,
    TnTensor,
    chain_dot,
    entries,
    full,
    node_tt_core,
    norm,
    promote_cp_node,
)
from .errors import (
    ChecksumError,
    ContractViolationError,
    DataError,
    MagicError,
    NativeError,
    SizeError,
    StructuralError,
    TntzError,
)
from .indexing import getitem
from .serialization import load, read_dense, read_header, save, write_dense

Tensor = TnTensor  # tntorch spelling

__version__ = "0.1.0"

__all__ = [
    "CP", "TT", "INTERIOR", "LEFT_BOUNDARY", "RIGHT_BOUNDARY", "ModeNode", "TnTensor", "Tensor",
    "chain_dot", "dot", "entries", "full", "getitem", "node_tt_core", "norm", "promote_cp_node",
    "ContractViolationError", "StructuralError", "TntzError", "NativeError", "DataError", "MagicError",
    "ChecksumError", "SizeError", "load", "save", "read_header", "read_dense", "write_dense",
]
