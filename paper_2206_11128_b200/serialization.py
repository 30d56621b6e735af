"""TNTZ1 containers and raw dense files, loaded straight onto the device.

Format (reference: serialization.py:1-8, 83-133 of
/root/reference/pkg/src/tntz): 5 magic bytes ``TNTZ1``, a little-endian u32
header length, a UTF-8 JSON header (object structure + CRC32 of the payload),
then the payload: the raw little-endian float64 arrays, row-major, in node
order, core before factor.

The loader validates like the reference (magic -> MagicError, truncated
header / wrong payload length -> SizeError, CRC mismatch -> ChecksumError),
then moves the WHOLE checked payload to the device in one pinned copy and
casts/splits it there; the cores land in the repacked layout on their first
contraction (``TnTensor._packed``).  Values become fp32 on the device, the
package's intended deviation; ``read_container`` gives the bit-exact float64
arrays on the host.  Only the ``tensor`` kind is a hot-path object; the
compressed-matrix kinds are outside this package's scope.
"""

from __future__ import annotations

import json
import struct
import zlib
from pathlib import Path
from typing import List, Optional, Tuple

import numpy as np
import torch

from .core import TnTensor, ModeNode, _default_device
from .errors import ChecksumError, ContractViolationError, MagicError, SizeError

MAGIC = b"TNTZ1"
KIND_TENSOR = "tensor"


def read_header(path) -> dict:
    """Parse and validate the container header (serialization.py:97-113)."""
    with open(path, "rb") as fh:
        magic = fh.read(len(MAGIC))
        if magic != MAGIC:
            raise MagicError(f"{path}: bad magic {magic!r}")
        raw_len = fh.read(4)
        if len(raw_len) != 4:
            raise SizeError(f"{path}: truncated header length")
        (blob_len,) = struct.unpack("<I", raw_len)
        blob = fh.read(blob_len)
        if len(blob) != blob_len:
            raise SizeError(f"{path}: truncated header")
    try:
        return json.loads(blob.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise SizeError(f"{path}: malformed header: {exc}") from exc


def _declared_floats(header: dict) -> int:
    """Payload length the header declares (serialization.py:136-149)."""
    kind = header.get("kind")
    if kind == KIND_TENSOR:
        total = 0
        for node in header["nodes"]:
            total += int(np.prod(node["core_shape"]))
            if node["factor_shape"] is not None:
                total += int(np.prod(node["factor_shape"]))
        return total
    if kind == "tt_matrix":
        return sum(int(np.prod(s)) for s in header["core_shapes"])
    if kind == "cp_matrix":
        return sum(int(np.prod(s)) for s in header["factor_shapes"])
    raise SizeError(f"unknown object kind {kind!r}")


def _checked_payload(path) -> Tuple[dict, bytes]:
    header = read_header(path)
    with open(path, "rb") as fh:
        fh.read(len(MAGIC))
        (blob_len,) = struct.unpack("<I", fh.read(4))
        fh.read(blob_len)
        payload = fh.read()
    expected = _declared_floats(header)
    if len(payload) != 8 * expected:
        raise SizeError(f"{path}: payload holds {len(payload)} bytes, header declares {8 * expected}")
    if (zlib.crc32(payload) & 0xFFFFFFFF) != header.get("checksum"):
        raise ChecksumError(f"{path}: payload checksum mismatch")
    return header, payload


def _layout(header: dict) -> List[Tuple[str, tuple, Optional[tuple]]]:
    if header.get("kind") != KIND_TENSOR:
        raise ContractViolationError(
            f"a {header.get('kind')!r} container is not a tensor network; compressed matrices are "
            "outside the GPU hot path")
    return [(e["kind"], tuple(e["core_shape"]),
             None if e["factor_shape"] is None else tuple(e["factor_shape"])) for e in header["nodes"]]


def read_container(path) -> Tuple[dict, List[Tuple[str, np.ndarray, Optional[np.ndarray]]]]:
    """Host view: (header, [(kind, core, factor)]) with the bit-exact float64
    arrays of the payload (serialization.py:116-133, 152-173)."""
    header, payload = _checked_payload(path)
    floats = np.frombuffer(payload, dtype="<f8")
    out, off = [], 0
    for kind, cs, fs in _layout(header):
        n = int(np.prod(cs))
        core = floats[off:off + n].reshape(cs).astype(np.float64)
        off += n
        factor = None
        if fs is not None:
            n = int(np.prod(fs))
            factor = floats[off:off + n].reshape(fs).astype(np.float64)
            off += n
        out.append((kind, core, factor))
    return header, out


def load(path, device=None, dtype=torch.float32) -> TnTensor:
    """Container -> TnTensor on ``device`` (default: the current CUDA
    device): one pinned H2D copy of the checked payload, then per-node views
    on the device -- cast to fp32 (the hot path) or, with
    ``dtype=torch.float64``, the payload floats bit for bit."""
    header, payload = _checked_payload(path)
    layout = _layout(header)
    dev = torch.device(device) if device is not None else _default_device()
    host = torch.frombuffer(bytearray(payload), dtype=torch.float64)
    if dev.type == "cuda":
        host = host.pin_memory()
    flat = host.to(dev, non_blocking=True).to(dtype)
    batch = header.get("batch_size")
    nodes, off = [], 0
    for kind, cs, fs in layout:
        n = int(np.prod(cs))
        core = flat[off:off + n].view(cs)
        off += n
        factor = None
        if fs is not None:
            n = int(np.prod(fs))
            factor = flat[off:off + n].view(fs)
            off += n
        nodes.append(ModeNode(kind, core, factor, batched=batch is not None, dtype=dtype))
    return TnTensor(nodes, batch)


def _f64_bytes(a: torch.Tensor) -> bytes:
    return np.ascontiguousarray(a.detach().cpu().numpy(), dtype="<f8").tobytes()


def save(t: TnTensor, path) -> None:
    """TnTensor -> container, byte-compatible with the reference's save()
    (serialization.py:34-94): the same header fields and key order, compact
    JSON, CRC32 of the float64 payload (fp32 values widen exactly)."""
    if not isinstance(t, TnTensor):
        raise ContractViolationError(f"cannot serialize a {type(t).__name__}")
    nodes, arrays = [], []
    for node in t.nodes:
        nodes.append({"kind": node.kind, "core_shape": list(node.core.shape),
                      "factor_shape": None if node.factor is None else list(node.factor.shape)})
        arrays.append(node.core)
        if node.factor is not None:
            arrays.append(node.factor)
    header = {"kind": KIND_TENSOR, "num_modes": t.ndim, "batch_size": t.batch_size,
              "physical_shape": list(t.shape), "rank_chain": list(t.ranks), "nodes": nodes}
    payload = b"".join(_f64_bytes(a) for a in arrays)
    header["checksum"] = zlib.crc32(payload) & 0xFFFFFFFF
    blob = json.dumps(header, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<I", len(blob)))
        fh.write(blob)
        fh.write(payload)


def write_dense(x, path) -> None:
    """Raw little-endian float64 dump, row-major (serialization.py:176-178);
    a device tensor (e.g. a full() result) is widened on the way out."""
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    np.ascontiguousarray(x, dtype="<f8").tofile(path)


def read_dense(path, shape, device=None):
    """Raw dense file -> float64 ndarray (serialization.py:181-192), or an
    fp32 tensor on ``device`` when one is given."""
    shape = tuple(int(s) for s in shape)
    if any(s < 1 for s in shape):
        raise ContractViolationError("dense shapes must be positive")
    expected = 8 * int(np.prod(shape))
    actual = Path(path).stat().st_size
    if actual != expected:
        raise SizeError(f"{path}: file holds {actual} bytes but shape {shape} needs {expected}")
    x = np.fromfile(path, dtype="<f8").reshape(shape).astype(np.float64)
    if device is None:
        return x
    return torch.from_numpy(x).to(device).to(torch.float32)
