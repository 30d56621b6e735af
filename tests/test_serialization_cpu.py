"""TNTZ1 containers and raw dense files on the host (no GPU): the golden
containers were written by the reference's own save()
(tests/golden/make_containers.py); cf. pkg/tests/test_serialization.py."""

import json
import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

import paper_2206_11128_b200 as tb
from paper_2206_11128_b200 import serialization as S

GOLD = Path(__file__).resolve().parent / "golden" / "containers"
NAMES = ["tt", "cp", "tucker", "blended", "tt_batched", "cp_batched", "hybrid"]


@pytest.fixture(scope="module")
def expected():
    return np.load(GOLD / "expected.npz")


@pytest.mark.parametrize("name", NAMES)
def test_payload_bit_exact(name, expected):
    header, nodes = S.read_container(GOLD / f"{name}.tntz")
    assert header["kind"] == "tensor" and header["num_modes"] == len(nodes)
    for k, (kind, core, factor) in enumerate(nodes):
        assert np.array_equal(core, expected[f"{name}/core{k}"])
        if factor is not None:
            assert np.array_equal(factor, expected[f"{name}/factor{k}"])
        else:
            assert f"{name}/factor{k}" not in expected


@pytest.mark.parametrize("name", NAMES)
def test_save_reproduces_reference_bytes(name, tmp_path):
    # our save() of the same values writes the reference's file byte for byte
    header, nodes = S.read_container(GOLD / f"{name}.tntz")
    batched = header["batch_size"] is not None
    t = tb.TnTensor([tb.ModeNode(k, c, f, batched=batched) for k, c, f in nodes], header["batch_size"])
    out = tmp_path / "x.tntz"
    tb.save(t, out)
    assert out.read_bytes() == (GOLD / f"{name}.tntz").read_bytes()


def test_header_fields():
    # test_serialization.py:112-118 style
    h = tb.read_header(GOLD / "tt.tntz")
    assert h["kind"] == "tensor" and h["num_modes"] == 3
    assert h["rank_chain"] == [1, 2, 3, 1] and h["physical_shape"] == [3, 4, 5]
    assert tb.read_header(GOLD / "tt_batched.tntz")["batch_size"] == 6


def test_container_errors(tmp_path):
    src = (GOLD / "tt.tntz").read_bytes()
    p = tmp_path / "e.tntz"
    p.write_bytes(b"NOPE!" + src[5:])
    with pytest.raises(tb.MagicError):
        S.read_container(p)
    p.write_bytes(src[:-16])
    with pytest.raises(tb.SizeError):
        S.read_container(p)
    p.write_bytes(src[:-8] + b"\x00" * 8)
    with pytest.raises(tb.ChecksumError):
        S.read_container(p)
    p.write_bytes(src[:7])
    with pytest.raises(tb.SizeError, match="truncated header length"):
        tb.read_header(p)
    for cls in (tb.MagicError, tb.ChecksumError, tb.SizeError):
        assert issubclass(cls, tb.DataError) and issubclass(cls, ValueError) and issubclass(cls, tb.TntzError)


def test_matrix_containers_are_out_of_scope(tmp_path):
    payload = np.zeros(24, "<f8").tobytes()
    header = {"kind": "tt_matrix", "num_modes": 1, "batch_size": None, "row_dims": [2], "col_dims": [3],
              "rank_chain": [1, 1], "core_shapes": [[1, 2, 3, 4]], "checksum": zlib.crc32(payload)}
    blob = json.dumps(header, separators=(",", ":")).encode()
    p = tmp_path / "m.tntz"
    p.write_bytes(b"TNTZ1" + struct.pack("<I", len(blob)) + blob + payload)
    with pytest.raises(tb.ContractViolationError, match="not a tensor network"):
        S.read_container(p)


def test_dense_files(tmp_path, expected):
    x = tb.read_dense(GOLD / "tucker_full.raw", (5, 4, 6))
    assert np.array_equal(x, expected["tucker/full"])
    with pytest.raises(tb.SizeError):
        tb.read_dense(GOLD / "tucker_full.raw", (5, 4, 5))
    with pytest.raises(tb.ContractViolationError):
        tb.read_dense(GOLD / "tucker_full.raw", (0, 4))
    p = tmp_path / "y.raw"
    tb.write_dense(x, p)
    assert p.read_bytes() == (GOLD / "tucker_full.raw").read_bytes()


def test_sampler_rejects_batched():
    _, nodes = S.read_container(GOLD / "tt_batched.tntz")
    t = tb.TnTensor([tb.ModeNode(k, c, f, batched=True) for k, c, f in nodes], 6)
    with pytest.raises(tb.ContractViolationError, match="batched"):
        tb.callers.sampler(t)
