"""TNTZ1 containers loaded onto the device and contracted there, against the
reference's own float64 outputs for those containers
(tests/golden/make_containers.py); GPU-backed callers of entries."""

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2206_11128_b200 as tb
from tests.helpers import assert_close, to_np

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "containers"
NAMES = ["tt", "cp", "tucker", "blended", "tt_batched", "cp_batched", "hybrid"]


@pytest.fixture(scope="module")
def expected():
    return np.load(GOLD / "expected.npz")


@pytest.mark.parametrize("name", NAMES)
def test_loaded_container_matches_reference(name, expected):
    t = tb.load(GOLD / f"{name}.tntz")
    assert t.device.type == "cuda"
    if f"{name}/full" in expected:
        assert_close(tb.full(t), expected[f"{name}/full"], what=f"{name} full")
    assert_close(tb.entries(t, expected[f"{name}/idx"]), expected[f"{name}/entries"], what=f"{name} entries")
    assert_close(tb.norm(t), expected[f"{name}/norm"], what=f"{name} norm")


def test_device_save_round_trip(tmp_path):
    t = tb.load(GOLD / "hybrid.tntz")
    out = tmp_path / "h.tntz"
    tb.save(t, out)
    assert out.read_bytes() == (GOLD / "hybrid.tntz").read_bytes()


def test_dense_file_to_device(expected):
    x = tb.read_dense(GOLD / "tucker_full.raw", (5, 4, 6), device="cuda")
    assert x.device.type == "cuda" and x.dtype == torch.float32
    t = tb.load(GOLD / "tucker.tntz")
    assert_close(tb.full(t), to_np(x), what="full vs dense file")


def test_elementwise_sampler_and_validation(expected):
    t = tb.load(GOLD / "hybrid.tntz")
    idx = expected["hybrid/idx"]
    ref = expected["hybrid/entries"]
    f = tb.callers.sampler(t, torch.sin)
    assert_close(f(idx), np.sin(ref), what="sin(t[idx])")
    ident = tb.callers.sampler(t)
    assert_close(ident(torch.from_numpy(idx).cuda()), ref, what="t[idx]")
    # cross.py:277-282: relative validation error of an approximation
    y = ref * (1 + 1e-3 * np.cos(np.arange(len(ref))))
    want = np.linalg.norm(y - ref) / np.linalg.norm(y)
    got = tb.callers.validation_error(t, idx, y)
    assert abs(got - want) <= 1e-4 * want
    assert tb.callers.validation_error(t, idx, np.zeros_like(ref)) == pytest.approx(np.linalg.norm(ref), rel=1e-5)
    tbat = tb.load(GOLD / "tt_batched.tntz")
    yb = expected["tt_batched/entries"]
    assert tb.callers.validation_error(tbat, expected["tt_batched/idx"], yb) < 1e-5
