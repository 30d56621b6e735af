"""the reference's OWN hot-path tests, run unmodified with
tntz's full / entries / chain_dot / norm re-pointed at the GPU's float64
instantiation (paper_2206_11128_b200.tntz_shim), at their native 1e-12 ..
1e-14 tolerances and exact-equality checks.

The reference package and its tests live in the git-ignored baseline/_ref/
(tools/install_reference.sh); gpurun ships that directory to the GPU box.
The tests run in a subprocess so the patch is in place before the reference
test modules import tntz.
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

# the reference tests that exercise the hot path:
# test_core.py:61-195, test_arithmetic.py:116-137, test_indexing.py:168-186,
# test_acceptance.py:87-96
NODES = [
    "test_core.py::TestFull",
    "test_core.py::TestNorm",
    "test_core.py::TestEntries",
    "test_arithmetic.py::TestDot",
    "test_indexing.py::TestArrayForm",
    "test_acceptance.py::test_criterion_02_representation_equivalence",
]


def _run(extra=()):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (REF / "tntz").is_dir() or not (REF / "tests").is_dir():
        pytest.skip("baseline/_ref (the reference package + its tests) is not installed: "
                    "run tools/install_reference.sh")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests"),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "tntz_shim_plugin", "-p", "no:cacheprovider", "-q",
           "-c", os.devnull, "--rootdir", str(REF / "tests"), "-s", *extra, *NODES]
    r = subprocess.run(cmd, cwd=REF / "tests", env=env, capture_output=True, text=True, timeout=1200)
    return r.returncode, r.stdout + r.stderr


def test_reference_hot_path_tests_pass_on_gpu_f64():
    rc, log = _run()
    assert "tntz shim installed" in log and "-> GPU (torch.float64)" in log, log[-3000:]
    assert rc == 0, log[-6000:]
    m = re.search(r"(\d+) passed", log)
    assert m and int(m.group(1)) >= 40, log[-3000:]
    calls = dict(re.findall(r"(full|entries|chain_dot|norm)=(\d+)", log.split("tntz shim calls:")[-1]))
    # every patched operation really ran on the GPU
    for op in ("full", "entries", "chain_dot", "norm"):
        assert int(calls.get(op, 0)) > 0, (op, calls)
