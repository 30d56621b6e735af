"""Small invocations of every fast kernel for compute-sanitizer (one tool
per gpurun call: memcheck, racecheck, synccheck; profiles/r02_sanitizer_*):
bucketed state kernel (r=32 tensor-core sorted modes, HBM prefix/suffix
tables), bucketed stream kernel (R=24, swizzled ring), the tcgen05 full()
GEMM with the TMA-store epilogue (ragged tiles), the rank-16 dot/norm
kernel, and the index codec's widen kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
from paper_2206_11128_b200 import _native as N  # noqa: E402

rng = np.random.default_rng(0)


def tt(shape, r, batch=None, scale=None):
    ranks = [1] + [r] * (len(shape) - 1) + [1]
    s = scale or r ** -0.5
    cores = [(rng.standard_normal(((batch,) if batch else ()) + (ranks[k], n, ranks[k + 1])) * s).astype(np.float32)
             for k, n in enumerate(shape)]
    return tb.TnTensor([tb.ModeNode("tt", c, batched=batch is not None) for c in cores], batch)


which = sys.argv[1:] or ["state", "stream", "full", "dot", "widen"]
if "state" in which:  # state kernel, r = 32, tensor-core sorted modes
    t = tt((32,) * 6, 32)
    m = 1 << 16
    print("state plan", N.entries_plan(t._packed().chain, m))
    idx = torch.randint(0, 32, (m, 6), device="cuda")
    tb.entries(t, idx)
if "stream" in which:  # stream kernel, R = 24
    t = tt((2048, 40, 2048), 24)
    m = 1 << 17
    print("stream plan", N.entries_plan(t._packed().chain, m))
    idx = torch.stack([torch.randint(0, s, (m,), device="cuda") for s in t.shape], 1)
    tb.entries(t, idx)
if "full" in which:  # tcgen05 GEMM + TMA epilogue with ragged row / column tiles
    t = tt((40, 37, 53, 29), 16)
    tb.full(t)
    t = tt((128, 96, 128), 16)
    tb.full(t)
if "dot" in which:
    a, b = tt((16,) * 5, 16, batch=8, scale=0.25), tt((16,) * 5, 16, batch=8, scale=0.25)
    tb.dot(a, b)
    tb.norm(a)
if "widen" in which:
    x = torch.randint(-100, 100, (1000003,), dtype=torch.int8, device="cuda")
    y = torch.empty(x.numel(), dtype=torch.int64, device="cuda")
    N.check(N.load().tnb_widen_indices(x.data_ptr(), 1, x.numel(), y.data_ptr(), N.stream_ptr(x.device)), "widen")
    assert torch.equal(y, x.long())
torch.cuda.synchronize()
print("sanitize cases done", which)
