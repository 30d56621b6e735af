"""CUDA-event timing of the widen kernel and of entries() right after host
narrowing work (the e2e probe saw both slow when timed by wall clock)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_11128_b200 import _native as N  # noqa: E402


def ev(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


m, shape = 1 << 24, W.CONFIGS["cfg2"][1]
t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
idx_host = torch.from_numpy(W.indices(shape, m, 2)).pin_memory()
dev = idx_host.cuda()
dnar = dev.to(torch.int8)
out64 = torch.empty_like(dev)
st = N.stream_ptr(dev.device)
lib = N.load()
print("entries(dev) before: %.3f ms" % ev(lambda: tb.entries(t, dev)))
print("widen 1.34 GB: %.3f ms" % ev(lambda: lib.tnb_widen_indices(dnar.data_ptr(), 1, dnar.numel(), out64.data_ptr(), st)))
print("torch int8->int64 copy: %.3f ms" % ev(lambda: out64.copy_(dnar)))
print("widen correct:", bool(torch.equal(out64, dev)))
nar = torch.empty(dev.numel(), dtype=torch.int8).pin_memory()
for _ in range(5):
    N.narrow_indices(idx_host.view(-1), nar, 1)
print("entries(dev) after narrowing: %.3f ms" % ev(lambda: tb.entries(t, dev)))
print("entries(widened) : %.3f ms" % ev(lambda: tb.entries(t, out64)))
