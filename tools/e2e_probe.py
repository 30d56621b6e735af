"""Where the end-to-end entries time goes: raw pinned H2D / D2H bandwidth,
the public call from pinned host indices, and the result read-back."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402


def wall(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


m = 1 << 24
shape = W.CONFIGS["cfg2"][1]
t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
idx_host = torch.from_numpy(W.indices(shape, m, 2)).pin_memory()
dev = torch.empty_like(idx_host, device="cuda")
out = torch.empty(m, device="cuda")
pin_out = torch.empty(m).pin_memory()
print("h2d 1.34 GB pinned: %.2f ms" % wall(lambda: dev.copy_(idx_host, non_blocking=True)))
print("d2h 64 MB pinned:   %.2f ms" % wall(lambda: pin_out.copy_(out, non_blocking=True)))
print("d2h 64 MB pageable: %.2f ms" % wall(lambda: out.cpu()))
print("entries(device idx): %.2f ms" % wall(lambda: tb.entries(t, dev)))
print("entries(pinned host idx): %.2f ms" % wall(lambda: tb.entries(t, idx_host)))
print("entries(pinned host idx) + .cpu(): %.2f ms" % wall(lambda: tb.entries(t, idx_host).cpu()))
