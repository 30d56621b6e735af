#!/usr/bin/env python
"""Pure HBM write bandwidth (torch fill_ / zero_ over 16 GiB): the roof for
the write-bound full() kernel, next to MEASURED_PEAKS.json's copy figure."""
import torch

x = torch.empty(2**32, dtype=torch.float32, device="cuda")
for name, f in [("fill", lambda: x.fill_(1.0)), ("zero", lambda: x.zero_())]:
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(name, round(best, 4), "ms", round(x.numel() * 4 / best / 1e6, 1), "GB/s")
