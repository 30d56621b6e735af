"""Small full() workload for ncu captures of the tcgen05 GEMM (cfg3 shapes,
a 32-row slab of the leading mode = 2.1 GB of output per launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402

t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores((256,) * 4, 64, 0)])
lo, hi = 0, int(sys.argv[1]) if len(sys.argv) > 1 else 32
for _ in range(3):
    out = tb.full(t, lead=(lo, hi))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    out = tb.full(t, lead=(lo, hi))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"full slab [{lo},{hi}): {ms:.3f} ms, {out.numel() * 4 / ms / 1e6:.1f} GB/s")
