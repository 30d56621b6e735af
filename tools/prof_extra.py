"""Small invocations of the round-2 kernels for ncu captures: the two-table
entries kernel (cfg3 chain, r=64, 2^20 tuples), the chunked dot kernel (r=32,
1024 pairs) and the batched state kernel (B=4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
m = 1 << 20
if which in ("all", "two_table"):
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores((256,) * 4, 64, 0)])
    idx = torch.randint(0, 256, (m, 4), device="cuda")
    for _ in range(3):
        tb.entries(t, idx)
if which in ("all", "dot_chunk"):
    a = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in W.tt_cores((64,) * 16, 32, 0, 1024, 0.25)], 1024)
    b = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in W.tt_cores((64,) * 16, 32, 1, 1024, 0.25)], 1024)
    for _ in range(3):
        tb.dot(a, b)
if which in ("all", "batched"):
    t = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in W.tt_cores((32,) * 10, 32, 0, 4)], 4)
    idx = torch.randint(0, 32, (m, 10), device="cuda")
    for _ in range(3):
        tb.entries(t, idx)
torch.cuda.synchronize()
print("ok", which)
