"""cfg2 chain, AUTO: step time against the number of tuples (the per-rank sizes of
strong scaling: 2^24 / N)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_11128_b200 import _native as N  # noqa: E402
from paper_2206_11128_b200 import core as C  # noqa: E402

t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores((32,) * 10, 32, 0)])
p = t._packed()
for lg in range(18, 25):
    m = 1 << lg
    idx = torch.randint(0, 32, (m, 10), dtype=torch.int64, device="cuda")
    out = torch.empty(m, device="cuda")
    err = torch.empty(1, dtype=torch.int32, device="cuda")
    ws = None
    for _ in range(3):
        ws = C.launch_entries(p, idx, out, err, 0, ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        ws = C.launch_entries(p, idx, out, err, 0, ws)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    pl = N.entries_plan(p.chain, m, 0)
    print(f"m=2^{lg} {ms:8.3f} ms  {m / ms / 1e6:7.2f} G entries/s  kernel {pl['compute_kernel']} n_virtual {pl['n_virtual']} "
          f"prefix_rows {pl['prefix_rows']}", flush=True)
    del idx, out, ws
