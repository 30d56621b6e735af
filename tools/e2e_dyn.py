"""Times entries() on pinned host indices (cfg2) under the current TNB_E2E_* environment."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_11128_b200 import core as C  # noqa: E402

m, shape = 1 << 24, W.CONFIGS["cfg2"][1]
t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
idx_host = torch.from_numpy(W.indices(shape, m, 2)).pin_memory()
pin_out = torch.empty(m).pin_memory()
for _ in range(2):
    tb.entries(t, idx_host, out=pin_out)
torch.cuda.synchronize()
ts = []
for _ in range(7):
    t0 = time.perf_counter()
    tb.entries(t, idx_host, out=pin_out)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("ms: min %.2f med %.2f  %s" % (min(ts), sorted(ts)[3], C.last_transfer), flush=True)
