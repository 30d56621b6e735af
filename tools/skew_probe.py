"""Entries throughput on skewed index distributions (cfg2 chain, 2^24
tuples): uniform, every sample on one index, fibers (all modes fixed but
one, as cross approximation samples), few distinct rows, zipf-like."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402


def ev(fn, n=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg2":
    m, shape = 1 << 24, (32,) * 10
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
else:
    m, shape = 1 << 26, (128,) * 8
    t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in W.hybrid_nodes(0)])
n = len(shape)
J = shape[0]
g = torch.Generator(device="cuda")
g.manual_seed(0)
cases = {
    "uniform": torch.randint(0, J, (m, n), device="cuda", generator=g),
    "all_zero": torch.zeros((m, n), dtype=torch.int64, device="cuda"),
    "fibers_last_mode": torch.randint(0, J, (m // J, n), device="cuda", generator=g).repeat_interleave(J, 0),
    "few_rows_64": torch.randint(0, J, (64, n), device="cuda", generator=g)[torch.randint(0, 64, (m,), device="cuda", generator=g)],
    "zipf_like": (torch.rand((m, n), device="cuda", generator=g) ** 4 * J).long().clamp_(0, J - 1),
}
cases["fibers_last_mode"][:, -1] = torch.arange(m, device="cuda") % J
fixed = torch.randint(0, J, (m, n), device="cuda", generator=g)
fixed[:, : n // 2] = torch.randint(0, J, (1, n // 2), device="cuda", generator=g)
cases["slice_query_prefix_fixed"] = fixed
fixed2 = torch.randint(0, J, (m, n), device="cuda", generator=g)
fixed2[:, n // 2:] = torch.randint(0, J, (1, n - n // 2), device="cuda", generator=g)
cases["slice_query_suffix_fixed"] = fixed2
from paper_2206_11128_b200 import _native as N  # noqa: E402

for name, idx in cases.items():
    ms = ev(lambda: tb.entries(t, idx))
    N.timing_enable(True)
    tb.entries(t, idx)
    torch.cuda.synchronize()
    kt = {k: round(N.timing_read(k)[0], 3) for k in ("entries_prep", "entries_sort", "entries_compute", "entries_tables")}
    N.timing_enable(False)
    print(f"{cfg} {name:20s} {ms:8.3f} ms  {m / ms / 1e6:8.3f} G entries/s  {kt}", flush=True)
