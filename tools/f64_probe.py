"""float64 instantiation timings (cfg shapes, subsets): entries chain vs
layered, full, dot / norm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_11128_b200 import _native as N  # noqa: E402


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


f64 = torch.float64
m = 1 << 20
t2 = tb.TnTensor([tb.ModeNode("tt", c, dtype=f64) for c in W.tt_cores((32,) * 10, 32, 0)])
i2 = torch.randint(0, 32, (m, 10), device="cuda")
for algo, nm in ((N.ALGO_CHAIN, "chain"), (N.ALGO_LAYERED, "layered")):
    print(f"f64 entries cfg2 2^20 {nm}: {ev(lambda: tb.entries(t2, i2, algo=algo)):.3f} ms", flush=True)
t5 = tb.TnTensor([tb.ModeNode(k, c, f, dtype=f64) for k, c, f in W.hybrid_nodes(0)])
i5 = torch.randint(0, 128, (m, 8), device="cuda")
for algo, nm in ((N.ALGO_CHAIN, "chain"), (N.ALGO_LAYERED, "layered")):
    print(f"f64 entries cfg5 2^20 {nm}: {ev(lambda: tb.entries(t5, i5, algo=algo)):.3f} ms", flush=True)
t3 = tb.TnTensor([tb.ModeNode("tt", c, dtype=f64) for c in W.tt_cores((256,) * 4, 64, 0)])
print(f"f64 full cfg3 slab 16: {ev(lambda: tb.full(t3, lead=(0, 16))):.3f} ms", flush=True)
print(f"f32 full cfg3 slab 16: {ev(lambda: tb.full(t3.float(), lead=(0, 16))):.3f} ms", flush=True)
