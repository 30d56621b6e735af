"""Device time of the paths the fast kernels do not cover (VERDICT r1
'missing' 3-5): batched-chain entries, rank > 32 entries, dot / norm at
ranks != 16, and the float64 instantiation; with each one's plan / kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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


def tt(shape, r, batch=None, scale=None, dtype=torch.float32, seed=0):
    cores = W.tt_cores(shape, r, seed, batch_size=batch, scale=scale)
    return tb.TnTensor([tb.ModeNode("tt", c, batched=batch is not None, dtype=dtype) for c in cores], batch)


def line(name, ms, units, unit):
    print(f"{name:60s} {ms:9.3f} ms  {units / ms / 1e3:12.4g} {unit}/s", flush=True)


m = 1 << 20
idx = torch.randint(0, 32, (m, 10), device="cuda")
for B in (1, 4, 16):
    t = tt((32,) * 10, 32, batch=None if B == 1 else B)
    line(f"entries cfg2-shape B={B} m=2^20 (algo auto)", ev(lambda: tb.entries(t, idx)), m * B, "entries")
t = tt((32,) * 10, 32, batch=4)
for algo, nm in ((N.ALGO_CHAIN, "chain"), (N.ALGO_LAYERED, "layered")):
    line(f"entries cfg2-shape B=4 algo={nm}", ev(lambda: tb.entries(t, idx, algo=algo)), m * 4, "entries")
t64 = tt((256,) * 4, 64)
i64 = torch.randint(0, 256, (m, 4), device="cuda")
for algo, nm in ((N.ALGO_AUTO, "auto"), (N.ALGO_LAYERED, "layered")):
    line(f"entries cfg3 chain r=64 m=2^20 algo={nm}", ev(lambda: tb.entries(t64, i64, algo=algo)), m, "entries")
for r in (8, 16, 24, 32):
    a, b = tt((64,) * 16, r, batch=1024, scale=0.25), tt((64,) * 16, r, batch=1024, scale=0.25, seed=1)
    line(f"dot cfg4-shape r={r} 1024 pairs", ev(lambda: tb.dot(a, b)), 1024, "pairs")
    line(f"norm cfg4-shape r={r} 1024 pairs", ev(lambda: tb.norm(a)), 1024, "pairs")
    os.environ["TNB_DOT_MMA"] = "0"
    line(f"dot cfg4-shape r={r} 1024 pairs (chunked SIMT)", ev(lambda: tb.dot(a, b)), 1024, "pairs")
    os.environ.pop("TNB_DOT_MMA")
t = tt((32,) * 10, 32, dtype=torch.float64)
line("f64 entries cfg2 m=2^20", ev(lambda: tb.entries(t, idx)), m, "entries")
t = tt((16,) * 6, 8, dtype=torch.float64)
line("f64 full cfg1 (16^6)", ev(lambda: tb.full(t)), 16 ** 6 * 8 / 1e9, "GB")
t = tt((256,) * 4, 64, dtype=torch.float64)
line("f64 full cfg3 slab 16 (1/16 of 256^4)", ev(lambda: tb.full(t, lead=(0, 16))), 16 * 256 ** 3 * 8 / 1e9, "GB")
a = tt((64,) * 16, 16, batch=1024, scale=0.25, dtype=torch.float64)
b = tt((64,) * 16, 16, batch=1024, scale=0.25, dtype=torch.float64, seed=1)
line("f64 dot cfg4 1024 pairs", ev(lambda: tb.dot(a, b)), 1024, "pairs")
