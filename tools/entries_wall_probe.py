"""Host vs device time of one entries() call on cfg2 through each layer:
the façade with a device index matrix, launch_entries with a fresh / reused
workspace, and the pipelined host path (CUDA events + wall clock)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_11128_b200 import _native as N  # noqa: E402
from paper_2206_11128_b200 import core as C  # noqa: E402

m, shape = 1 << 24, W.CONFIGS["cfg2"][1]
t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
p = t._packed()
idx_host = torch.from_numpy(W.indices(shape, m, 2)).pin_memory()
idx = idx_host.cuda()
out = torch.empty(m, device="cuda")
err = torch.empty(1, dtype=torch.int32, device="cuda")
pin_out = torch.empty(m).pin_memory()


def both(name, fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h = 0.0
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        a = time.perf_counter()
        fn()
        h += time.perf_counter() - a
    e1.record()
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) / n * 1e3
    print(f"{name}: device {e0.elapsed_time(e1) / n:.3f} ms  wall {w:.3f} ms  host-in-call {h / n * 1e3:.3f} ms",
          flush=True)


ws = [None]


def reuse():
    ws[0] = C.launch_entries(p, idx, out, err, 0, ws[0])


both("launch_entries reused ws", reuse)
both("launch_entries fresh ws", lambda: C.launch_entries(p, idx, out, err, 0))
both("tb.entries(device idx)", lambda: tb.entries(t, idx))
both("tb.entries(device idx, out=dev)", lambda: tb.entries(t, idx, out=out))
sub = idx[: 1 << 21].contiguous()
both("launch_entries 2^21 rows", lambda: C.launch_entries(p, sub, out[: 1 << 21], err, 0))
print(N.entries_plan(p.chain, 1 << 21))
for codec in ("0", "1"):
    os.environ["TNB_E2E_CODEC"] = codec
    both(f"pipelined host codec={codec}", lambda: tb.entries(t, idx_host, out=pin_out), n=3)
    print(C.last_transfer)
