"""Where the end-to-end entries time goes: raw pinned H2D / D2H bandwidth,
the host index codec's throughput per thread count, and the public call from
pinned host indices with and without the codec (TNB_E2E_CODEC)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_11128_b200 import _native as N  # noqa: E402


def wall(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg2":
    m, shape = 1 << 24, W.CONFIGS["cfg2"][1]
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
else:
    m, shape = 1 << 26, W.CONFIGS["cfg5"][1]
    t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in W.hybrid_nodes(0)])
print("host threads:", N.load().tnb_host_threads(), "os.cpu_count:", os.cpu_count(),
      "affinity:", len(os.sched_getaffinity(0)))
idx_host = torch.from_numpy(W.indices(shape, m, 2)).pin_memory()
gb = idx_host.numel() * 8 / 1e9
dev = torch.empty_like(idx_host, device="cuda")
out = torch.empty(m, device="cuda")
pin_out = torch.empty(m).pin_memory()
nar = torch.empty(idx_host.numel(), dtype=torch.int8).pin_memory()
dnar = torch.empty(idx_host.numel(), dtype=torch.int8, device="cuda")
print("h2d %.2f GB pinned int64: %.2f ms" % (gb, wall(lambda: dev.copy_(idx_host, non_blocking=True))))
print("h2d %.2f GB pinned int8:  %.2f ms" % (gb / 8, wall(lambda: dnar.copy_(nar, non_blocking=True))))
print("d2h out pinned: %.2f ms" % wall(lambda: pin_out.copy_(out, non_blocking=True)))
flat = idx_host.view(-1)
for nt in (1, 2, 4, 8, 16, 32, 0):
    ms = wall(lambda: N.narrow_indices(flat, nar, 1, nt))
    print("narrow int64->int8 nthreads=%d: %.2f ms (%.1f GB/s read)" % (nt, ms, gb / ms * 1e3))
print("widen kernel: %.3f ms" % wall(lambda: N.load().tnb_widen_indices(dnar.data_ptr(), 1, dnar.numel(),
                                                                        dev.data_ptr(), N.stream_ptr(dev.device))))
print("entries(device idx): %.2f ms" % wall(lambda: tb.entries(t, dev)))
from paper_2206_11128_b200 import core as C  # noqa: E402

for codec, frac in (("0", "1"), ("1", "0"), ("1", "0.3"), ("1", "0.4"), ("1", "0.5")):
    os.environ["TNB_E2E_CODEC"] = codec
    os.environ["TNB_E2E_RAW_FRAC"] = frac
    print("codec=%s raw_frac=%s entries(pinned host idx, out=pinned): %.2f ms %s" % (
        codec, frac, wall(lambda: tb.entries(t, idx_host, out=pin_out)), C.last_transfer), flush=True)
os.environ["TNB_E2E_CODEC"] = "1"
os.environ.pop("TNB_E2E_RAW_FRAC", None)
for rep in range(3):
    print("codec=1 dynamic entries(pinned host idx, out=pinned): %.2f ms %s" % (
        wall(lambda: tb.entries(t, idx_host, out=pin_out)), C.last_transfer), flush=True)
got = pin_out.clone()
os.environ["TNB_E2E_RAW_FRAC"] = "0.35"
tb.entries(t, idx_host, out=pin_out)
torch.cuda.synchronize()
assert torch.equal(pin_out, got), "the self-balancing pipeline differs from the static one"
print("dynamic == static pipeline (bitwise)")
