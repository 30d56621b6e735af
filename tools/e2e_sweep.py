"""e2e entries from pinned host memory (cfg2): sweep of the pipeline knobs
(raw-chunk fraction, narrowing threads, chunk size); wall time per call."""
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
import workloads as W  # noqa: E402

m, shape = 1 << 24, W.CONFIGS["cfg2"][1]
t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
ih = torch.from_numpy(W.indices(shape, m, 2)).pin_memory()
po = torch.empty(m).pin_memory()
FRACS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0.25", "0.35", "0.45"]
THREADS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["12", "15", "16"]
CHUNKS = sys.argv[3].split(",") if len(sys.argv) > 3 else ["20", "21"]
for frac, thr, ch in itertools.product(FRACS, THREADS, CHUNKS):
    os.environ.update(TNB_E2E_RAW_FRAC=frac, TNB_E2E_THREADS=thr, TNB_E2E_CHUNK_LOG2=ch)
    tb.entries(t, ih, out=po)
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        tb.entries(t, ih, out=po)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"raw_frac={frac} threads={thr} chunk=2^{ch}: {min(ts):.2f} ms (median {sorted(ts)[2]:.2f})", flush=True)
