"""cfg4 dot / norm: device time per launch (CUDA events) and error of pairs
0-255 against the float64 oracle.  TNB_LIB selects a variant build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
from oracle import tntz_oracle as O  # noqa: E402
from tests.helpers import facade, to_np  # noqa: E402

a = O.random_tt((64,) * 16, 16, seed=0, batch_size=4096, scale=0.25)
b = O.random_tt((64,) * 16, 16, seed=1, batch_size=4096, scale=0.25)
ta = facade([("tt", c, None) for c in a], 4096)
tb_ = facade([("tt", c, None) for c in b], 4096)
oa, ob = O.make_chain([("tt", c) for c in a], 4096), O.make_chain([("tt", c) for c in b], 4096)


def timed(fn, n=10):
    for _ in range(3):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(n):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / n


rd = O.chain_dot(O.batch_slice(oa, 0, 256), O.batch_slice(ob, 0, 256))
rn = O.norm(O.batch_slice(oa, 0, 256))
print("dot  %.3f ms  %s" % (timed(lambda: tb.dot(ta, tb_)), O.rel_errors(to_np(tb.dot(ta, tb_))[:256], rd)))
print("norm %.3f ms  %s" % (timed(lambda: tb.norm(ta)), O.rel_errors(to_np(tb.norm(ta))[:256], rn)))
