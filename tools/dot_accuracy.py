"""cfg4 dot/norm error against the float64 oracle for both K3 variants
(run once per variant: TNB_DOT_SIMT=1 selects the FFMA kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_11128_b200 as tb  # noqa: E402
from oracle import tntz_oracle as O  # noqa: E402
from tests.helpers import facade, to_np  # noqa: E402

a = O.random_tt((64,) * 16, 16, seed=0, batch_size=4096, scale=0.25)
b = O.random_tt((64,) * 16, 16, seed=1, batch_size=4096, scale=0.25)
ta = facade([("tt", c, None) for c in a], 4096)
tb_ = facade([("tt", c, None) for c in b], 4096)
oa, ob = O.make_chain([("tt", c) for c in a], 4096), O.make_chain([("tt", c) for c in b], 4096)
dots, norms = to_np(tb.dot(ta, tb_)), to_np(tb.norm(ta))
for lo, hi in ((0, 256), (3840, 4096)):
    rd = O.chain_dot(O.batch_slice(oa, lo, hi), O.batch_slice(ob, lo, hi))
    rn = O.norm(O.batch_slice(oa, lo, hi))
    print(os.environ.get("TNB_DOT_SIMT", "0"), lo, "dot", O.rel_errors(dots[lo:hi], rd), "norm", O.rel_errors(norms[lo:hi], rn))
