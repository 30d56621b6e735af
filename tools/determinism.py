"""Checks that K1 results are bitwise reproducible (run twice) and compares
the pipelined host path with the device path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_11128_b200 as tb  # noqa: E402
from oracle import tntz_oracle as O  # noqa: E402
from paper_2206_11128_b200 import core as C  # noqa: E402

for shape, r in (((32,) * 6, 16), ((32,) * 10, 32), ((16,) * 6, 8)):
    cores = O.random_tt(shape, r, seed=11, scale=r ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    m = 2 * C._PIPELINE_ROWS + 12345
    idx = torch.from_numpy(O.uniform_indices(shape, m, 3))
    d = idx.cuda()
    a = tb.entries(t, d)
    b = tb.entries(t, d)
    c = tb.entries(t, idx.pin_memory())
    e = tb.entries(t, d[: C._PIPELINE_ROWS])
    print(shape, r, "rerun equal:", torch.equal(a, b), "pipelined equal:", torch.equal(a, c),
          "chunk equal:", torch.equal(a[: C._PIPELINE_ROWS], e),
          "max|a-c|:", float((a - c).abs().max()), "n diff:", int((a != c).sum()),
          "first diff at:", int(torch.nonzero(a != c)[0]) if (a != c).any() else -1)
