"""Multi-process (world_size 2, gloo, CPU) checks of the sharding plan and the
result gather used by the multi-GPU path; the per-shard compute is the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tntz_oracle as O
from paper_2206_11128_b200 import shard as S


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 64, 1001, 4096):
        for w in (1, 2, 3, 8):
            spans = [S.shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        chain = O.make_chain([("tt", c) for c in O.random_tt((5, 4, 6), 3, seed=3)])
        idx = torch.from_numpy(O.uniform_indices((5, 4, 6), 1001, 4))
        got = S.entries_sharded(chain, idx, compute=lambda c, i: torch.from_numpy(O.entries(c, i.numpy())))
        res["entries"] = float(np.abs(got.numpy() - O.entries(chain, idx.numpy())).max())
        a = O.make_chain([("tt", c) for c in O.random_tt((3, 4, 5), 2, seed=5, batch_size=5)], 5)
        b = O.make_chain([("tt", c) for c in O.random_tt((3, 4, 5), 3, seed=6, batch_size=5)], 5)
        dots = S.dot_sharded(a, b, compute=lambda x, y: torch.from_numpy(O.chain_dot(x, y)),
                             slicer=O.batch_slice)
        res["dot"] = float(np.abs(dots.numpy() - O.chain_dot(a, b)).max())
        norms = S.norm_sharded(a, compute=lambda x: torch.from_numpy(O.norm(x)), slicer=O.batch_slice)
        res["norm"] = float(np.abs(norms.numpy() - O.norm(a)).max())
        # batch < world: rank 1's pair shard is empty and must still join the gather
        a1 = O.batch_slice(a, 0, 1)
        b1 = O.batch_slice(b, 0, 1)
        d1 = S.dot_sharded(a1, b1, compute=lambda x, y: torch.from_numpy(O.chain_dot(x, y)),
                           slicer=O.batch_slice)
        n1 = S.norm_sharded(a1, compute=lambda x: torch.from_numpy(O.norm(x)), slicer=O.batch_slice)
        res["dot_small"] = float(np.abs(d1.numpy() - O.chain_dot(a1, b1)).max()) if d1.shape == (1,) else 1.0
        res["norm_small"] = float(np.abs(n1.numpy() - O.norm(a1)).max()) if n1.shape == (1,) else 1.0
        slab, (lo, hi) = S.full_sharded(chain, compute=lambda c, l, h: torch.from_numpy(O.full_slab(c, l, h)))
        res["full"] = float(np.abs(slab.numpy() - O.full(chain)[lo:hi]).max())
        res["span"] = (lo, hi)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        for k in ("entries", "dot", "norm", "full", "dot_small", "norm_small"):
            assert out[r][k] <= 1e-12, (r, k, out[r][k])
    assert out[0]["span"] == (0, 3) and out[1]["span"] == (3, 5)


def test_sharded_dot_rejects_unbatched():
    from paper_2206_11128_b200.errors import ContractViolationError

    chain = O.make_chain([("tt", c) for c in O.random_tt((5, 4), 3, seed=3)])
    with pytest.raises(ContractViolationError, match="not batched"):
        S.dot_sharded(chain, chain, compute=lambda x, y: None, slicer=O.batch_slice)
    with pytest.raises(ContractViolationError, match="not batched"):
        S.norm_sharded(chain, compute=lambda x: None, slicer=O.batch_slice)
