"""SURVEY 8(e) on the CUDA path: two ranks (processes) share cuda:0 and run
the sharded entries / full / dot / norm through libtnb, gathering over gloo.
The ranks' kernels never wait on one another (no device-side collective),
so sharing one GPU is safe; the results must equal the single-process
oracle exactly as the N=1 path does."""

import os
import socket

import numpy as np
import pytest

from oracle import tntz_oracle as O
from tests.helpers import assert_close, assert_dot_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import shard as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        cores = O.random_tt((32,) * 6, 32, seed=3, scale=32 ** -0.5)
        t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
        idx = torch.from_numpy(O.uniform_indices((32,) * 6, 300001, 4)).cuda()
        got = S.entries_sharded(t, idx)  # each rank's 150k rows take the bucketed kernels
        res["entries"] = got.cpu().numpy()
        a = O.random_tt((16,) * 5, 16, seed=5, batch_size=9, scale=0.25)
        b = O.random_tt((16,) * 5, 16, seed=6, batch_size=9, scale=0.25)
        ta = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in a], 9)
        tb_ = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in b], 9)
        res["dot"] = S.dot_sharded(ta, tb_).cpu().numpy()
        res["norm"] = S.norm_sharded(ta).cpu().numpy()
        f = O.random_tt((24, 40, 64), 16, seed=7, scale=0.25)
        tf = tb.TnTensor([tb.ModeNode("tt", c) for c in f])
        slab, span = S.full_sharded(tf)
        res["full"], res["span"] = slab.cpu().numpy(), span
        q.put((rank, res))
    except Exception as e:  # noqa: BLE001
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu():
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        assert "error" not in out[r], out[r]
    cores = O.random_tt((32,) * 6, 32, seed=3, scale=32 ** -0.5)
    o = O.make_chain([("tt", c) for c in cores])
    idx = O.uniform_indices((32,) * 6, 300001, 4)
    sel = np.arange(0, 300001, 7)
    ref = O.entries(o, idx[sel])
    a = O.make_chain([("tt", c) for c in O.random_tt((16,) * 5, 16, seed=5, batch_size=9, scale=0.25)], 9)
    b = O.make_chain([("tt", c) for c in O.random_tt((16,) * 5, 16, seed=6, batch_size=9, scale=0.25)], 9)
    fo = O.make_chain([("tt", c) for c in O.random_tt((24, 40, 64), 16, seed=7, scale=0.25)])
    full = O.full(fo)
    for r in range(2):
        assert out[r]["entries"].shape == (300001,)
        assert_close(out[r]["entries"][sel], ref, what=f"rank {r} entries")
        assert np.array_equal(out[r]["entries"], out[0]["entries"])  # every rank holds the gather
        assert_dot_close(out[r]["dot"], O.chain_dot(a, b), O.norm(a) * O.norm(b), what="dot")
        assert_close(out[r]["norm"], O.norm(a), what="norm")
        lo, hi = out[r]["span"]
        assert_close(out[r]["full"], full[lo:hi], what=f"rank {r} full slab")
    assert out[0]["span"] == (0, 12) and out[1]["span"] == (12, 24)
