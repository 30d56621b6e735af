"""AUTO with and without the global-sort path over a spread of TT shapes: step
time and agreement (both against each other; the parity tests hold the oracle)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [  # (J, r, modes, log2 m)
    (32, 32, 10, 22), (32, 32, 8, 20), (16, 16, 12, 22), (64, 32, 6, 22), (32, 24, 10, 23), (128, 16, 5, 22),
    (8, 8, 20, 22), (32, 16, 10, 24), (256, 32, 4, 22), (48, 20, 7, 22), (32, 32, 10, 19), (10, 12, 9, 21),
    (48, 32, 7, 22), (48, 24, 7, 23), (40, 8, 9, 22), (20, 28, 8, 21),
]


def one(J, r, n, lg):
    import torch

    import paper_2206_11128_b200 as tb
    from oracle import tntz_oracle as O
    from paper_2206_11128_b200 import _native as N
    from paper_2206_11128_b200 import core as C

    cores = O.random_tt((J,) * n, r, seed=3, scale=r ** -0.5)
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    p = t._packed()
    m = 1 << lg
    torch.manual_seed(5)
    idx = torch.randint(0, J, (m, n), dtype=torch.int64, device="cuda")
    out = torch.empty(m, device="cuda")
    err = torch.empty(1, dtype=torch.int32, device="cuda")
    ws = None
    for _ in range(2):
        ws = C.launch_entries(p, idx, out, err, 0, ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        ws = C.launch_entries(p, idx, out, err, 0, ws)
    b.record()
    torch.cuda.synchronize()
    pl = N.entries_plan(p.chain, m, 0)
    torch.save(out.cpu(), f"/tmp/auto_sweep_{os.environ.get('TNB_ENTRIES_GSORT', '1')}.pt")
    print(f"{a.elapsed_time(b) / 5:.3f} {pl['compute_kernel']} {pl['n_virtual']} {pl['prefix_rows']} {pl['suffix_rows']}")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(*map(int, sys.argv[1:5]))
        sys.exit(0)
    import torch

    for J, r, n, lg in SHAPES:
        res = {}
        for g in ("1", "0"):
            q = subprocess.run([sys.executable, __file__, str(J), str(r), str(n), str(lg)],
                               env=dict(os.environ, TNB_ENTRIES_GSORT=g), capture_output=True, text=True)
            res[g] = q.stdout.split() if q.returncode == 0 else ["fail", q.stderr[-200:]]
        x, y = torch.load("/tmp/auto_sweep_1.pt"), torch.load("/tmp/auto_sweep_0.pt")
        rel = float((x - y).norm() / y.norm())
        print(f"J={J:4d} r={r:3d} N={n:3d} m=2^{lg}: auto {res['1'][0]} ms (kernel {res['1'][1]}, {res['1'][2]} virtual modes) | "
              f"bucketed {res['0'][0]} ms (kernel {res['0'][1]}, {res['0'][2]} modes) | rel diff {rel:.2e}", flush=True)
