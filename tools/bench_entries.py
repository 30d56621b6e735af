"""Times K1 on cfg2 / cfg5 (device-resident inputs, CUDA events); used to
compare kernel variants selected by environment variables in subprocesses.

    python tools/bench_entries.py            # runs the variant matrix
    python tools/bench_entries.py --one cfg2 # one measurement in-process
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(cfg, algo=0, reps=5):
    import torch

    import paper_2206_11128_b200 as tb
    import workloads as W
    from paper_2206_11128_b200 import core as C

    if cfg == "cfg2":
        t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores((32,) * 10, 32, 0)])
        shape, m = (32,) * 10, 1 << 24
    else:
        t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in W.hybrid_nodes(0)])
        shape, m = (128,) * 8, 1 << 26
    p = t._packed()
    modes = [("diag" if md.layout == 1 else "dense", md.r_left, md.r_right) for md in p.modes]
    idx = torch.randint(0, shape[0], (m, len(shape)), dtype=torch.int64, device="cuda")
    out = torch.empty(m, device="cuda")
    err = torch.empty(1, dtype=torch.int32, device="cuda")
    from paper_2206_11128_b200 import _native as N

    ws = None
    for _ in range(3):
        ws = C.launch_entries(p, idx, out, err, algo, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N.timing_enable(True)
    e0.record()
    for _ in range(reps):
        ws = C.launch_entries(p, idx, out, err, algo, ws)
    e1.record()
    torch.cuda.synchronize()
    kt = {k: N.timing_read(k) for k in ("entries_prep", "entries_sort", "entries_compute", "entries_tables", "entries_mid")}
    N.timing_enable(False)
    ms = e0.elapsed_time(e1) / reps
    flops = W.entry_flops(modes) * m
    plan = N.entries_plan(p.chain, m, algo)
    return {"cfg": cfg, "algo": algo, "ms": round(ms, 3), "Gentries/s": round(m / ms / 1e6, 3),
            "TFLOP/s": round(flops / ms / 1e9, 2),
            "kernels_ms": {k: round(v[0] / v[1], 3) for k, v in kt.items() if v[1]},
            "plan": {k: plan[k] for k in ("n_virtual", "prefix_modes", "suffix_modes", "prefix_rows",
                                          "suffix_rows", "diag_tables", "compute_kernel", "tile")}}


if __name__ == "__main__":
    if "--one" in sys.argv:
        cfg = sys.argv[sys.argv.index("--one") + 1]
        algo = int(sys.argv[sys.argv.index("--algo") + 1]) if "--algo" in sys.argv else 0
        print(json.dumps(one(cfg, algo)))
        sys.exit(0)
    variants = [{}, {"TNB_ENTRIES_MERGE": "0"}, {"TNB_LANE_MAJOR": "0"}]
    cfgs = ("cfg2", "cfg5")
    if "--sweep" in sys.argv:  # variants as JSON objects on the command line after --sweep
        i = sys.argv.index("--sweep")
        cfgs = (sys.argv[i + 1],)
        variants = [json.loads(a) for a in sys.argv[i + 2:]]
    for v in variants:
        for cfg in cfgs:
            env = dict(os.environ, **v)
            r = subprocess.run([sys.executable, __file__, "--one", cfg], env=env, capture_output=True, text=True)
            print(json.dumps(v), r.stdout.strip() or r.stderr[-500:], flush=True)
    if "--sweep" not in sys.argv:
        r = subprocess.run([sys.executable, __file__, "--one", "cfg5", "--algo", "2"], capture_output=True, text=True)
        print("chain", r.stdout.strip() or r.stderr[-300:])
