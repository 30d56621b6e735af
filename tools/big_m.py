"""cfg2 / cfg5 chains at 2^26 tuples on the global-sort path with and without
result windows (TNB_GS_CHUNK_LOG2=0): python tools/big_m.py [cfg2|cfg5]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2206_11128_b200 as tb
import workloads as W
from paper_2206_11128_b200 import _native as N
cfg, m = sys.argv[1], 1 << int(sys.argv[2])
if cfg == "cfg2":
    shape = W.CONFIGS["cfg2"][1]
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, 32, 0)])
else:
    shape = W.CONFIGS["cfg5"][1]
    t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in W.hybrid_nodes(0)])
torch.manual_seed(5)
idx = torch.stack([torch.randint(0, s, (m,), device="cuda") for s in shape], 1)
algo = N.ALGO_GSORT
N.timing_enable(True)
for _ in range(3):
    out = tb.entries(t, idx, algo=algo)
torch.cuda.synchronize()
N.timing_enable(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    out = tb.entries(t, idx, algo=algo)
e1.record()
torch.cuda.synchronize()
print("%s m=2^%s windows=%s: %.3f ms/step  checksum %.6e" % (cfg, sys.argv[2], os.environ.get("TNB_GS_CHUNK_LOG2", "auto"),
      e0.elapsed_time(e1) / 5, out.double().sum().item()), flush=True)
'''
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
for lg in (sys.argv[2:] or ["26"]):
    for w in (os.environ.get("BIG_M_WINDOWS", "0,auto,23").split(",")):
        w = None if w == "auto" else w
        env = dict(os.environ)
        if w is None:
            env.pop("TNB_GS_CHUNK_LOG2", None)
        else:
            env["TNB_GS_CHUNK_LOG2"] = w
        subprocess.run([sys.executable, "-c", CHILD, cfg, lg], env=env, check=False)
