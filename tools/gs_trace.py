"""Per-role phase times of the global-sort compute kernel: build the trace
variant (python tools/build_variant.py trace -DTNB_GS_TRACE=1), run
TNB_LIB=build/variants/trace/libtnb.so TNB_GS_TRACE_FILE=/tmp/gs.trace python tools/bench_entries.py --one cfg2
then python tools/gs_trace.py /tmp/gs.trace TILES_PER_CTA"""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
a = raw[:256 * 24].reshape(256, 4, 6).astype(np.float64)[:148]
tiles = float(sys.argv[2])
names = {0: ("mma", ["wait a_ready(+loop, image)", "wait acc_empty", "issue", "", "", ""]),
         1: ("epilogue", ["wait full_raw", "closing rows + wait acc_full", "tmem ld, dot, store", "", "", ""]),
         2: ("producer", ["(trace)", "wait stage", "issue gathers", "record ring refill", "row prefetch", "wait record"]),
         3: ("splitter", ["wait full_raw", "wait alo", "split", "", "", ""])}
for r in range(4):
    tot = a[:, r, :].sum(axis=1).mean()
    print(f"{names[r][0]:9s} total {tot / tiles:8.1f} cyc/tile")
    for e in range(6):
        if names[r][1][e]:
            print(f"    {names[r][1][e]:32s} {a[:, r, e].mean() / tiles:8.1f} cyc/tile")

st = raw[8192:8192 + 32 * 16].reshape(32, 16).astype(np.int64)
b = st[st > 0].min()
print("tile | prod: rec stage issued | split: full_raw done | mma: a_ready issued | epi: acc_full done   (cycles, CTA 0)")
for i in range(32):
    r = [int(st[i, e] - b) if st[i, e] else -1 for e in (0, 1, 2, 3, 5, 6, 7, 8, 9)]
    print(f"{256 + i:4d} | {r[0]:6d} {r[1]:6d} {r[2]:6d} | {r[3]:6d} {r[4]:6d} | {r[5]:6d} {r[6]:6d} | {r[7]:6d} {r[8]:6d}")
