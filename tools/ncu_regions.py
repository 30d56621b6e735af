"""Stall samples of the entries compute kernel grouped by code region (line
ranges located by markers in entries_bucketed.cu; inlined helpers above the
kernel count as 'helpers').

    python tools/ncu_regions.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

SRC = Path(__file__).resolve().parents[1] / "paper_2206_11128_b200" / "csrc" / "entries_bucketed.cu"
lines = SRC.read_text().splitlines()


def find(text, start=0):
    for i in range(start, len(lines)):
        if text in lines[i]:
            return i + 1
    raise KeyError(text)


k0 = find("entries_compute_kernel(const __grid_constant__ ChainDev ch")
marks = [
    ("helpers (lds/ffma2/shfl, ks_passes)", 1),
    ("kernel setup / tile loop", k0),
    ("first mode", find("if (k == 0) {", k0)),
    ("diag run", find("} else if (md.layout == TNB_LAYOUT_DIAG) {", k0)),
    ("last mode", find("} else if (k == N - 1) {", k0)),
    ("sorted: setup + G loads", find("// ---- sorted mode", k0)),
    ("sorted R32 pass loop", find("while (bend - p >= 8) {", k0)),
    ("sorted R<=24 (Geo)", find("if (!bp.rounds) {", k0)),
    ("mode barrier + prefetch", find("// cidx rows k..k2 of this tile are dead", k0) - 2),
    ("after kernel", find("int pick_R(int rmax)")),
]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
agg = {name: 0 for name, _ in marks}
tot = 0
for r in rows:
    if len(r) < len(hdr) or not r[0].isdigit():
        continue
    try:
        ln, smp = int(r[0]), int(r[i_s] or 0)
    except ValueError:  # source text with unescaped quotes: skip the row
        continue
    tot += smp
    name = marks[0][0]
    for nm, start in marks:
        if ln >= start:
            name = nm
    if ln < k0 and "ks_passes" not in name:
        name = marks[0][0]
    agg[name] += smp
for nm, _ in marks:
    if agg[nm]:
        print(f"{100 * agg[nm] / max(tot, 1):5.1f}%  {nm}")
