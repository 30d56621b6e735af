"""Per-source-line view of an ncu report: stall samples and executed
instructions for each CUDA line (inlined helpers aggregate over call sites).

    python tools/ncu_lines.py report.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_samp = hdr.index("Warp Stall Sampling (All Samples)")
i_exec = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows:
    if len(r) < len(hdr) or not r[0].isdigit():
        continue
    try:
        s = int(r[i_samp] or 0)
        n = int(r[i_exec] or 0)
    except ValueError:
        continue
    st = sorted(((int(r[i] or 0), h[6:]) for i, h in stall_cols if (r[i] or "0").isdigit()), reverse=True)
    lines.append((s, n, int(r[0]), r[1].strip()[:70], st[:3]))
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot}")
for s, n, ln, src, st in sorted(lines, reverse=True)[:top]:
    sts = " ".join(f"{h}:{100 * v / max(s, 1):.0f}%" for v, h in st if v)
    print(f"{100 * s / tot:5.1f}% L{ln:<4d} exec={n:<11d} {src:70s} {sts}")
