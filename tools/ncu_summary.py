"""Summarise an ncu report: time, key throughput metrics, stall reasons and
the hottest SASS instruction groups (grouped by execution count)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr, vals = raw[0], raw[2]
want = ["gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
d = dict(zip(hdr, zip(raw[1], vals)))
for w in want:
    for h in hdr:
        if h == w or (w.endswith("*") and h.startswith(w[:-1])):
            print(f"{h:80s} {d[h][1]} {d[h][0]}")
items = []
for h, v in zip(hdr, vals):
    if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
        try:
            items.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in items) or 1
print("stalls:", ", ".join(f"{h} {100 * v / tot:.1f}%" for v, h in sorted(items, reverse=True)[:10]))
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
h2 = rows[1]
ia, isrc, ist = h2.index("Instructions Executed"), h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)")
by, cnt, ops = collections.Counter(), collections.Counter(), collections.Counter()
tots = 0
for r in rows[2:]:
    try:
        n, s = int(r[ia]), int(r[ist] or 0)
    except (ValueError, IndexError):
        continue
    by[n] += s
    cnt[n] += 1
    tots += s
    t = r[isrc].split()
    if t:
        ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += n
print("hot groups (exec count: #instr, % of stall samples):")
for n, s in by.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    print(f"  exec={n:>10} ninstr={cnt[n]:4d} {100 * s / max(tots, 1):5.1f}%")
itot = sum(ops.values()) or 1
print("opcodes:", ", ".join(f"{k} {100 * v / itot:.1f}%" for k, v in ops.most_common(12)))
