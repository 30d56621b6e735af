"""Turn ncu outputs from gpurun_out/ into committed summaries under profiles/.

    python tools/summarize_ncu.py <tag> [launches.csv] [report.ncu-rep ...]

Writes profiles/<tag>_launches.txt (per-kernel launch counts, mean device
time and share of the step, from the `--metrics gpu__time_duration.sum` pass)
and profiles/<tag>_<kernel>.txt (key `--set full` metrics, stall reasons and
the hottest SASS instruction groups) plus profiles/ncu_<tag>.json with the
per-launch DRAM traffic that bench.py reports as roofline.traffic.
"""

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[hi + 1:]:
        try:
            d.setdefault(r[ik], []).append(float(r[iv].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in d.values()) or 1
    lines = [f"# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)",
             f"{'kernel':90s} {'launches':>8s} {'mean_us':>12s} {'share':>7s}"]
    for k, v in d.items():
        lines.append(f"{k[:90]:90s} {len(v):8d} {sum(v) / len(v) / 1e3:12.3f} {100 * sum(v) / tot:6.1f}%")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def report(tag, rep):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = raw[0], raw[1]
    out = {}
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"]
        short = name.split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
        stalls = sorted(((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for h, v in d.items()
                         if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and v),
                        reverse=True)
        st = sum(v for v, _ in stalls) or 1
        lines = [f"# {tag} / {name}", "", "## key metrics (ncu --set full --clock-control none)"]
        for k in KEYS:
            if k in d:
                lines.append(f"{k:80s} {d[k]} {u.get(k, '')}")
        lines += ["", "## stall reasons (share of samples)"]
        lines += [f"{h:40s} {100 * v / st:5.1f}%" for v, h in stalls[:10]]
        traffic = None
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            traffic = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
                to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        out[short] = {"kernel": name, "duration": d.get("gpu__time_duration.sum"),
                      "duration_unit": u.get("gpu__time_duration.sum"), "dram_bytes_per_launch": traffic}
        open(os.path.join(PROF, f"{tag}_{short}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines[:20]))
    return out


if __name__ == "__main__":
    tag = sys.argv[1]
    summary = {}
    for p in sys.argv[2:]:
        if p.endswith(".csv"):
            launches(tag, p)
        else:
            summary.update(report(tag, p))
    if summary:
        path = os.path.join(PROF, f"ncu_{tag}.json")
        json.dump(summary, open(path, "w"), indent=1)
