"""Benchmark of the contraction hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--op entries|entries5|full|dot|norm] [--no-secondary]

Headline (BASELINE.json metric, configs[1] = "cfg2"): batched entry
evaluation t[idx] of a TT chain with N=10 modes of size 32 and ranks 32 on
2^24 uniform int64 index tuples.  A step is one K1 launch over the whole
resident batch; inputs (1.34 GB of indices) exceed the 126 MB L2, so no
flush is needed between steps.

Multi-GPU: ``--gpus N`` without a torchrun environment
re-launches itself under ``torch.distributed.run`` with N ranks (one per
GPU, NCCL).  The 2^24 tuples are split into N contiguous row shards
(strong scaling, cores replicated, no data-path collective); the time is the
max over ranks, and ``with_gather`` repeats the steps followed by the NCCL
all-gather of the fp32 outputs.  ``--op full`` / ``dot`` / ``norm`` shard
leading-mode slabs / pairs the same way.

``--impl reference`` times the reference's own CPU implementation on the
host cores, rank 0 only: the real tntz from ``baseline/_ref`` when that
install is present (kind "reference"), else the numpy port in oracle/
(a restatement of core.py:394-444, kind "port").
"""

from __future__ import annotations

import argparse
import faulthandler
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PROFILES = os.path.join(ROOT, "profiles")
M_TOTAL = 1 << 24          # cfg2 tuples per step, split across the ranks (strong scaling)
M5_TOTAL = 1 << 26         # cfg5 tuples per step
CPU_SAMPLE = 1 << 20       # cpu_baseline sample (rows of the same workload)
REF_STEP_SAMPLE = 1 << 19  # --impl reference: rows per timed step


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--op", default="entries", choices=["entries", "entries5", "full", "dot", "norm"])
    ap.add_argument("--algo", type=int, default=0)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML; the recipe's nvidia-smi query)

class ClockSampler:
    REASONS = {
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            import torch

            props = torch.cuda.get_device_properties(device_index)
            ids = [getattr(props, a, None) for a in ("pci_domain_id", "pci_bus_id", "pci_device_id")]
            if all(isinstance(v, int) for v in ids):
                busid = "%08X:%02X:%02X.0" % tuple(ids)
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(busid)
            else:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(int(device_index))
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self.stop_ev.wait(0.005)  # the timed regions are tens of ms

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.th.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------

def load_json(name):
    p = os.path.join(PROFILES, name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def ncu_traffic(tag, kernel):
    """dram read+write bytes per launch of `kernel` from the newest committed
    `ncu --set full` summary profiles/ncu_r<NN>_<tag>.json (None if absent)."""
    import glob

    for path in sorted(glob.glob(os.path.join(PROFILES, f"ncu_r*_{tag}.json")), reverse=True):
        with open(path) as f:
            d = json.load(f)
        if kernel in d and d[kernel].get("dram_bytes_per_launch") is not None:
            return d[kernel]["dram_bytes_per_launch"], os.path.relpath(path, ROOT)
    return None, None


def _tc_tf32_peak():
    pk = load_json("peaks_r01.json") or {}
    return pk.get("hmma_tf32_mma_sync_tflops") or 277.6


def hbm_write_peak():
    """Write-only HBM roof: torch fill_ over 16 GiB (tools/write_peak.py),
    committed in profiles/peaks_r02.json when measured, else r01's figure."""
    for name in ("peaks_r02.json", "peaks_r01.json"):
        pk = load_json(name) or {}
        for key in ("hbm_write_fill_gbs", "hbm_write_gbs"):
            if pk.get(key):
                return pk[key], f"measured (profiles/{name} {key})"
    return None, None


def pick_roof(kernel, k_ms, pipes, traffic=None, traffic_src=None, extra=None):
    """The roofline block of one kernel.  ``pipes``: the hardware roofs the
    kernel actually exercises, each {"bound", "work" (flop or bytes per
    launch), "unit", "peak", "peak_source", "what"}; achieved = work / the
    kernel's event-timed launch duration, frac = achieved / peak, and the
    roof with the highest fraction is the binding one (the primary fields).
    DRAM traffic from an ncu capture of the same launch is its own pipe."""
    rows = []
    for pp in pipes:
        scale = 1e12 if pp["unit"] == "TFLOP/s" else 1e9
        ach = pp["work"] / (k_ms * 1e-3) / scale
        rows.append(dict(pp, achieved=ach, frac=ach / pp["peak"]))
    if traffic:
        hb, hsrc = hbm_peak()
        ach = traffic / (k_ms * 1e-3) / 1e9
        rows.append({"bound": "hbm", "work": traffic, "unit": "GB/s", "peak": hb, "peak_source": hsrc,
                     "what": f"ncu dram__bytes_read.sum + dram__bytes_write.sum per launch ({traffic_src})",
                     "achieved": ach, "frac": ach / hb})
    best = max(rows, key=lambda r: r["frac"])
    roof = {"bound": best["bound"], "achieved": best["achieved"], "peak": best["peak"], "unit": best["unit"],
            "frac": best["frac"], "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": best["peak_source"], "kernel": kernel, "kernel_ms": k_ms,
            "binding": best["what"], "pipes": rows}
    if extra:
        roof.update(extra)
    return roof


def fp32_peak():
    """Measured FFMA peak (tools/peaks.cu, committed in profiles/), else the
    nominal 148 SMs x 128 FMA/clk x 2 x 1.965 GHz."""
    pk = load_json("peaks_r01.json")
    if pk and pk.get("fp32_ffma_tflops"):
        return pk["fp32_ffma_tflops"], "measured (profiles/peaks_r01.json, tools/peaks.cu FFMA)"
    return 148 * 128 * 2 * 1.965e9 / 1e12, "nominal (148 SM x 128 FMA/clk x 2 x 1.965 GHz)"


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


TC_TF32_PEAK = None  # set in main() (profiles/peaks_r01.json)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU algorithm on the host

REF_ROOT = os.path.join(ROOT, "baseline", "_ref")


def _real_tntz():
    """The reference itself (tntz, pure numpy) from the git-ignored
    baseline/_ref install when present; None otherwise."""
    for sub in ("", "pkg/src", "src"):
        d = os.path.join(REF_ROOT, sub)
        if os.path.isdir(os.path.join(d, "tntz")):
            if d not in sys.path:
                sys.path.insert(0, d)
            try:
                import tntz  # noqa: F401

                return sys.modules["tntz"]
            except Exception:  # noqa: BLE001
                return None
    return None


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    seed = W.base_seed()
    shape, rank_ = W.CONFIGS["cfg2"][1], W.CONFIGS["cfg2"][2]
    cores = W.tt_cores(shape, rank_, seed)
    idx = W.indices(shape, REF_STEP_SAMPLE, seed + 2)
    tz = _real_tntz()
    if tz is not None:
        # the unmodified reference through its own public API: ModeNode
        # upcasts the same fp32 cores to float64 (core.py:37-38, 54)
        chain = tz.TnTensor([tz.ModeNode("tt", c) for c in cores])
        run = lambda: tz.core.entries(chain, idx)  # noqa: E731
        kind, what = "reference", ("tntz.core.entries (core.py:394-444), the unmodified reference from "
                                   "baseline/_ref, float64, OpenBLAS threads")
    else:
        from oracle import tntz_oracle as O

        chain = O.make_chain([("tt", c) for c in cores])
        run = lambda: O.entries(chain, idx)  # noqa: E731
        kind, what = "port", ("numpy port of tntz entries (oracle/, core.py:394-444), float64, "
                              "OpenBLAS threads")
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = REF_STEP_SAMPLE * args.steps / total
    cores_used = blas_threads()
    line = {
        "impl": "reference", "metric": "TT entries/sec (t[idx])", "value": value, "unit": "entries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg2_config(args.gpus, REF_STEP_SAMPLE),
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": cores_used, "kind": kind,
                         "sample": f"{REF_STEP_SAMPLE} rows of the cfg2 workload per step; {what}"},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cfg2_config(n, m):
    return {"workload": "cfg2: " + W.CONFIGS["cfg2"][0], "samples_per_step": m,
            "samples_per_step_total": M_TOTAL, "modes": 10, "mode_size": 32, "rank": 32,
            "index_dtype": "int64", "parallelism": f"dp{n} (contiguous sample shards, cores replicated)",
            "l2": "inputs larger than L2 (1.34 GB of int64 indices per step), no flush"}


# ---------------------------------------------------------------------------
# our arm

def timed_steps(fn, steps, warmup, stream, dist, kernel_timing=False):
    """Device time of exactly `steps` calls (CUDA events on `stream`, max over
    ranks).  kernel_timing: libtnb brackets its own launches inside the timed
    region with CUDA events (read back with _native.timing_read)."""
    import torch

    from paper_2206_11128_b200 import _native as N

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if kernel_timing:
        N.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def gate(err, tol=1e-5):
    """Parity gate (north_star bar): relative Frobenius AND max|d|/max|ref|."""
    return {**err, "pass": bool(err["rel_fro"] <= tol and err["max_rel"] <= tol)}


def entries_chain(cfg):
    """(façade tensor, oracle node list, shape, total tuples) of cfg2 / cfg5."""
    import paper_2206_11128_b200 as tb

    seed = W.base_seed()
    if cfg == "cfg2":
        shape, r = W.CONFIGS["cfg2"][1], W.CONFIGS["cfg2"][2]
        nodes = [("tt", c, None) for c in W.tt_cores(shape, r, seed)]
        total = M_TOTAL
    else:
        shape = W.CONFIGS["cfg5"][1]
        nodes = W.hybrid_nodes(seed)
        total = M5_TOTAL
    t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in nodes])
    return t, nodes, shape, total


def bench_entries(args, cfg, dev, dist, ws, rank, gate_rows=None):
    """K1 on cfg2 (default) or cfg5; returns the JSON fields.  The cfg's
    tuples are split into ws contiguous row shards (strong scaling); this rank
    evaluates shard_bounds(total, ws, rank)."""
    import torch

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import _native as N
    from paper_2206_11128_b200 import core as C
    from paper_2206_11128_b200.shard import shard_bounds

    seed = W.base_seed()
    t, nodes, shape, total = entries_chain(cfg)
    lo, hi = shard_bounds(total, ws, rank)
    m = hi - lo
    p = t._packed()
    modes = [("diag" if md.layout == 1 else "dense", md.r_left, md.r_right) for md in p.modes]
    chain_flops_per_entry = W.entry_flops(modes)
    plan = N.entries_plan(p.chain, m, args.algo)
    idx_np = W.indices(shape, total, seed + 2)[lo:hi]
    idx_host = torch.from_numpy(idx_np).pin_memory()
    del idx_np
    idx = idx_host.to(dev)
    out = torch.empty(m, dtype=torch.float32, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    wsbuf = [None]

    def step():
        wsbuf[0] = C.launch_entries(p, idx, out, err, args.algo, wsbuf[0])

    with ClockSampler(dev.index) as clk:
        ms = timed_steps(step, args.steps, args.warmup, stream, dist, kernel_timing=True)
    kt = {k: N.timing_read(k) for k in ("entries_prep", "entries_sort", "entries_compute", "entries_tables",
                                        "entries_mid")}
    N.timing_enable(False)
    assert int(err.item()) >= t.ndim, "bench inputs must be in bounds"
    ms_step = ms / args.steps
    value = total / (ms_step * 1e-3)
    gsort = plan["compute_kernel"] == 3
    kname = {0: "entries_compute_kernel", 1: "entries_stream_kernel", 2: "two_table_kernel",
             3: "entries_gsort_kernel"}.get(plan["compute_kernel"], "entries_compute_kernel")
    kms, kn = kt["entries_compute"]
    if kn:  # bucketed: the per-entry compute kernel, timed on its own stream
        k_ms = kms / kn
        kernel = kname
        traffic, traffic_src = ncu_traffic(f"{cfg}_entries", kname) if ws == 1 else (None, None)
    else:  # chain / layered algorithm: one kernel is the whole step
        k_ms = ms_step
        kernel = "entries_chain_kernel"
        traffic, traffic_src = None, None
    fpk, fsrc = fp32_peak()
    sorted_flops = plan["tensor_flops"] / 3.0
    pipes = [{"bound": "fp32", "work": plan["kernel_flops"] - sorted_flops, "unit": "TFLOP/s", "peak": fpk,
              "peak_source": fsrc,
              "what": "FFMA work the kernel issues outside the tensor-core modes (first-mode copy, diagonal "
                      "modes, the closing dot), per launch"}]
    if gsort:
        # global-sort kernel: per entry one gathered row of the first table,
        # one of the last (and diag) table, its 16-byte record, a 4-byte result
        r0 = p.modes[plan["prefix_modes"] - 1].r_right
        r1 = p.modes[len(p.modes) - plan["suffix_modes"]].r_left
        per_entry = 4 * r0 + 4 * r1 * (2 if plan["n_virtual"] == 4 else 1) + 16 + 4
        hb, hsrc = hbm_peak()
        gb = load_json("gather_bench_r02.json") or {}
        pipes.append({"bound": "hbm", "work": float(per_entry) * m, "unit": "GB/s", "peak": hb, "peak_source": hsrc,
                      "what": (f"gathered bytes the kernel requests per launch ({per_entry} B per entry: table rows, "
                               "record, result); the measured ceiling of random 128-byte row gathers from HBM is "
                               f"{gb.get('hbm_random_row_gather_gbs', 5320)} GB/s (tools/gather_bench.cu, "
                               "profiles/gather_bench_r02.json)")})
        bf = None
        mp_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(mp_path):
            with open(mp_path) as f:
                bf = json.load(f).get("bf16_tflops")
        pipes.append({"bound": "tensor", "work": plan["tensor_flops"], "unit": "TFLOP/s",
                      "peak": (bf or 2250.0) / 2.0,
                      "peak_source": ("half the measured dense bf16 cuBLAS rate (MEASURED_PEAKS.json bf16_tflops): "
                                      "tcgen05 kind::tf32 runs at half the bf16 rate" if bf else
                                      "nominal dense tf32 (half of 2.25 PFLOP/s bf16)"),
                      "what": "3xTF32 tcgen05.mma work of the merged sorted mode (2 MMAs per k-step: Ahi x [Bhi|Blo], "
                              "Alo x Bhi; 3 * 2*r0*r1 flop per entry), per launch"})
    elif plan["tensor_flops"] > 0:
        pipes.append({"bound": "tensor", "work": plan["tensor_flops"], "unit": "TFLOP/s", "peak": TC_TF32_PEAK,
                      "peak_source": "measured (profiles/peaks_r01.json, tools/peaks.cu mma.sync m16n8k8 tf32)",
                      "what": "split-TF32 mma.sync work of the sorted modes (3 MMAs per product, 2*r_l*r_r "
                              "flop each), per launch"})
    algo_flops = chain_flops_per_entry * m
    extra = {
        "kernel_share_of_step": k_ms / ms_step,
        "algorithmic_rate": {
            "tflops": algo_flops / (k_ms * 1e-3) / 1e12, "vs_fp32_peak": algo_flops / (k_ms * 1e-3) / 1e12 / fpk,
            "what": (f"the reference chain's {chain_flops_per_entry} flop/entry (SURVEY 8(d): 2*r_l*r_r per dense "
                     f"mode, R per CP interior mode) x {m} entries / compute-kernel time; above 1 because mode "
                     "merging leaves the kernel a shorter virtual chain -- a rate, not a pipe utilisation")},
        "plan": {k: plan[k] for k in ("algo", "n_virtual", "prefix_modes", "suffix_modes", "prefix_rows",
                                      "suffix_rows", "diag_tables", "table_flops", "compute_kernel", "tile")},
        "other_kernels_ms": {k: (v[0] / v[1] if v[1] else None) for k, v in kt.items() if k != "entries_compute"},
        "other_kernels_note": ("entries_tables (and entries_mid, the merged sorted mode's slice images) run on a side "
                               "stream concurrently with entries_prep / entries_sort (joined before the compute "
                               "kernel): their span overlaps those"),
        "algorithmic_bytes": {"per_entry": 8 * len(shape) + 4, "what": "int64 index row + fp32 output",
                              "step_gbs": (8 * len(shape) + 4) * m / (ms_step * 1e-3) / 1e9},
    }
    roof = pick_roof(kernel, k_ms, pipes, traffic, traffic_src, extra)
    # event-timed launches (prep, sort, compute) + per step the table builds,
    # detect_hot_kernel and the second (HOT) compute instantiation that
    # returns at once when the flag does not match (the timer brackets both)
    if gsort:  # prep, detect_hot, scan, scatter, compute + the table / slice-image builds
        launches = args.steps * (5 + plan["table_launches"])
    else:
        launches = sum(n for k_, (_, n) in kt.items() if k_ not in ("entries_tables", "entries_mid")) + (
            args.steps * (plan["table_launches"] + (2 if plan["compute_kernel"] in (0, 1) else 0)) if kn else 0)
    fields = {"value": value, "ms_per_step": ms_step, "roofline": roof, "clocks": clk.summary(),
              "gpu_launches": launches, "shard": [lo, hi]}
    if dist:
        # the same steps followed by the NCCL all-gather of every
        # rank's output block to every rank (the only collective entries has)
        base = (total + ws - 1) // ws
        pad = torch.zeros(base, dtype=torch.float32, device=dev)
        gath = torch.empty(ws * base, dtype=torch.float32, device=dev)

        gloo = torch.distributed.get_backend() == "gloo"

        def step_gather():
            step()
            pad[:m].copy_(out)
            if gloo:  # host round trip (gloo gathers CPU tensors)
                g = gath.cpu()
                torch.distributed.all_gather_into_tensor(g, pad.cpu())
                gath.copy_(g)
            else:
                torch.distributed.all_gather_into_tensor(gath, pad)

        ms_g = timed_steps(step_gather, args.steps, 1, stream, dist) / args.steps
        fields["with_gather"] = {"ms_per_step": ms_g, "value": total / (ms_g * 1e-3), "unit": "entries/s",
                                 "gathered_bytes_per_rank": ws * base * 4,
                                 "collective": ("gloo (host) " if gloo else "NCCL ") +
                                               "all_gather_into_tensor of the fp32 outputs"}
        del gath, pad
    # e2e through the public API from pinned host memory: H2D of the step's
    # indices + K1 + D2H of the step's output, every step
    e2e_steps = max(2, min(args.steps, 3))
    out_pin = torch.empty(m, dtype=torch.float32).pin_memory()  # reused, like a serving loop would

    def e2e_step():
        # façade: chunked, codec-narrowed H2D of the pinned indices, launches,
        # error-word check and the D2H of every chunk's values
        return tb.entries(t, idx_host, out=out_pin)

    e2e_step()
    torch.cuda.synchronize()
    xfer = dict(C.last_transfer)
    if dist:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    h2d_sum = 0
    for _ in range(e2e_steps):
        e2e_step()
        # the self-balancing pipeline picks the raw / narrowed chunk mix per call
        h2d_sum += C.last_transfer.get("h2d_bytes", idx_host.numel() * 8)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist:
        tt_ = torch.tensor([el], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt_, op=torch.distributed.ReduceOp.MAX)
        el = float(tt_.item())
    fields["e2e"] = {"value": total * e2e_steps / el, "unit": "entries/s",
                     "h2d_bytes_per_step": h2d_sum // e2e_steps * ws,
                     "d2h_bytes_per_step": m * 4 * ws, "steps": e2e_steps,
                     "index_codec": xfer.get("codec", "int64"),
                     "path": "paper_2206_11128_b200.entries(t, pinned host int64, out=pinned host float32)",
                     "note": ("host int64 indices cross PCIe narrowed to int8 by the index transport codec "
                              "(tnb_narrow_indices_host, a pure range check on host threads) and are widened "
                              "on the device; wrap / bounds / OOB report stay in the device prep kernel")}
    # parity gate on this rank's timed output (rank 0 prints it)
    if rank == 0 and not args.no_cpu:
        from oracle import tntz_oracle as O

        rows = gate_rows if gate_rows is not None else min(CPU_SAMPLE, m)
        sel = np.arange(rows) if gate_rows is None else np.linspace(0, m - 1, rows).astype(np.int64)
        chain = O.make_chain(nodes)
        sub = idx_host.numpy()[sel]
        t0 = time.perf_counter()
        ref = O.entries(chain, sub)
        el_cpu = time.perf_counter() - t0
        got = out.double().cpu().numpy()[sel]
        fields["parity_gate"] = {"rows": int(rows), "rows_from": "first rows" if gate_rows is None else
                                 "evenly spaced over the shard", **gate(O.rel_errors(got, ref))}
        fields["_cpu"] = {"value": rows / el_cpu, "unit": "entries/s", "cores": blas_threads(), "kind": "port",
                          "sample": f"{rows} rows of the same workload; numpy port of tntz entries "
                                    "(oracle/, core.py:394-444), float64, OpenBLAS threads"}
        if not fields["parity_gate"]["pass"]:
            fields["value"] = None
            fields["error"] = "parity gate failed: throughput not reported"
    fields["_t"] = t
    return fields


def entries_secondary(args, dev, dist, ws, rank):
    """cfg5 (BASELINE configs[4], the hybrid CP-TT-Tucker chain, 2^26 tuples)
    as a secondary line of the default run: device-resident throughput, the
    compute kernel's roofline, the end-to-end rate and a parity gate on 2^18
    rows spread over the whole batch."""
    import copy

    a = copy.copy(args)
    a.steps, a.warmup = 3, 3
    f = bench_entries(a, "cfg5", dev, dist, ws, rank, gate_rows=1 << 18)
    f.pop("_t")
    f.pop("_cpu", None)
    res = {"op": "entries", "workload": "cfg5: " + W.CONFIGS["cfg5"][0], "ms_per_step": f["ms_per_step"],
           "entries/s": f["value"], "roofline": f["roofline"], "e2e": f["e2e"], "gpu_launches": f["gpu_launches"]}
    if "parity_gate" in f:
        res["parity_gate"] = f["parity_gate"]
    return res


def bench_entries_batched(dev, steps, warmup, B=16, m=1 << 20):
    """Batched-chain entries (core.py:425-429, 447-460): a batch of B cfg2-shape
    chains (N=10, I=32, r=32) on the same 2^20 tuples, output [m, B], on the
    global-sort kernels when the merge allows (records sorted once, per-element
    tables / compute), else the bucketed kernels (shared tile records)."""
    import torch

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import _native as N
    from paper_2206_11128_b200 import core as C

    seed = W.base_seed()
    shape = W.CONFIGS["cfg2"][1]
    cores = W.tt_cores(shape, 32, seed + 7, batch_size=B)
    t = tb.TnTensor([tb.ModeNode("tt", c, batched=True) for c in cores], B)
    p = t._packed()
    idx_np = W.indices(shape, m, seed + 8)
    idx = torch.from_numpy(idx_np).to(dev)
    out = torch.empty((m, B), dtype=torch.float32, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    plan = N.entries_plan(p.chain, m)
    wsbuf = [None]

    def step():
        wsbuf[0] = C.launch_entries(p, idx, out, err, 0, wsbuf[0])

    ms = timed_steps(step, steps, warmup, torch.cuda.current_stream(dev), False, kernel_timing=True) / steps
    kt = {k: N.timing_read(k) for k in ("entries_prep", "entries_sort", "entries_compute", "entries_tables",
                                        "entries_mid")}
    N.timing_enable(False)
    kms, kn = kt["entries_compute"]
    k_ms = kms / steps if kn else ms  # the B compute launches of one step
    fpk, fsrc = fp32_peak()
    gsort = plan["compute_kernel"] == 3
    if gsort:
        # global-sort kernel per element over records sorted once: per entry and
        # element one row of each table (128 B each), the 16-byte record, a result
        hb, hsrc = hbm_peak()
        pipes = [{"bound": "hbm", "work": float(2 * 128 + 16 + 4) * m * B, "unit": "GB/s", "peak": hb,
                  "peak_source": hsrc,
                  "what": "gathered bytes the B compute launches request (two 128-byte table rows, record, result "
                          "per entry and element); the step is dominated by the per-element table builds, which "
                          "cannot overlap the persistent compute kernel (both fill the GPU)"}]
    else:
        pipes = [{"bound": "tensor", "work": plan["tensor_flops"], "unit": "TFLOP/s", "peak": TC_TF32_PEAK,
                  "peak_source": "measured (profiles/peaks_r01.json, tools/peaks.cu mma.sync m16n8k8 tf32)",
                  "what": "split-TF32 mma.sync work of the sorted modes over the B compute launches"},
                 {"bound": "fp32", "work": plan["kernel_flops"] - plan["tensor_flops"] / 3, "unit": "TFLOP/s",
                  "peak": fpk, "peak_source": fsrc, "what": "FFMA work outside the tensor-core modes"}]
    roof = pick_roof(("entries_gsort_kernel" if gsort else "entries_compute_kernel") + " x B", k_ms, pipes,
                     extra={"kernel_share_of_step": k_ms / ms,
                            "plan": {k: plan[k] for k in ("algo", "n_virtual", "prefix_rows", "suffix_rows",
                                                          "compute_kernel")},
                            "tables_ms_per_step": (kt["entries_tables"][0] + kt["entries_mid"][0]) / steps})
    from oracle import tntz_oracle as O

    sel = np.linspace(0, m - 1, 4096).astype(np.int64)
    o = O.make_chain([("tt", c) for c in cores], B)
    ref = O.entries(o, idx_np[sel])
    pg = gate(O.rel_errors(out.double().cpu().numpy()[sel], ref))
    return {"op": "entries_batched", "workload": f"B={B} cfg2-shape chains (N=10, I=32, r=32), {m} tuples, "
                                                 f"output [m, B]", "ms_per_step": ms,
            "entries/s": m * B / (ms * 1e-3), "roofline": roof,
            "parity_gate": {"rows": len(sel), "what": "evenly spaced rows x all B", **pg}}


def bench_full(dev, steps, warmup, dist, ws=1, rank=0, parity=True):
    """K2 on cfg3: full() of a TT N=4, I=256, r=64 -> 17.18 GB fp32.  With N
    ranks, rank r writes the leading-mode slab shard_bounds(256, N, r)
    (SURVEY 8(e), strong scaling: the 17.18 GB are split across the GPUs).
    Parity gate: the first and last leading-mode slices of this rank's slab
    against the oracle's full_slab (core.py:337-359)."""
    import ctypes

    import torch

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import _native as N
    from paper_2206_11128_b200.shard import shard_bounds

    shape, r = W.CONFIGS["cfg3"][1], W.CONFIGS["cfg3"][2]
    cores = W.tt_cores(shape, r, W.base_seed())
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in cores])
    lo, hi = shard_bounds(shape[0], ws, rank)
    out = torch.empty((hi - lo,) + tuple(shape[1:]), dtype=torch.float32, device=dev)
    p = t._packed()
    lib = N.load()
    wsb = lib.tnb_full_workspace_bytes(ctypes.byref(p.chain), lo, hi)
    wsbuf = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    st = N.stream_ptr(dev)

    def step():
        N.check(lib.tnb_full_f32(ctypes.byref(p.chain), lo, hi, out.data_ptr(),
                                 wsbuf.data_ptr(), wsb, st), "full")

    with ClockSampler(dev.index) as clk:
        ms = timed_steps(step, steps, warmup, torch.cuda.current_stream(dev), dist, kernel_timing=True) / steps
    g_ms, g_n = N.timing_read("full_gemm")
    N.timing_enable(False)
    nbytes = out.numel() * 4  # this rank's slab
    res = {}
    if parity and rank == 0:
        from oracle import tntz_oracle as O

        o = O.make_chain([("tt", c) for c in cores])
        errs = []
        for s_ in sorted({lo, hi - 1}):
            ref = O.full_slab(o, s_, s_ + 1)
            errs.append(O.rel_errors(out[s_ - lo:s_ - lo + 1].double().cpu().numpy(), ref))
        worst = {k: max(e[k] for e in errs) for k in errs[0]}
        res["parity_gate"] = {"slabs": sorted({lo, hi - 1}), "what": "full(t[i:i+1]) of the oracle", **gate(worst)}
    del out
    peak, src = hbm_peak()
    k_ms = g_ms / g_n if g_n else ms
    traffic, tsrc = ncu_traffic("cfg3_full", "full_tc_gemm_kernel") if ws == 1 else (None, None)
    wpk, wsrc = hbm_write_peak()
    K = r
    pipes = [{"bound": "hbm", "work": nbytes, "unit": "GB/s", "peak": peak, "peak_source": src,
              "what": f"{nbytes} output bytes written per launch (4 B x the slab's elements)"}]
    extra = {"kernel_share_of_step": k_ms / ms,
             "algorithmic": f"{nbytes} output bytes written per launch (4 B x the slab's elements)",
             "tensor_view": {"tflops": 3 * 2 * (nbytes / 4) * K / (k_ms * 1e-3) / 1e12,
                             "what": "3xTF32 tcgen05.mma work of the final GEMM (3 MMAs per product) over the "
                                     "kernel time; nominal dense tf32 is 1100 TFLOP/s (no measured figure)"}}
    if wpk:
        extra["frac_vs_write_only"] = nbytes / (k_ms * 1e-3) / 1e9 / wpk
        extra["write_only_peak"] = {"gbs": wpk, "source": wsrc}
    roof = pick_roof("full_tc_gemm_kernel (tcgen05 3xTF32)", k_ms, pipes, None, None, extra)
    roof["traffic"], roof["traffic_source"] = traffic, tsrc
    if traffic:
        roof["traffic_over_algorithmic"] = traffic / nbytes
    total = 4 * int(np.prod(shape))
    res.update({"op": "full", "workload": "cfg3", "ms_per_step": ms, "GB/s": total / (ms * 1e-3) / 1e9,
                "bytes_written": nbytes, "slab": [lo, hi], "roofline": roof, "clocks": clk.summary()})
    return res


_CFG4 = {}


def cfg4_cores(seed):
    """cfg4 operand cores from the pinned generator (random_tt(..., batch_size
    =4096, scale=0.25), random.py:28-40), generated once per process."""
    if seed not in _CFG4:
        shape, r = W.CONFIGS["cfg4"][1], W.CONFIGS["cfg4"][2]
        _CFG4[seed] = W.tt_cores(shape, r, seed, batch_size=4096, scale=0.25)
    return _CFG4[seed]


def bench_dot(dev, steps, warmup, dist, is_norm=False, ws=1, rank=0, parity=True):
    """K3 on cfg4: 4096 pairs of TTs (N=16, I=64, r=16), cores from the pinned
    generator (a: seed, b: seed + 1).  With N ranks each rank holds and
    contracts its shard_bounds(4096, N, r) pairs (SURVEY 8(e), strong
    scaling).  Parity gate: 256 pairs spread over the batch against the
    oracle's chain_dot / norm (core.py:362-391)."""
    import ctypes

    import torch

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import _native as N
    from paper_2206_11128_b200.shard import shard_bounds

    shape, r = W.CONFIGS["cfg4"][1], W.CONFIGS["cfg4"][2]
    seed = W.base_seed()
    ranks = [1] + [r] * (len(shape) - 1) + [1]
    plo, phi = shard_bounds(4096, ws, rank)
    npair = phi - plo

    def mk(sd):
        return tb.TnTensor([tb.ModeNode("tt", torch.from_numpy(c[plo:phi]).to(dev), batched=True)
                            for c in cfg4_cores(sd)], npair)

    a = mk(seed)
    b = a if is_norm else mk(seed + 1)
    pa, pb = a._packed(), b._packed()
    out = torch.empty(npair, dtype=torch.float32, device=dev)
    lib = N.load()
    st = N.stream_ptr(dev)

    def step():
        if is_norm:
            N.check(lib.tnb_norm_f32(ctypes.byref(pa.chain), out.data_ptr(), st), "norm")
        else:
            N.check(lib.tnb_dot_f32(ctypes.byref(pa.chain), ctypes.byref(pb.chain), out.data_ptr(), st), "dot")

    with ClockSampler(dev.index) as clk:
        ms = timed_steps(step, steps, warmup, torch.cuda.current_stream(dev), dist, kernel_timing=True) / steps
    d_ms, d_n = N.timing_read("dot")
    N.timing_enable(False)
    k_ms = d_ms / d_n if d_n else ms
    per_pair = sum(ranks[k] * s * ranks[k + 1] for k, s in enumerate(shape)) * 4
    nbytes = npair * per_pair * (1 if is_norm else 2)
    peak, src = hbm_peak()
    traffic, tsrc = ncu_traffic("cfg4_norm" if is_norm else "cfg4_dot", "dot_r16_kernel") \
        if ws == 1 else (None, None)
    # 2 * sum_k I_k (r_l r_l r_r + r_r r_l r_r) flop per pair
    # (Y = M B_j, then A_j^T Y), the same for norm
    flop = npair * 2 * sum(s * (ranks[k] * ranks[k] * ranks[k + 1] + ranks[k + 1] * ranks[k] * ranks[k + 1])
                          for k, s in enumerate(shape))
    fpk, fsrc = fp32_peak()
    # interior modes run as split-TF32 mma.sync (3 MMAs per product); the
    # rank-1 boundary modes (2 of 16) as FFMA
    interior = npair * 2 * sum(s * 2 * ranks[k] * ranks[k] * ranks[k + 1] for k, s in enumerate(shape)
                               if 0 < k < len(shape) - 1)
    pipes = [{"bound": "hbm", "work": nbytes, "unit": "GB/s", "peak": peak, "peak_source": src,
              "what": f"{nbytes} core bytes read per launch (each core read once)"},
             {"bound": "tensor", "work": 3 * interior, "unit": "TFLOP/s", "peak": TC_TF32_PEAK,
              "peak_source": "measured (profiles/peaks_r01.json, tools/peaks.cu mma.sync m16n8k8 tf32)",
              "what": "split-TF32 mma.sync work of the interior modes (3 MMAs per product), per launch"}]
    extra = {"algorithmic_rate": {"tflops": flop / (k_ms * 1e-3) / 1e12,
                                  "vs_fp32_peak": flop / (k_ms * 1e-3) / 1e12 / fpk,
                                  "what": f"{flop} flop per launch (SURVEY 8(d)) over the kernel time"}}
    roof = pick_roof("dot_r16_kernel" + ("<norm>" if is_norm else ""), k_ms, pipes, None, None, extra)
    roof["traffic"], roof["traffic_source"] = traffic, tsrc
    if traffic:
        roof["traffic_over_algorithmic"] = traffic / nbytes
    res = {"op": "norm" if is_norm else "dot", "workload": "cfg4", "ms_per_step": ms,
           "pairs/s": 4096 / (ms * 1e-3), "GB/s": nbytes * ws / (ms * 1e-3) / 1e9, "roofline": roof,
           "pairs_this_rank": npair, "clocks": clk.summary()}
    if parity and rank == 0:
        from oracle import tntz_oracle as O

        sel = np.linspace(0, npair - 1, min(256, npair)).astype(np.int64)
        ca = [c[plo:phi][sel] for c in cfg4_cores(seed)]
        oa = O.make_chain([("tt", c) for c in ca], len(sel))
        got = out.double().cpu().numpy()[sel]
        if is_norm:
            ref = O.norm(oa)
            errs = np.abs(got - ref) / np.abs(ref)
        else:
            cb = [c[plo:phi][sel] for c in cfg4_cores(seed + 1)]
            ob = O.make_chain([("tt", c) for c in cb], len(sel))
            ref = O.chain_dot(oa, ob)
            # dots cancel: the error is measured against ||a|| ||b|| (tests/helpers.assert_dot_close)
            errs = np.abs(got - ref) / (O.norm(oa) * O.norm(ob))
        res["parity_gate"] = {"pairs": len(sel), "what": "evenly spaced over the batch",
                              "max_err": float(errs.max()), "pass": bool(errs.max() <= 1e-5),
                              "err_scale": "|ref|" if is_norm else "||a|| ||b||"}
    return res


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    dist = ws > 1
    if dist:
        # TNB_BENCH_BACKEND=gloo: the same multi-rank path with ranks sharing
        # one GPU (harness check on a one-GPU box; collectives via host memory)
        torch.distributed.init_process_group(os.environ.get("TNB_BENCH_BACKEND", "nccl"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    line = {"metric": "TT entries/sec (t[idx])", "unit": "entries/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic"}
    if args.op in ("entries", "entries5"):
        cfg = "cfg2" if args.op == "entries" else "cfg5"
        f = bench_entries(args, cfg, dev, dist, ws, rank, gate_rows=None if cfg == "cfg2" else 1 << 18)
        f.pop("_t")
        cpu = f.pop("_cpu", None)
        line.update(f)
        line["config"] = cfg2_config(ws, f["shard"][1] - f["shard"][0]) if cfg == "cfg2" else {
            "workload": "cfg5: " + W.CONFIGS["cfg5"][0], "samples_per_step_total": M5_TOTAL,
            "parallelism": f"dp{ws} (contiguous sample shards)", "l2": "inputs larger than L2, no flush"}
        if rank == 0 and ws == 1 and cpu is not None:
            line["cpu_baseline"] = cpu
        torch.cuda.empty_cache()
        if not args.no_secondary and ws == 1:
            sec = []
            for fn in ((lambda: entries_secondary(args, dev, dist, ws, rank)) if cfg == "cfg2" else (lambda: None),
                       lambda: bench_entries_batched(dev, 5, 3),
                       lambda: bench_full(dev, 3, 3, dist), lambda: bench_dot(dev, 5, 3, dist),
                       lambda: bench_dot(dev, 5, 3, dist, True)):
                try:
                    r = fn()
                    if r is not None:
                        sec.append(r)
                except Exception as e:  # noqa: BLE001
                    sec.append({"error": repr(e)})
                torch.cuda.empty_cache()
            line["secondary"] = sec
    elif args.op == "full":
        r = bench_full(dev, args.steps, args.warmup, dist, ws, rank, parity=not args.no_cpu)
        line.update({"metric": "full() GB/s", "unit": "GB/s", "value": r["GB/s"],
                     "ms_per_step": r["ms_per_step"], "roofline": r["roofline"], "clocks": r["clocks"],
                     "config": {"workload": "cfg3", "parallelism": f"dp{ws} (leading-mode slabs)",
                                "l2": "17 GB output, larger than L2"}})
        if "parity_gate" in r:
            line["parity_gate"] = r["parity_gate"]
    else:
        r = bench_dot(dev, args.steps, args.warmup, dist, args.op == "norm", ws, rank, parity=not args.no_cpu)
        line.update({"metric": f"{args.op}s/sec", "unit": "pairs/s", "value": r["pairs/s"],
                     "ms_per_step": r["ms_per_step"], "roofline": r["roofline"], "clocks": r["clocks"],
                     "config": {"workload": "cfg4", "parallelism": f"dp{ws} (pair shards)",
                                "l2": "4096 x 16 cores = 3.8 GB per operand, larger than L2"}})
        if "parity_gate" in r:
            line["parity_gate"] = r["parity_gate"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        torch.distributed.destroy_process_group()


def _free_port():
    import socket

    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    return port


def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` outside torchrun: re-exec as N ranks (one
    per GPU) under torch.distributed.run on 127.0.0.1, NCCL INFO on so the
    log shows the communicator (nranks, NVLS / NVLink transport)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    os.execvpe(sys.executable, cmd, env)


def main():
    global TC_TF32_PEAK
    TC_TF32_PEAK = _tc_tf32_peak()
    faulthandler.enable()
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    run_ours(args)


if __name__ == "__main__":
    main()
