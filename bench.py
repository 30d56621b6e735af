"""Benchmark of the contraction hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--op entries|entries5|full|dot|norm] [--no-secondary]

Headline (BASELINE.json metric, configs[1] = "cfg2"): batched entry
evaluation t[idx] of a TT chain with N=10 modes of size 32 and ranks 32 on
2^24 uniform int64 index tuples per GPU.  A step is one K1 launch over the
whole resident batch; inputs (1.34 GB of indices) exceed the 126 MB L2, so
no flush is needed between steps.  Multi-GPU runs shard samples: every rank
evaluates its own 2^24 tuples (weak scaling, no data-path collective); the
time is the max over ranks.

``--impl reference`` times the reference's CPU algorithm (the numpy port in
oracle/, a restatement of core.py:394-444) on the host cores, rank 0 only.
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
M_PER_GPU = 1 << 24
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

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import tntz_oracle as O

    seed = W.base_seed()
    shape, rank_ = W.CONFIGS["cfg2"][1], W.CONFIGS["cfg2"][2]
    chain = O.make_chain([("tt", c) for c in W.tt_cores(shape, rank_, seed)])
    idx = W.indices(shape, REF_STEP_SAMPLE, seed + 2)
    for _ in range(args.warmup):
        O.entries(chain, idx)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.entries(chain, idx)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = REF_STEP_SAMPLE * args.steps / total
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": "TT entries/sec (t[idx])", "value": value, "unit": "entries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg2_config(args.gpus, REF_STEP_SAMPLE),
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": cores, "kind": "port",
                         "sample": f"{REF_STEP_SAMPLE} rows of the cfg2 workload per step; numpy port "
                                   "of tntz entries (core.py:394-444), float64, OpenBLAS threads"},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cfg2_config(n, m):
    return {"workload": "cfg2: " + W.CONFIGS["cfg2"][0], "samples_per_step_per_gpu": m,
            "modes": 10, "mode_size": 32, "rank": 32, "index_dtype": "int64",
            "parallelism": f"dp{n} (sample shards)",
            "l2": "inputs larger than L2 (1.34 GB of indices per step per GPU), no flush"}


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


def bench_entries(args, cfg, dev, dist, ws, rank):
    """K1 on cfg2 (default) or cfg5; returns the JSON fields."""
    import torch

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import core as C

    seed = W.base_seed()
    if cfg == "cfg2":
        shape, r = W.CONFIGS["cfg2"][1], W.CONFIGS["cfg2"][2]
        t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, r, seed)])
        m = M_PER_GPU
    else:
        shape = W.CONFIGS["cfg5"][1]
        t = tb.TnTensor([tb.ModeNode(k, c, f) for k, c, f in W.hybrid_nodes(seed)])
        m = 1 << 26
    p = t._packed()
    from paper_2206_11128_b200 import _native as N

    modes = [("diag" if md.layout == 1 else "dense", md.r_left, md.r_right) for md in p.modes]
    chain_flops_per_entry = W.entry_flops(modes)
    plan = N.entries_plan(p.chain, m, args.algo)
    idx_host = torch.from_numpy(W.indices(shape, m, seed + 2 + rank)).pin_memory()
    idx = idx_host.to(dev)
    out = torch.empty(m, dtype=torch.float32, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    wsbuf = [None]

    def step():
        wsbuf[0] = C.launch_entries(p, idx, out, err, args.algo, wsbuf[0])

    with ClockSampler(dev.index) as clk:
        ms = timed_steps(step, args.steps, args.warmup, stream, dist, kernel_timing=True)
    kt = {k: N.timing_read(k) for k in ("entries_prep", "entries_sort", "entries_compute", "entries_tables")}
    N.timing_enable(False)
    assert int(err.item()) >= t.ndim, "bench inputs must be in bounds"
    ms_step = ms / args.steps
    value = ws * m / (ms_step * 1e-3)
    peak, peak_src = fp32_peak()
    stream_k = plan["compute_kernel"] == 1
    kname = "entries_stream_kernel" if stream_k else "entries_compute_kernel"
    traffic, traffic_src = ncu_traffic(f"{cfg}_entries", kname)
    kms, kn = kt["entries_compute"]
    if kn:  # bucketed: the per-entry compute kernel, timed on its own stream
        k_ms = kms / kn
        kernel = kname
    else:  # chain / layered algorithm: one kernel is the whole step
        k_ms = ms_step
        kernel = "entries_chain_kernel"
    # algorithmic work = the reference chain's flops per entry
    # (2*r_l*r_r per dense mode, R per CP interior mode, 2R per CP end) x the
    # entries one launch processes, over the dominant kernel's launch time
    algo_flops = chain_flops_per_entry * m
    achieved = algo_flops / (k_ms * 1e-3) / 1e12
    executed = plan["kernel_flops"] / (k_ms * 1e-3) / 1e12
    per_entry = plan["kernel_flops"] / m
    launches = sum(n for k_, (_, n) in kt.items() if k_ != "entries_tables") + (
        args.steps * plan["table_launches"] if kn else 0)
    roof = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peak_src, "kernel": kernel,
            "kernel_ms": k_ms, "kernel_share_of_step": k_ms / ms_step,
            "algorithmic": (f"{chain_flops_per_entry} flop/entry (SURVEY 8(d): 2*r_l*r_r per dense mode, R per "
                            f"CP interior mode) x {m} entries per launch / compute-kernel launch time"),
            "frac_note": ("frac > 1 is possible: the kernel runs a shorter virtual chain than the reference's "
                          "(mode merging); 'executed' is its real arithmetic rate"),
            "executed": {"tflops": executed, "frac_of_fp32_peak": executed / peak,
                         "flop_per_entry": per_entry,
                         "pipe": ("tensor (mma.sync m16n8k8 split-TF32, 3 MMAs per product) for the sorted mode, "
                                  "FFMA for the closing dot" if stream_k else "fp32 (FFMA2)"),
                         "what": (f"useful arithmetic of the {plan['n_virtual']}-mode virtual chain the kernel runs "
                                  f"after merging modes 0..{plan['prefix_modes'] - 1} and the last "
                                  f"{plan['suffix_modes']} modes into prefix / suffix tables (built every call, "
                                  f"{plan['table_flops']:.3g} flop) and {plan['diag_tables']} CP run(s) into "
                                  "diagonal product tables")},
            "tensor_view": {
                "executed_tflops": plan["tensor_flops"] / (k_ms * 1e-3) / 1e12,
                "peak": TC_TF32_PEAK,
                "frac": plan["tensor_flops"] / (k_ms * 1e-3) / 1e12 / TC_TF32_PEAK,
                "what": ("split-TF32 mma.sync work of the sorted modes (3 MMAs per product) over the same kernel "
                         "time, against the measured mma.sync m16n8k8 tf32 peak (profiles/peaks_r01.json)")},
            "plan": {k: plan[k] for k in ("algo", "n_virtual", "prefix_modes", "suffix_modes",
                                          "prefix_rows", "suffix_rows", "diag_tables", "table_flops",
                                          "compute_kernel", "tile")},
            "other_kernels_ms": {k: (v[0] / v[1] if v[1] else None) for k, v in kt.items()
                                 if k != "entries_compute"},
            "other_kernels_note": ("entries_tables runs on a side stream concurrently with entries_prep / "
                                   "entries_sort (joined before the compute kernel): its span overlaps theirs"),
            "step_tflops": algo_flops / (ms_step * 1e-3) / 1e12,
            "hbm_view": {"bytes_per_launch": (8 * len(shape) + 4) * m,
                         "achieved_gbs": (8 * len(shape) + 4) * m / (ms_step * 1e-3) / 1e9}}
    fields = {"value": value, "ms_per_step": ms_step, "roofline": roof, "clocks": clk.summary(),
              "gpu_launches": launches}
    if dist:
        # the same steps followed by the NCCL all-gather of every
        # rank's output block to every rank (the only collective entries has)
        gath = torch.empty(ws * m, dtype=torch.float32, device=dev)

        def step_gather():
            step()
            torch.distributed.all_gather_into_tensor(gath, out)

        ms_g = timed_steps(step_gather, args.steps, 1, stream, dist) / args.steps
        fields["with_gather"] = {"ms_per_step": ms_g, "value": ws * m / (ms_g * 1e-3), "unit": "entries/s",
                                 "gathered_bytes_per_rank": ws * m * 4,
                                 "collective": "NCCL all_gather_into_tensor of the fp32 outputs"}
        del gath
    # e2e through the public API from pinned host memory: H2D of the step's
    # indices + K1 + D2H of the step's output, every step
    e2e_steps = max(2, min(args.steps, 3))

    out_pin = torch.empty(m, dtype=torch.float32).pin_memory()  # reused, like a serving loop would

    def e2e_step():
        # façade: chunked H2D of the pinned indices, launches, error-word
        # check and the D2H of every chunk's values into pinned host memory
        return tb.entries(t, idx_host, out=out_pin)

    e2e_step()
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist:
        tt_ = torch.tensor([el], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt_, op=torch.distributed.ReduceOp.MAX)
        el = float(tt_.item())
    fields["e2e"] = {"value": ws * m * e2e_steps / el, "unit": "entries/s",
                     "h2d_bytes_per_step": idx_host.numel() * 8, "d2h_bytes_per_step": m * 4,
                     "steps": e2e_steps, "path": "paper_2206_11128_b200.entries(t, pinned host int64, out=pinned host float32)"}
    fields["_t"], fields["_out"], fields["_idx_host"] = t, out, idx_host
    return fields


def entries_secondary(args, dev, dist, ws, rank):
    """cfg5 (BASELINE configs[4], the hybrid CP-TT-Tucker chain, 2^26 tuples)
    as a secondary line of the default run: device-resident throughput, the
    compute kernel's roofline and the end-to-end rate."""
    import copy

    a = copy.copy(args)
    a.steps, a.warmup = 3, 3
    f = bench_entries(a, "cfg5", dev, dist, ws, rank)
    for k in ("_t", "_out", "_idx_host"):
        f.pop(k)
    return {"op": "entries", "workload": "cfg5: " + W.CONFIGS["cfg5"][0], "ms_per_step": f["ms_per_step"],
            "entries/s": f["value"], "roofline": f["roofline"], "e2e": f["e2e"], "gpu_launches": f["gpu_launches"]}


def cpu_baseline_entries(t_nodes_fn, idx_host, out_dev, m_sample):
    """The oracle (numpy port of core.py:394-444) on the first m_sample rows
    of the same workload; doubles as the parity gate for the timed output."""
    from oracle import tntz_oracle as O

    chain = O.make_chain(t_nodes_fn())
    idx = idx_host[:m_sample].numpy()
    O.entries(chain, idx[:4096])  # warm-up
    t0 = time.perf_counter()
    ref = O.entries(chain, idx)
    el = time.perf_counter() - t0
    got = out_dev[:m_sample].double().cpu().numpy()
    err = O.rel_errors(got, ref)
    return {"value": m_sample / el, "unit": "entries/s", "cores": blas_threads(), "kind": "port",
            "sample": f"first {m_sample} rows of the same workload; numpy port of tntz entries "
                      "(core.py:394-444), float64, OpenBLAS threads"}, err


def bench_full(dev, steps, warmup, dist, ws=1, rank=0):
    """K2 on cfg3: full() of a TT N=4, I=256, r=64 -> 17.18 GB fp32.  With N
    ranks, rank r writes the leading-mode slab shard_bounds(256, N, r)
    (SURVEY 8(e), strong scaling: the 17.18 GB are split across the GPUs)."""
    import torch

    import paper_2206_11128_b200 as tb

    shape, r = W.CONFIGS["cfg3"][1], W.CONFIGS["cfg3"][2]
    t = tb.TnTensor([tb.ModeNode("tt", c) for c in W.tt_cores(shape, r, W.base_seed())])
    t._packed()
    from paper_2206_11128_b200 import _native as N
    from paper_2206_11128_b200.shard import shard_bounds
    import ctypes

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

    ms = timed_steps(step, steps, warmup, torch.cuda.current_stream(dev), dist, kernel_timing=True) / steps
    g_ms, g_n = N.timing_read("full_gemm")
    N.timing_enable(False)
    nbytes = out.numel() * 4  # this rank's slab
    del out
    peak, src = hbm_peak()
    k_ms = g_ms / g_n if g_n else ms
    traffic, tsrc = ncu_traffic("cfg3_full", "full_tc_gemm_kernel")
    total = 4 * int(np.prod(shape))
    return {"op": "full", "workload": "cfg3", "ms_per_step": ms, "GB/s": total / (ms * 1e-3) / 1e9,
            "bytes_written": nbytes, "slab": [lo, hi],
            "roofline": {"bound": "hbm", "achieved": nbytes / (k_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": nbytes / (k_ms * 1e-3) / 1e9 / peak, "traffic": traffic,
                         "traffic_source": tsrc, "peak_source": src, "kernel": "full_gemm (tcgen05 3xTF32)",
                         "kernel_ms": k_ms, "kernel_share_of_step": k_ms / ms,
                         "algorithmic": f"{nbytes} output bytes written per launch (4 B x 256^4)"}}


def bench_dot(dev, steps, warmup, dist, is_norm=False, ws=1, rank=0):
    """K3 on cfg4: 4096 pairs of TTs (N=16, I=64, r=16); cores drawn on the
    device (torch, seeded) since only their shapes matter for timing.  With N
    ranks each rank holds and contracts its shard_bounds(4096, N, r) pairs
    (SURVEY 8(e), strong scaling)."""
    import ctypes

    import torch

    import paper_2206_11128_b200 as tb
    from paper_2206_11128_b200 import _native as N

    shape, r = W.CONFIGS["cfg4"][1], W.CONFIGS["cfg4"][2]
    g = torch.Generator(device=dev)
    g.manual_seed(W.base_seed())
    ranks = [1] + [r] * (len(shape) - 1) + [1]
    from paper_2206_11128_b200.shard import shard_bounds

    plo, phi = shard_bounds(4096, ws, rank)
    npair = phi - plo

    def mk():
        return tb.TnTensor([tb.ModeNode("tt", torch.randn((npair, ranks[k], s, ranks[k + 1]), device=dev,
                                                          generator=g) * 0.25, batched=True)
                            for k, s in enumerate(shape)], npair)

    a, b = mk(), mk()
    pa, pb = a._packed(), b._packed()
    out = torch.empty(npair, dtype=torch.float32, device=dev)
    lib = N.load()
    st = N.stream_ptr(dev)

    def step():
        if is_norm:
            N.check(lib.tnb_norm_f32(ctypes.byref(pa.chain), out.data_ptr(), st), "norm")
        else:
            N.check(lib.tnb_dot_f32(ctypes.byref(pa.chain), ctypes.byref(pb.chain), out.data_ptr(), st), "dot")

    ms = timed_steps(step, steps, warmup, torch.cuda.current_stream(dev), dist, kernel_timing=True) / steps
    d_ms, d_n = N.timing_read("dot")
    N.timing_enable(False)
    k_ms = d_ms / d_n if d_n else ms
    per_pair = sum(ranks[k] * s * ranks[k + 1] for k, s in enumerate(shape)) * 4
    nbytes = npair * per_pair * (1 if is_norm else 2)
    peak, src = hbm_peak()
    traffic, tsrc = ncu_traffic("cfg4_dot", "dot_r16_kernel") if not is_norm else (None, None)
    # 2 * sum_k I_k (r_l r_l r_r + r_r r_l r_r) flop per pair
    # (Y = M B_j, then A_j^T Y), the same for norm
    flop = npair * 2 * sum(s * (ranks[k] * ranks[k] * ranks[k + 1] + ranks[k + 1] * ranks[k] * ranks[k + 1])
                          for k, s in enumerate(shape))
    hbm = {"bound": "hbm", "achieved": nbytes / (k_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
           "frac": nbytes / (k_ms * 1e-3) / 1e9 / peak, "traffic": traffic, "traffic_source": tsrc,
           "peak_source": src, "kernel": "dot_r16_kernel", "kernel_ms": k_ms,
           "algorithmic": f"{nbytes} core bytes read per launch (each core read once)"}
    fpk, fsrc = fp32_peak()
    fp = {"bound": "fp32", "achieved": flop / (k_ms * 1e-3) / 1e12, "peak": fpk, "unit": "TFLOP/s",
          "frac": flop / (k_ms * 1e-3) / 1e12 / fpk, "traffic": traffic, "traffic_source": tsrc,
          "peak_source": fsrc, "kernel": "dot_r16_kernel", "kernel_ms": k_ms,
          "algorithmic": f"{flop} flop per launch (SURVEY 8(d)); executed on tensor cores as split-TF32 "
                         "mma.sync (3 MMAs per product)"}
    # binding roofs per SURVEY 8(d): dot -> HBM read bandwidth, norm -> FP32
    roof, other = (fp, hbm) if is_norm else (hbm, fp)
    roof = dict(roof, other_roof=other)
    return {"op": "norm" if is_norm else "dot", "workload": "cfg4", "ms_per_step": ms,
            "pairs/s": 4096 / (ms * 1e-3), "GB/s": nbytes * ws / (ms * 1e-3) / 1e9, "roofline": roof,
            "pairs_this_rank": npair}


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    dist = ws > 1
    if dist:
        torch.distributed.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    line = {"metric": "TT entries/sec (t[idx])", "unit": "entries/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic"}
    if args.op in ("entries", "entries5"):
        cfg = "cfg2" if args.op == "entries" else "cfg5"
        f = bench_entries(args, cfg, dev, dist, ws, rank)
        t, out, idx_host = f.pop("_t"), f.pop("_out"), f.pop("_idx_host")
        line.update(f)
        line["config"] = cfg2_config(ws, M_PER_GPU) if cfg == "cfg2" else {
            "workload": "cfg5: " + W.CONFIGS["cfg5"][0], "samples_per_step_per_gpu": 1 << 26,
            "parallelism": f"dp{ws} (sample shards)", "l2": "inputs larger than L2, no flush"}
        if rank == 0 and ws == 1 and not args.no_cpu:
            seed = W.base_seed()
            nodes_fn = (lambda: [("tt", c) for c in W.tt_cores(W.CONFIGS["cfg2"][1], 32, seed)]) \
                if cfg == "cfg2" else (lambda: W.hybrid_nodes(seed))
            cb, perr = cpu_baseline_entries(nodes_fn, idx_host, out, CPU_SAMPLE)
            line["cpu_baseline"] = cb
            line["parity_gate"] = {"rows": CPU_SAMPLE, **perr,
                                   "pass": perr["rel_fro"] <= 1e-5 and perr["max_rel"] <= 1e-5}
            if not line["parity_gate"]["pass"]:
                line["value"] = None
                line["error"] = "parity gate failed: throughput not reported"
        del out
        torch.cuda.empty_cache()
        if not args.no_secondary and ws == 1:
            sec = []
            for fn in ((lambda: entries_secondary(args, dev, dist, ws, rank)) if cfg == "cfg2" else (lambda: None),
                       lambda: bench_full(dev, 3, 2, dist), lambda: bench_dot(dev, 5, 2, dist),
                       lambda: bench_dot(dev, 5, 2, dist, True)):
                try:
                    r = fn()
                    if r is not None:
                        sec.append(r)
                except Exception as e:  # noqa: BLE001
                    sec.append({"error": repr(e)})
                torch.cuda.empty_cache()
            line["secondary"] = sec
    elif args.op == "full":
        r = bench_full(dev, args.steps, args.warmup, dist, ws, rank)
        line.update({"metric": "full() GB/s", "unit": "GB/s", "value": r["GB/s"],
                     "scaling": "strong" if ws > 1 else "weak",
                     "ms_per_step": r["ms_per_step"], "roofline": r["roofline"],
                     "config": {"workload": "cfg3", "l2": "17 GB output, larger than L2"}})
    else:
        r = bench_dot(dev, args.steps, args.warmup, dist, args.op == "norm", ws, rank)
        line.update({"metric": f"{args.op}s/sec", "unit": "pairs/s", "value": r["pairs/s"],
                     "scaling": "strong" if ws > 1 else "weak",
                     "ms_per_step": r["ms_per_step"], "roofline": r["roofline"],
                     "config": {"workload": "cfg4", "l2": "4096 x 16 cores = 268 MB per operand, larger than L2"}})
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        torch.distributed.destroy_process_group()


def main():
    global TC_TF32_PEAK
    TC_TF32_PEAK = _tc_tf32_peak()
    faulthandler.enable()
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
