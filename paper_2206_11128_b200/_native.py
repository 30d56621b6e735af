"""ctypes binding of libtnb.so (the C ABI declared in include/tnb.h).

There is deliberately no fallback: if the library is missing or no sm_100
device is present, every compute entry point raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

from .errors import ContractViolationError, NativeError

# TNB_LIB: an alternative build of the same library (tools/build_variant.py
# compiles kernel variants for A/B timing); the default is the in-tree build
LIB_PATH = Path(os.environ.get("TNB_LIB") or Path(__file__).resolve().parent / "libtnb.so")

TNB_OK, TNB_EINVAL, TNB_EINDEX, TNB_ECUDA, TNB_EWORKSPACE = 0, 1, 2, 3, 4
KIND_TT, KIND_CP = 0, 1
LAYOUT_DENSE, LAYOUT_DIAG = 0, 1
POS_INTERIOR, POS_LEFT, POS_RIGHT, POS_SINGLE = 0, 1, 2, 3
ALGO_AUTO, ALGO_LAYERED, ALGO_CHAIN, ALGO_BUCKETED, ALGO_GSORT = 0, 1, 2, 3, 4


class TnbNode(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("internal", c_int32), ("phys", c_int32),
                ("r_left", c_int32), ("r_right", c_int32), ("pad_", c_int32),
                ("core", c_void_p), ("factor", c_void_p)]


class TnbMode(ctypes.Structure):
    _fields_ = [("layout", c_int32), ("phys", c_int32), ("r_left", c_int32),
                ("r_right", c_int32), ("slices", c_void_p)]


class TnbChain(ctypes.Structure):
    _fields_ = [("n_modes", c_int32), ("pad_", c_int32), ("batch", c_int64),
                ("modes", POINTER(TnbMode))]


class TnbEntriesInfo(ctypes.Structure):
    _fields_ = [("algo", c_int32), ("n_virtual", c_int32), ("prefix_modes", c_int32),
                ("suffix_modes", c_int32), ("prefix_rows", c_int64), ("suffix_rows", c_int64),
                ("kernel_flops", c_double), ("table_flops", c_double), ("diag_tables", c_int32),
                ("table_launches", c_int32), ("compute_kernel", c_int32), ("tile", c_int32),
                ("tensor_flops", c_double)]


# name -> (restype, argtypes); exactly the declarations of include/tnb.h
SIGNATURES = {
    "tnb_version": (c_char_p, []),
    "tnb_last_error": (c_char_p, []),
    "tnb_device_check": (c_int, []),
    "tnb_plan_modes": (c_int, [POINTER(TnbNode), c_int32, POINTER(TnbMode)]),
    "tnb_mode_floats": (c_int64, [POINTER(TnbMode), c_int64]),
    "tnb_repack_f32": (c_int, [POINTER(TnbNode), c_int32, c_int64, POINTER(TnbMode), c_void_p]),
    "tnb_tt_core_f32": (c_int, [POINTER(TnbChain), c_int32, c_void_p, c_void_p]),
    "tnb_promote_cp_f32": (c_int, [POINTER(TnbNode), c_int32, c_int64, c_void_p, c_void_p]),
    "tnb_entries_workspace_bytes": (c_int64, [POINTER(TnbChain), c_int64, c_int32]),
    "tnb_entries_f32": (c_int, [POINTER(TnbChain), c_void_p, c_int64, c_void_p, c_void_p,
                                c_int32, c_void_p, c_int64, c_void_p]),
    "tnb_full_workspace_bytes": (c_int64, [POINTER(TnbChain), c_int64, c_int64]),
    "tnb_full_f32": (c_int, [POINTER(TnbChain), c_int64, c_int64, c_void_p, c_void_p,
                             c_int64, c_void_p]),
    "tnb_dot_f32": (c_int, [POINTER(TnbChain), POINTER(TnbChain), c_void_p, c_void_p]),
    "tnb_norm_f32": (c_int, [POINTER(TnbChain), c_void_p, c_void_p]),
    "tnb_repack_f64": (c_int, [POINTER(TnbNode), c_int32, c_int64, POINTER(TnbMode), c_void_p]),
    "tnb_tt_core_f64": (c_int, [POINTER(TnbChain), c_int32, c_void_p, c_void_p]),
    "tnb_promote_cp_f64": (c_int, [POINTER(TnbNode), c_int32, c_int64, c_void_p, c_void_p]),
    "tnb_entries_workspace_bytes_f64": (c_int64, [POINTER(TnbChain), c_int64, c_int32]),
    "tnb_entries_f64": (c_int, [POINTER(TnbChain), c_void_p, c_int64, c_void_p, c_void_p,
                                c_int32, c_void_p, c_int64, c_void_p]),
    "tnb_full_workspace_bytes_f64": (c_int64, [POINTER(TnbChain), c_int64, c_int64]),
    "tnb_full_f64": (c_int, [POINTER(TnbChain), c_int64, c_int64, c_void_p, c_void_p,
                             c_int64, c_void_p]),
    "tnb_dot_f64": (c_int, [POINTER(TnbChain), POINTER(TnbChain), c_void_p, c_void_p]),
    "tnb_norm_f64": (c_int, [POINTER(TnbChain), c_void_p, c_void_p]),
    "tnb_narrow_indices_host": (c_int, [c_void_p, c_int64, c_int32, c_void_p, c_int32, POINTER(c_int32)]),
    "tnb_widen_indices": (c_int, [c_void_p, c_int32, c_int64, c_void_p, c_void_p]),
    "tnb_host_threads": (c_int, []),
    "tnb_entries_plan": (c_int, [POINTER(TnbChain), c_int64, c_int32, POINTER(TnbEntriesInfo)]),
    "tnb_timing_enable": (c_int, [c_int32]),
    "tnb_timing_read": (c_int, [c_char_p, POINTER(c_double), POINTER(c_int64)]),
}

_lock = threading.Lock()
_lib = None
_device_ok = set()


def load() -> ctypes.CDLL:
    """Loads libtnb.so once; raises NativeError when it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_2206_11128_b200._build` (no CPU fallback exists)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def last_error() -> str:
    return load().tnb_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Maps a libtnb status to the reference's exception classes."""
    if rc == TNB_OK:
        return
    msg = last_error()
    if rc in (TNB_EINVAL, TNB_EINDEX):
        raise ContractViolationError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg} (status {rc})")


def require_device(device) -> None:
    """Fails loudly unless ``device`` is an sm_100 CUDA device."""
    import torch

    if device is None or device.type != "cuda" or not torch.cuda.is_available():
        raise NativeError("paper_2206_11128_b200 computes on a CUDA (sm_100a) device only; "
                          "no CPU fallback exists")
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx in _device_ok:
        return
    lib = load()
    with torch.cuda.device(idx):
        check(lib.tnb_device_check(), "device check")
    _device_ok.add(idx)


def stream_ptr(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def entries_plan(chain: TnbChain, m: int, algo: int = ALGO_AUTO) -> dict:
    """What tnb_entries_f32 would run for (chain, m, algo): algorithm, mode
    merging and the per-call algorithmic flops (no device work)."""
    info = TnbEntriesInfo()
    check(load().tnb_entries_plan(ctypes.byref(chain), m, algo, ctypes.byref(info)), "entries plan")
    return {f: getattr(info, f) for f, _ in TnbEntriesInfo._fields_}


def narrow_indices(src, dst, width: int, nthreads: int = 0) -> bool:
    """Host transport codec (tnb_narrow_indices_host): int64 host tensor
    ``src`` -> int8/int16 host tensor ``dst`` of the same element count.
    True when every value fit (``dst`` holds them), False otherwise.  Runs
    on host threads with the GIL released (ctypes)."""
    if src.numel() != dst.numel() or dst.element_size() != width:
        raise ContractViolationError("narrow_indices: size / width mismatch")
    fits = c_int32(0)
    check(load().tnb_narrow_indices_host(src.data_ptr(), src.numel(), width, dst.data_ptr(), nthreads,
                                         ctypes.byref(fits)), "narrow indices")
    return bool(fits.value)


def timing_enable(on: bool) -> None:
    check(load().tnb_timing_enable(1 if on else 0), "timing")


def timing_read(kernel: str) -> tuple:
    """(total milliseconds, launches) of libtnb's kernel ``kernel`` since the
    last timing_enable(True); waits for the recorded events."""
    ms, n = c_double(), c_int64()
    check(load().tnb_timing_read(kernel.encode(), ctypes.byref(ms), ctypes.byref(n)), "timing")
    return ms.value, n.value
