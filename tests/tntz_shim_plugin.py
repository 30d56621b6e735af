"""pytest plugin (``-p tntz_shim_plugin``): before the reference's own test
modules import tntz, re-point its hot path at the GPU
(paper_2206_11128_b200.tntz_shim) and count the calls that went there."""

import collections

CALLS = collections.Counter()


def pytest_configure(config):
    import torch
    import tntz

    from paper_2206_11128_b200 import tntz_shim

    dtype = torch.float32 if config.getoption("--shim-f32", False) else torch.float64
    tntz_shim.install(tntz, dtype=dtype)
    for mod in {tntz.core, tntz, tntz.arithmetic, tntz.indexing}:
        for name in ("full", "entries", "chain_dot", "norm"):
            fn = getattr(mod, name, None)
            if fn is not None and getattr(fn, "__module__", "") == "paper_2206_11128_b200.tntz_shim":
                setattr(mod, name, _counted(name, fn))
    print(f"tntz shim installed: {tntz.__file__} -> GPU ({dtype})")


def pytest_addoption(parser):
    parser.addoption("--shim-f32", action="store_true", default=False)


def _counted(name, fn):
    def call(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)

    call.__wrapped__ = fn
    return call


def pytest_unconfigure(config):
    print("tntz shim calls: " + " ".join(f"{k}={v}" for k, v in sorted(CALLS.items())))
