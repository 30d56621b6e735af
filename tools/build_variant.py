"""Builds a variant of libtnb.so with extra preprocessor defines, for A/B
timing of kernel alternatives on the GPU box:

    python tools/build_variant.py NAME -DTNB_STREAM_RS=0 ...
    TNB_LIB=build/variants/NAME/libtnb.so python tools/bench_entries.py --one cfg5
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2206_11128_b200 import _build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = ROOT / "build" / "variants" / name
    out.mkdir(parents=True, exist_ok=True)

    def comp(src):
        obj = out / (src.stem + (".o" if src.suffix == ".cu" else ".cpp.o"))
        if src.suffix == ".cpp":
            cmd = [B.CXX, *B.CXXFLAGS, *defs, "-I", str(B.INCLUDE), "-c", str(src), "-o", str(obj)]
        else:
            cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-I", str(B.INCLUDE), "-I", str(B.CSRC), "-c", str(src), "-o",
                   str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, B._sources()))
    lib = out / "libtnb.so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart=static", "-Xcompiler", "-pthread", "-o", str(lib),
                    *map(str, objs)], check=True)
    print(lib)


if __name__ == "__main__":
    main()
