"""Build libsylvsketch.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsylvsketch.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("engine.cu", "host_solve.cpp")]
HEADERS = sorted(os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
                 if f.endswith((".cuh", ".hpp", ".h")))
HEADERS.append(os.path.join(ROOT, "include", "sylv_sketch.h"))
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.isabs(p) and os.path.exists(p) or not os.path.isabs(p)):
            return p
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False, out: str = None, extra=()) -> str:
    """Build the library (out / extra nvcc flags: development A/B variants, e.g.
    build(out="build_ab/libsylvsketch_ns2.so", extra=["-DSYLV_ST25_NS8=2"]))."""
    lib = os.path.abspath(out) if out else LIB
    if not force and not out and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(os.path.abspath(lib)), exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-shared", "-cudart", "static", "-o", tmp, *SOURCES, "-ldl",
           "-L/usr/local/cuda/lib64", "-lcublas", "-lcusolver", "-lcufft", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
