"""In-tree build of the CUDA library (sm_100a) — ``libfsk_b200.so``.

nvcc cross-compiles without a GPU, so this runs in the CPU container as the
driver's "does it build" check and the resulting ``.so`` travels to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfsk_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O2", "-I", INCLUDE, "-I", CSRC]
# extra -D flags for tuning sweeps (e.g. FSK_NVCC_DEFS="-DFSK_SEARCH_MINB=2")
NVCC_FLAGS += os.environ.get("FSK_NVCC_DEFS", "").split()

LIBS = ["-lcudart", "-lnccl"]
CU_SOURCES = ["fsk_ctx.cu", "fsk_search.cu", "fsk_bwd.cu", "fsk_mlp.cu", "fsk_multi.cu"]
CXX_SOURCES = ["fskin_api.cpp", "fsk_io.cpp"]


def _sources():
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES + CXX_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    deps += [os.path.join(INCLUDE, "fsk.h")]
    inc = os.path.join(INCLUDE, "fskin")
    if os.path.isdir(inc):
        deps += [os.path.join(inc, f) for f in os.listdir(inc)]
    return srcs, deps


def build(force: bool = False, verbose: bool = False) -> str:
    srcs, deps = _sources()
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB
    cmd = ["nvcc", *NVCC_FLAGS, "-shared", "-o", LIB, *srcs, *LIBS]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
