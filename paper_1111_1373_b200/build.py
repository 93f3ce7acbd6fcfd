"""Build the sm_100a CUDA library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_1111_1373_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo (ncu source
view), no --use_fast_math and no -ftz=true (bit-exact IEEE compares).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "csrc", "st_capi.cu"), os.path.join(HERE, "csrc", "st_io.cu"),
        os.path.join(HERE, "csrc", "st_synth.cpp")]
DEPS = [*SRCS, os.path.join(HERE, "csrc", "st_kernels.cuh"),
        os.path.join(ROOT, "include", "spectree_b200.h")]
OUT = os.path.join(HERE, "libspectree_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-ftz=false", "-prec-div=true", "-fmad=true",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or not up_to_date():
        cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp", *SRCS]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
