"""Build the sm_100a CUDA library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_1111_1373_b200.build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo (ncu source
view), no --use_fast_math and no -ftz=true (bit-exact IEEE compares).  The
translation units (one kernel family each) compile in parallel into
build/obj/ and link into paper_1111_1373_b200/libspectree_b200.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRCS = [os.path.join(CSRC, f) for f in
        ("st_capi.cu", "st_data.cu", "st_spec.cu", "st_forest.cu", "st_frames.cu", "st_io.cu", "st_synth.cpp")]
HEADERS = [os.path.join(CSRC, "st_kernels.cuh"), os.path.join(CSRC, "st_internal.cuh"),
           os.path.join(ROOT, "include", "spectree_b200.h")]
OUT = os.path.join(HERE, "libspectree_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-ftz=false", "-prec-div=true", "-fmad=true",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.basename(src) + ".o")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def up_to_date() -> bool:
    return not _stale(OUT, SRCS + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = _obj(src)
        if force or _stale(obj, [src] + HEADERS):
            cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj + ".tmp", src]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            os.replace(obj + ".tmp", obj)
        return obj

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(SRCS), os.cpu_count() or 1))) as pool:
        objs = list(pool.map(compile_one, SRCS))
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
