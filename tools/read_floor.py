"""Practical floors for small single launches (C1, C3): the same record
buffer read by torch's sum reduction (a streaming read with no tree work),
our data kernel on a one-node-deep tree (staging + streaming + label store,
almost no walk), and the real workload -- every launch L2-flushed, timed by
CUDA-graph replay (tools/workloads.py graph_time).

    python tools/read_floor.py [--iters 50]  -> gpurun_out/read_floor.json
"""
import argparse
import json
import os
import sys

import ctypes as C

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    flush = wl.make_flush()
    rk = C.CDLL(os.path.join(ROOT, "tools", "micro", "libreadk.so"))  # tools/micro/read_kernel.cu
    rk.read_floor.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    res = {}
    for name in ("C1", "C3"):
        w = bench.WORKLOADS[name]
        x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
        out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
        acc = torch.empty(w["a"], dtype=torch.float32, device="cuda")
        tree = st.generate_synthetic_tree(*w["tree"])
        stump = st.generate_synthetic_tree(1, 2, w["a"], 2, 7)
        def rfl(mode, bps):
            return lambda: rk.read_floor(x.data_ptr(), x.numel() * 4, out.data_ptr(), mode, bps,
                                         torch.cuda.current_stream().cuda_stream)
        rows = {
            "read_v4_4b": rfl(0, 4),
            "read_v4_2b": rfl(0, 2),
            "read_v4_8b": rfl(0, 8),
            "read_label_4b": rfl(1, 4),
            "read_v4_labels_4b": rfl(2, 4),
            "data_stump": lambda: st.eval_device(stump, x, out, st.GpuGeom(algo="data")),
            "data": lambda: st.eval_device(tree, x, out, st.GpuGeom(algo="data")),
            "speculative": lambda: st.eval_device(tree, x, out, st.GpuGeom(algo="speculative")),
        }
        res[name] = {"bytes": int(x.numel() * 4)}
        for k, fn in rows.items():
            ms = wl.graph_time(fn, args.iters, flush)
            res[name][k] = {"us": round(ms * 1e3, 2), "GBs": round(x.numel() * 4 / (ms * 1e-3) / 1e9, 1)}
            print(name, k, res[name][k], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "read_floor.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
