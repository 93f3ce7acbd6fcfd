"""Quick GPU probe: parity of every kernel on the canonical configs vs the C
oracle, plus CUDA-event timings.  Development aid (not the bench contract).

    python tools/gpu_probe.py [--configs C1,C2,...] [--iters 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
from support import APPENDIX_A, workload  # noqa: E402


def time_kernel(fn, iters, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="paper,C1,C2,C3")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--geoms", default="")
    args = ap.parse_args()
    co = oracle.COracle()
    peak = 6455.6
    res = []
    for name in args.configs.split(","):
        t0 = time.time()
        nodes, x = workload(co, name)
        want = co.eval_serial(nodes, x)
        gen_s = time.time() - t0
        tree = st.EncodedTree(nodes)
        xd = torch.from_numpy(x).cuda()
        m, a = x.shape
        out = torch.empty(m, dtype=torch.int32, device="cuda")
        geoms = [("data", st.GpuGeom(algo="data")),
                 ("data-S1", st.GpuGeom(algo="data", samples_per_thread=1)),
                 ("data-global", st.GpuGeom(algo="data", tree_loc="global")),
                 ("data-const", st.GpuGeom(algo="data", tree_loc="constant")),
                 ("spec", st.GpuGeom(algo="speculative")),
                 ("spec-G8", st.GpuGeom(algo="speculative", group_lanes=8)),
                 ("spec-G32", st.GpuGeom(algo="speculative", group_lanes=32)),
                 ("spec-G4", st.GpuGeom(algo="speculative", group_lanes=4))]
        for gname, g in geoms:
            out.zero_()
            try:
                st.eval_device(tree, xd, out, g)
                torch.cuda.synchronize()
            except Exception as ex:  # report and continue
                res.append({"config": name, "geom": gname, "error": str(ex)})
                print(res[-1], flush=True)
                continue
            got = out.cpu().numpy().view(np.uint32)
            mism = int((got != want).sum())
            ms = time_kernel(lambda: st.eval_device(tree, xd, out, g), args.iters)
            gbs = m * a * 4 / (ms * 1e-3) / 1e9
            r = {"config": name, "geom": gname, "mismatches": mism, "ms": round(ms, 4),
                 "Gsamples_s": round(m / (ms * 1e-3) / 1e9, 3), "GBs": round(gbs, 1),
                 "frac_measured": round(gbs / peak, 3), "gen_s": round(gen_s, 1)}
            res.append(r)
            print(json.dumps(r), flush=True)
        del xd, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "probe.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
