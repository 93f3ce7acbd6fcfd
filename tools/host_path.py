"""Host-buffer path throughput (the reference-facing call a user makes with
host arrays): st_eval on C2 from pageable (numpy) and pinned (torch) records,
and st_eval_timed's phases (pageable).  Labels checked against
the workload hash.  ST_HOST_COPY_THREADS sets the packing threads for
pageable inputs (read once per process).

    python tools/host_path.py [--reps 5]  -> one JSON line
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
from paper_1111_1373_b200 import bench_flow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--workload", default="C2")
args = ap.parse_args()
w = bench.WORKLOADS[args.workload]
tree = st.generate_synthetic_tree(*w["tree"])
x = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
m, a = x.shape
gb = x.nbytes / 1e9
res = {"workload": args.workload, "records": m, "bytes": x.nbytes,
       "copy_threads": os.environ.get("ST_HOST_COPY_THREADS", "default"), "cpus": os.cpu_count()}


def timed(fn):
    fn()
    ts = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    assert st.fnv1a64(out) == w["labels_fnv"]
    return min(ts)


out = np.empty(m, np.uint32)
t = timed(lambda: st.eval_gpu(tree, x, out=out))
res["pageable_aos"] = {"s": t, "GBs": gb / t, "Msamples_s": m / t / 1e6}
xp = torch.from_numpy(x).pin_memory().numpy()
outp = torch.empty(m, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
t = timed(lambda: st.eval_gpu(tree, xp, out=outp))
res["pinned_aos"] = {"s": t, "GBs": gb / t, "Msamples_s": m / t / 1e6}
del xp
ph = []
for _ in range(args.reps + 1):
    lab, tm = bench_flow.eval_timed(tree, x)
    ph.append(tm)
assert st.fnv1a64(lab) == w["labels_fnv"]
best = min(ph[1:], key=lambda d: d["outer_us"])
best["h2d_GBs"] = x.nbytes / best["h2d_us"] / 1e3
res["eval_timed_pageable"] = best
print(json.dumps(res), flush=True)
