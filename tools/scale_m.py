"""Kernel time vs record count for one workload (L2 read-flushed graph replay):
fits t = a + b*m to split fixed launch/ramp/tail cost from the streaming rate.

    python tools/scale_m.py C1 [algo]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
import workloads  # noqa: E402

name = sys.argv[1]
algo = sys.argv[2] if len(sys.argv) > 2 else "data"
w = bench.WORKLOADS[name]
tree = st.generate_synthetic_tree(*w["tree"])
xs = st.generate_synthetic_dataset(8 * w["m"], w["a"], w["seed"])
flush = workloads.make_flush()
rows = []
for f in (0.125, 0.25, 0.5, 1, 2, 4, 8):
    m = int(f * w["m"]) // 128 * 128
    xd = torch.from_numpy(xs[:m]).cuda()
    out = torch.empty(m, dtype=torch.int32, device="cuda")
    g = st.GpuGeom(algo=algo)
    ms = workloads.graph_time(lambda: st.eval_device(tree, xd, out, g), 20, flush)
    rows.append((m, ms))
    print(m, round(ms * 1e3, 2), "us", flush=True)
m = np.array([r[0] for r in rows], float)
t = np.array([r[1] for r in rows], float) * 1e3
b, a = np.polyfit(m, t, 1)
print(json.dumps({"workload": name, "algo": algo, "fixed_us": round(a, 2),
                  "per_Mrecord_us": round(b * 1e6, 3),
                  "streaming_GBs": round(4 * w["a"] / (b * 1e-6) / 1e9, 1)}))
