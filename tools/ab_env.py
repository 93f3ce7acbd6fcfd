"""A/B an environment knob on one box (development aid):
    python tools/ab_env.py VAR "v0,v1" W1 [W2 ...] [--tile N]  -> data-kernel CUDA-event ms"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

var, vals = sys.argv[1], sys.argv[2].split(",")
tile = 1
flush = False
names = []
for a in sys.argv[3:]:
    if a.startswith("--tile="):
        tile = int(a.split("=")[1])
    elif a == "--flush":
        flush = True
    else:
        names.append(a)
if flush:
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import workloads  # noqa: E402
    fl = workloads.make_flush()
for name in names:
    w = bench.WORKLOADS[name]
    tree = st.generate_synthetic_tree(*w["tree"])
    x = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
    if tile > 1:
        x = np.tile(x, (tile, 1))
    xd = torch.from_numpy(x).cuda()
    out = torch.empty(len(x), dtype=torch.int32, device="cuda")
    g = st.GpuGeom(algo="data")
    res = {v: [] for v in vals}
    for rep in range(3):
        for v in vals:
            os.environ[var] = v
            if flush:  # L2 read-flushed graph replay (tools/workloads.py)
                res[v].append(round(workloads.graph_time(lambda: st.eval_device(tree, xd, out, g), 20, fl), 5))
                continue
            for _ in range(3):
                st.eval_device(tree, xd, out, g)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                st.eval_device(tree, xd, out, g)
            b.record()
            torch.cuda.synchronize()
            res[v].append(round(a.elapsed_time(b) / 20, 4))
    print(name, f"x{tile}", {f"{var}={v}": t for v, t in res.items()}, flush=True)
