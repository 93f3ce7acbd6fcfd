"""What the ~7 us fixed per-launch cost of the data kernel is made of
(L2 read-flushed graph replay): an empty torch kernel, one 32-record tile
with the tree in shared memory / read through L1, and C1 with 1M records."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
import workloads  # noqa: E402

flush = workloads.make_flush()
w = bench.WORKLOADS["C1"]
tree = st.generate_synthetic_tree(*w["tree"])
x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
z = torch.empty(1, device="cuda")
rows = [("empty torch kernel", lambda: z.zero_())]
for m in (32, 4736 * 32, w["m"]):
    for tl in ("shared", "global"):
        g = st.GpuGeom(algo="data", tree_loc=tl)
        xs, os_ = x[:m], out[:m]
        rows.append((f"data m={m} tree={tl}", (lambda xs=xs, os_=os_, g=g: st.eval_device(tree, xs, os_, g))))
for name, fn in rows:
    us = workloads.graph_time(fn, 20, flush) * 1e3
    print(f"{name:40s} {us:8.2f} us", flush=True)
