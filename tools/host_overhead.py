"""Host time per eval_device call (plan + launch) vs the kernel's device time,
for each canonical tree (development aid): a launch-bound stream of launches
shows up as host time >= device time.

    python tools/host_overhead.py [W ...]
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

for name in sys.argv[1:] or ["C2", "C1", "C5d12"]:
    w = bench.WORKLOADS[name]
    tree = st.generate_synthetic_tree(*w["tree"])
    x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
    out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
    for algo in ("data", "speculative"):
        g = st.GpuGeom(algo=algo)
        for _ in range(5):
            st.eval_device(tree, x, out, g)
        torch.cuda.synchronize()
        n = 50
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        for _ in range(n):
            st.eval_device(tree, x, out, g)
        b.record()
        t_host = (time.perf_counter() - t0) / n
        torch.cuda.synchronize()
        t_dev = a.elapsed_time(b) / n * 1e-3
        print(f"{name:6s} {algo:12s} host {t_host * 1e6:8.1f} us/call   device {t_dev * 1e6:8.1f} us/launch", flush=True)
