"""A/B data-kernel geometries on canonical workloads (development aid):
    python tools/ab_geoms.py W1,W2 'dict(record_regs=3, samples_per_thread=2, stages=1)' ... [--flush]
Alternates the geometries for 5 rounds on one box; prints per-geometry ms."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
import workloads  # noqa: E402

flush = "--flush" in sys.argv
args = [a for a in sys.argv[1:] if a != "--flush"]
names, specs = args[0].split(","), ["dict()"] + args[1:]
fl = workloads.make_flush() if flush else None
for name in names:
    w = bench.WORKLOADS[name]
    tree = st.generate_synthetic_tree(*w["tree"])
    xd = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
    out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
    geoms = [st.GpuGeom(algo="data", **eval(s)) for s in specs]
    res = {s: [] for s in specs}
    for g, s in zip(geoms, specs):
        st.eval_device(tree, xd, out, g)
        torch.cuda.synchronize()
        assert st.fnv1a64(out.cpu().numpy()) == w["labels_fnv"], (name, s)
    for _ in range(5):
        for g, s in zip(geoms, specs):
            res[s].append(round(workloads.graph_time(lambda: st.eval_device(tree, xd, out, g), 20, fl) * 1e3, 2))
    print(name, {s: (min(v), sorted(v)[2]) for s, v in res.items()}, "us (min, median)", flush=True)
