"""A/B an environment knob for the speculative kernel on one box (development aid):
    python tools/ab_spec_env.py VAR "v0,v1" W1 [W2 ...] [--G=0,2,4]

W may be PAPER: the paper's tree(11,16,19,7,1) on 256 copies of its
data(16384,19,2) (16.8M records).  G=0 is the default geometry."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

var, vals = sys.argv[1], sys.argv[2].split(",")
Gs = [2, 4]
names = []
for arg in sys.argv[3:]:
    if arg.startswith("--G="):
        Gs = [int(v) for v in arg[4:].split(",")]
    else:
        names.append(arg)
for name in names:
    if name == "PAPER":
        tree = st.generate_synthetic_tree(11, 16, 19, 7, 1)
        xh = np.tile(st.generate_synthetic_dataset(16384, 19, 2), (256, 1))
        w = {"m": len(xh), "labels_fnv": st.fnv1a64(st.eval_gpu(tree, xh, st.GpuGeom(algo="data")))}
    else:
        w = bench.WORKLOADS[name]
        tree = st.generate_synthetic_tree(*w["tree"])
        xh = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
    x = torch.from_numpy(xh).cuda()
    out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
    for G in Gs:
        g = st.GpuGeom(algo="speculative", group_lanes=G)
        res = {v: [] for v in vals}
        for rep in range(3):
            for v in vals:
                os.environ[var] = v
                for _ in range(3):
                    st.eval_device(tree, x, out, g)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    st.eval_device(tree, x, out, g)
                b.record()
                torch.cuda.synchronize()
                res[v].append(round(a.elapsed_time(b) / 20, 4))
                ok = st.fnv1a64(out.cpu().numpy()) == w["labels_fnv"]
                assert ok, (name, G, var, v)
        print(name, f"G{G}", {f"{var}={v}": t for v, t in res.items()}, flush=True)
