"""A/B an environment knob for the speculative kernel on one box (development aid):
    python tools/ab_spec_env.py VAR "v0,v1" W1 [W2 ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

var, vals = sys.argv[1], sys.argv[2].split(",")
for name in sys.argv[3:]:
    w = bench.WORKLOADS[name]
    tree = st.generate_synthetic_tree(*w["tree"])
    x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
    out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
    for G in (2, 4):
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
