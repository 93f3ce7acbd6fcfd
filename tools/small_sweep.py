"""Geometry sweep of the data kernel on a small single launch (C1 / C3
shapes), with the real tree and with a one-split stump (pipeline floor),
L2-flushed graph replay.  python tools/small_sweep.py [C1|C3]"""
import itertools
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
import workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
w = bench.WORKLOADS[name]
x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
trees = {"real": st.generate_synthetic_tree(*w["tree"]), "stump": st.generate_synthetic_tree(1, 2, w["a"], 2, 7)}
flush = wl.make_flush()
res = []
grid = [dict()]
for ns, (wp, bps), spt in itertools.product((1, 2, 3, 4), ((8, 4), (16, 2), (32, 1), (4, 8), (8, 2), (16, 1)), (1, 2)):
    grid.append(dict(stages=ns, warps_per_cta=wp, blocks_per_sm=bps, samples_per_thread=spt))
for tn, tree in trees.items():
    for gd in grid:
        try:
            g = st.GpuGeom(algo="data", **gd)
            st.eval_device(tree, x, out, g)
            torch.cuda.synchronize()
            us = wl.graph_time(lambda: st.eval_device(tree, x, out, g), 30, flush) * 1e3
        except Exception as e:  # geometry does not fit
            us = None
        res.append({"tree": tn, "geom": gd, "us": None if us is None else round(us, 2)})
        print(tn, gd, res[-1]["us"], flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", f"small_sweep_{name}.json"), "w"), indent=1)
best = {}
for r in res:
    if r["us"] is not None and (r["tree"] not in best or r["us"] < best[r["tree"]]["us"]):
        best[r["tree"]] = r
print("best", json.dumps(best))
