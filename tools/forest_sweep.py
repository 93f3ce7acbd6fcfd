"""C4 forest geometry sweep (development aid): U trees per lane step, tree-ring
depth NT, CTA width W via st_geom (forest_chains, forest_slots,
warps_per_cta); CUDA-event timing, vote hash checked against Appendix A.

    python tools/forest_sweep.py [records]
"""
import itertools
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_1373_b200 as st  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
trees = [st.generate_synthetic_tree(12, 1024, 64, 8, 401 + t) for t in range(128)]
x = torch.from_numpy(st.generate_synthetic_dataset(m, 64, 499)).cuda()
f = st.Forest(trees, 8)
lab = torch.empty(m, dtype=torch.int32, device="cuda")
res = []
grid = [(0, 0, 0)] + [(u, u + k, w) for u, k, w in itertools.product([1, 2, 4], [1, 2, 3], [0, 17, 25])]
if len(sys.argv) > 2 and sys.argv[2] == "deep":  # deeper rings at fewer consumer warps
    grid = [(0, 0, 0)] + [(u, nt, 0) for u in (1, 2, 3, 4) for nt in range(u + 1, 11)]
if len(sys.argv) > 2 and sys.argv[2] == "fine":  # around the folded-tree optimum
    grid = [(0, 0, 0)] + [(u, nt, w) for u in (2, 3, 4) for nt in range(u + 2, u + 5) for w in (0, 24, 20, 16)]
for u, nt, w in grid:
    env = {"forest_chains": u, "forest_slots": nt, "warps_per_cta": w}
    geom = st.GpuGeom(**env)
    try:
        st.eval_forest_device(f, x, lab, geom)
        torch.cuda.synchronize()
    except Exception as e:  # geometry does not fit
        print("skip", env, e, flush=True)
        continue
    ok = m != 8_000_000 or st.fnv1a64(lab.cpu().numpy()) == 0x1b2543c41e436ce0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        st.eval_forest_device(f, x, lab, geom)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    r = dict(env, ms=round(ms, 3), ok=bool(ok))
    res.append(r)
    print(json.dumps(r), flush=True)
res.sort(key=lambda r: r["ms"])
print("BEST", json.dumps(res[:5]))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "forest_sweep.json"), "w"), indent=0)
