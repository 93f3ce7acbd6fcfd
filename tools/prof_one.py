"""Run one canonical workload a few times (target for ncu -k regex:... -s N -c 1).

    python tools/prof_one.py C1 data [reps] ['dict(variant=("spec_pred",))']
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

name, algo = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
w = bench.WORKLOADS[name]
tree = st.generate_synthetic_tree(*w["tree"])
x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
g = st.GpuGeom(algo=algo, **(eval(sys.argv[4]) if len(sys.argv) > 4 else {}))
for _ in range(reps):
    st.eval_device(tree, x, out, g)
torch.cuda.synchronize()
ok = st.fnv1a64(out.cpu().numpy()) == bench.golden_labels(w, 0)
print(name, algo, "labels_ok", ok)
