"""Run one canonical workload a few times (target for ncu -k regex:... -s N -c 1).

    python tools/prof_one.py C1 data [reps] ['dict(variant=("spec_pred",))'] [--tile=N]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

tile = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--tile=")), 1))
argv = [a for a in sys.argv if not a.startswith("--tile=")]
name, algo = argv[1], argv[2]
reps = int(argv[3]) if len(argv) > 3 else 4
w = bench.WORKLOADS[name]
tree = st.generate_synthetic_tree(*w["tree"])
x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda().repeat(tile, 1)
out = torch.empty(w["m"] * tile, dtype=torch.int32, device="cuda")
g = st.GpuGeom(algo=algo, **(eval(argv[4]) if len(argv) > 4 else {}))
for _ in range(reps):
    st.eval_device(tree, x, out, g)
torch.cuda.synchronize()
ok = st.fnv1a64(out[: w["m"]].cpu().numpy()) == bench.golden_labels(w, 0)
print(name, algo, "labels_ok", ok)
