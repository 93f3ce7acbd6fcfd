"""A/B of the spec-ring slot-generation handshake on one box (development aid):
alternates ST_SPEC_RING_UNSAFE_NO_GEN=0/1 on C2 and prints CUDA-event times."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
tree = st.generate_synthetic_tree(*w["tree"])
x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
res = {}
for rep in range(3):
    for flag in ("0", "1"):
        os.environ["ST_SPEC_RING_UNSAFE_NO_GEN"] = flag
        for G in (2, 4):
            g = st.GpuGeom(algo="speculative", group_lanes=G)
            for _ in range(3):
                st.eval_device(tree, x, out, g)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                st.eval_device(tree, x, out, g)
            b.record()
            torch.cuda.synchronize()
            res.setdefault((flag, G), []).append(round(a.elapsed_time(b) / 20, 4))
for k, v in sorted(res.items()):
    print("no_gen" if k[0] == "1" else "gen   ", "G", k[1], v)
