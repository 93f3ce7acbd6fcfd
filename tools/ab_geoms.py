"""A/B kernel geometries / variants on canonical workloads (development aid):
    python tools/ab_geoms.py W1,W2 'dict(record_regs=3, samples_per_thread=2, stages=1)' ... \
        [--algo=data|speculative] [--flush] [--tile=N]
    e.g. ... C2 'dict(variant=("spec_wide",))' 'dict(slot_records=1)' --algo=speculative
W may be PAPER: the paper's tree(11,16,19,7,1) on 256 copies of its
data(16384,19,2) (16.8M records).  Every st_geom field (including the
ST_VAR_* variants) is reachable per call.  Alternates the geometries for 5
rounds on one box; prints per-geometry us."""
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
tile = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--tile=")), 1))
algo = next((a.split("=")[1] for a in sys.argv if a.startswith("--algo=")), "data")
args = [a for a in sys.argv[1:] if a != "--flush" and not a.startswith("--tile=") and not a.startswith("--algo=")]
names, specs = args[0].split(","), ["dict()"] + args[1:]
fl = workloads.make_flush() if flush else None
for name in names:
    if name == "PAPER":
        import numpy as np
        tree = st.generate_synthetic_tree(11, 16, 19, 7, 1)
        x = np.tile(st.generate_synthetic_dataset(16384, 19, 2), (256, 1))
        w = {"m": len(x), "labels_fnv": st.fnv1a64(st.eval_gpu(tree, x, st.GpuGeom(algo="data")))}
    else:
        w = bench.WORKLOADS[name]
        tree = st.generate_synthetic_tree(*w["tree"])
        x = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
    xd = torch.from_numpy(x).cuda().repeat(tile, 1)
    out = torch.empty(len(xd), dtype=torch.int32, device="cuda")
    geoms = [st.GpuGeom(algo=algo, **eval(s)) for s in specs]
    res = {s: [] for s in specs}
    for g, s in zip(geoms, specs):
        st.eval_device(tree, xd, out, g)
        torch.cuda.synchronize()
        want = w["labels_fnv"] if name == "PAPER" else bench.golden_labels(w, 0)
        assert want is None or st.fnv1a64(out[: w["m"]].cpu().numpy()) == want, (name, s)
        if tile > 1:
            assert torch.equal(out.view(tile, -1), out[: w["m"]].expand(tile, -1)), (name, s)
    for _ in range(5):
        for g, s in zip(geoms, specs):
            res[s].append(round(workloads.graph_time(lambda: st.eval_device(tree, xd, out, g), 20, fl) * 1e3, 2))
    print(name, f"x{tile}", {s: (min(v), sorted(v)[2]) for s, v in res.items()}, "us (min, median)", flush=True)
