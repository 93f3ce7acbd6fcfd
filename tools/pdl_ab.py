"""Back-to-back launches on distinct record buffers (a frame stream larger
than L2), captured in one CUDA graph, with and without programmatic dependent
launch (st_geom.pdl): per-launch device time (development aid).
    python tools/pdl_ab.py [W ...] [--frames=16] [--algo=data]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

frames = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--frames=")), 16))
algo = next((a.split("=")[1] for a in sys.argv if a.startswith("--algo=")), "data")
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C3"]
for name in names:
    w = bench.WORKLOADS[name]
    tree = st.generate_synthetic_tree(*w["tree"])
    x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
    xs = [x.clone() for _ in range(frames)]
    outs = [torch.empty(w["m"], dtype=torch.int32, device="cuda") for _ in range(frames)]
    res = {}
    for pdl in ("off", "1", "2", "auto", "off", "1", "2", "auto"):
        g = st.GpuGeom(algo=algo, pdl={"off": 3, "1": 1, "2": 2, "auto": 0}[pdl])
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for xi, oi in zip(xs, outs):
                st.eval_device(tree, xi, oi, g)
        torch.cuda.synchronize()
        for oi in outs:
            assert st.fnv1a64(oi.cpu().numpy()) == w["labels_fnv"], (name, pdl)
            oi.zero_()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for xi, oi in zip(xs, outs):
                st.eval_device(tree, xi, oi, g)
        graph.replay()
        torch.cuda.synchronize()
        for oi in outs:
            assert st.fnv1a64(oi.cpu().numpy()) == w["labels_fnv"], (name, pdl, "graph")
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graph.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / frames)
        res.setdefault(f"pdl={pdl}", []).append(round(best, 2))
    print(name, algo, f"{frames} launches on distinct buffers, us per launch (best of 5 replays):", res, flush=True)
