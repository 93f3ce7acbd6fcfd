"""Geometry sweep on one workload (development aid): CUDA-event timing of
every (algo, geometry) on device-resident records."""
import argparse, json, os, sys, itertools
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_1373_b200 as st
import bench
sys.path.insert(0, os.path.join(ROOT, "tools"))

def timeit(fn, iters=30, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--grid", default="data")
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--tile", type=int, default=1, help="repeat the records N times (L2-sized configs)")
ap.add_argument("--flush", action="store_true",
                help="L2 read-flush before every launch, graph-replay timing (tools/workloads.py)")
args = ap.parse_args()
W = bench.WORKLOADS[args.workload]
m, a = W["m"], W["a"]
tree = st.generate_synthetic_tree(*W["tree"])
x = st.generate_synthetic_dataset(m, a, W["seed"])
if args.tile > 1:
    import numpy as np
    x = np.tile(x, (args.tile, 1))
    m = len(x)
xd = torch.from_numpy(x).cuda(); out = torch.empty(m, dtype=torch.int32, device="cuda")
peak, _ = bench.peaks()
geoms = []
if "data" in args.grid:
    for tl, S, ns, bps, w in itertools.product(["shared", "global"], [1, 2, 4], [2, 3], [0, 2], [0, 8, 16, 32]):
        geoms.append(st.GpuGeom(algo="data", tree_loc=tl, samples_per_thread=S, stages=ns, blocks_per_sm=bps,
                                warps_per_cta=w))
if "spec" in args.grid and "spec2" not in args.grid:
    for G, pl in itertools.product([2, 4, 8, 16], [1, 2]):
        geoms.append(st.GpuGeom(algo="speculative", group_lanes=G, pipeline=pl))
if "spec2" in args.grid:
    for G, sr in itertools.product([2, 4, 8], [1, 2]):
        geoms.append(st.GpuGeom(algo="speculative", group_lanes=G, samples_per_thread=sr))
if "regs1" in args.grid:
    for S, ns, w in itertools.product([1, 2, 4], [1, 2], [0, 32]):
        geoms.append(st.GpuGeom(algo="data", samples_per_thread=S, record_regs=1, stages=ns, warps_per_cta=w))
if "regs0" in args.grid:
    for S in [0, 1, 2]:
        geoms.append(st.GpuGeom(algo="data", samples_per_thread=S, record_regs=2))
if "regs" in args.grid and "regs1" not in args.grid and "regs0" not in args.grid:
    for S, rr, w in itertools.product([0, 1, 2, 4], [1, 2], [0, 16]):
        geoms.append(st.GpuGeom(algo="data", samples_per_thread=S, record_regs=rr, warps_per_cta=w))
if "small" in args.grid:
    for S, ns, w, bps in itertools.product([0, 1, 2, 4], [0, 3], [0, 8, 16], [0, 1, 2, 4]):
        geoms.append(st.GpuGeom(algo="data", samples_per_thread=S, stages=ns, warps_per_cta=w,
                                blocks_per_sm=bps))
if "trans" in args.grid:  # transposed (attribute-major) tiles vs the defaults
    geoms.append(st.GpuGeom(algo="data"))
    for S, ns, w, bps in itertools.product([1, 2, 4], [1, 2], [0, 8], [0, 4]):
        geoms.append(st.GpuGeom(algo="data", samples_per_thread=S, record_regs=3, stages=ns,
                                warps_per_cta=w, blocks_per_sm=bps))
if "stages" in args.grid:
    for S, ns, w in itertools.product([0, 1, 2, 4], [2, 3, 4], [0, 16, 24]):
        geoms.append(st.GpuGeom(algo="data", samples_per_thread=S, stages=ns, warps_per_cta=w))
if "warps" in args.grid:
    for tl, S, w in itertools.product(["shared"], [0, 1, 2, 4], [0, 8, 16, 32]):
        geoms.append(st.GpuGeom(algo="data", tree_loc=tl, samples_per_thread=S, warps_per_cta=w))
res = []
want = None
for g in geoms:
    try:
        st.eval_device(tree, xd, out, g); torch.cuda.synchronize()
        got = st.fnv1a64(out.cpu().numpy())
        ok = got == W["labels_fnv"] if args.tile == 1 else None
        if args.flush:
            import workloads
            fl = getattr(workloads, "_sweep_flush", None) or workloads.make_flush()
            workloads._sweep_flush = fl
            ms = workloads.graph_time(lambda: st.eval_device(tree, xd, out, g), args.iters, fl)
        else:
            ms = timeit(lambda: st.eval_device(tree, xd, out, g), args.iters)
    except Exception as e:
        print("ERR", g, e, flush=True)
        import paper_1111_1373_b200._lib as L
        continue
    r = dict(g.__dict__, ok=ok, ms=round(ms, 4), frac=round(4 * a * m / (ms * 1e-3) / 1e9 / peak, 3))
    res.append(r); print(json.dumps(r), flush=True)
res.sort(key=lambda r: r["ms"])
print("BEST", json.dumps(res[:5], indent=0))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", f"sweep_{args.workload}x{args.tile}_{args.grid}{'_flush' if args.flush else ''}.json"), "w"), indent=0)
