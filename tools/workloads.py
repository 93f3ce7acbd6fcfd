"""Measure every canonical configuration on one B200:
C1, C2, C3 (frames/s), C4 (128-tree forest), C5 depth sweep 8..20 with the
speculative / data ratio per depth.  CUDA-event timing of device-resident
records; L2 is flushed before every timed launch for the configs whose inputs
fit in L2: --flush read (default) reads a 256 MB buffer, leaving L2 full of
clean lines; --flush write zeroes it, which leaves ~126 MB of dirty lines whose
write-back then competes with the timed kernel's reads (reported for
comparison).  Writes gpurun_out/workloads.json.

    python tools/workloads.py [--only C1,C5] [--iters 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

PEAK, _ = bench.peaks()
L2 = 126 * 2**20


def timed(fn, iters, flush=None):
    """Average device time of fn over iters launches (events around each
    launch; optional L2 flush between launches, outside the events)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    evs = []
    for _ in range(iters):
        if flush is not None:
            flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    for a, b in evs:
        tot += a.elapsed_time(b)
    return tot / iters


def graph_time(fn, iters, flush=None):
    """Per-launch device time from CUDA-graph replay (no host launch overhead
    inside the timed region): graph(iters x [flush, fn]) minus graph(iters x
    [flush])."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g1, g0 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1):
        for _ in range(iters):
            if flush is not None:
                flush()
            fn()
    with torch.cuda.graph(g0):
        for _ in range(iters):
            if flush is not None:
                flush()
    def t(g):
        g.replay()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)
    return max(0.0, (t(g1) - t(g0)) / iters)


FLUSH_MODE = "read"


def make_flush():
    buf = torch.ones(2 * L2 // 4, dtype=torch.float32, device="cuda")
    acc = torch.empty((), dtype=torch.float32, device="cuda")
    if FLUSH_MODE == "write":
        return lambda: buf.zero_()
    return lambda: torch.sum(buf, dim=0, out=acc)


def run_tree(name, tree, x, labels_fnv, geoms, iters, unit_div=1.0, unit="samples/s"):
    m, a = x.shape
    xd = torch.from_numpy(x).cuda()
    out = torch.empty(m, dtype=torch.int32, device="cuda")
    flush = make_flush() if 4 * a * m < 2 * L2 else None
    res = {}
    for gname, g in geoms:
        st.eval_device(tree, xd, out, g)
        torch.cuda.synchronize()
        ok = labels_fnv is None or st.fnv1a64(out.cpu().numpy()) == labels_fnv
        ms = timed(lambda: st.eval_device(tree, xd, out, g), iters, flush)
        timing = "events per launch (host launch latency included)"
        if flush is not None:  # small input: replay a CUDA graph to drop host overhead
            ms = graph_time(lambda: st.eval_device(tree, xd, out, g), iters, flush)
            timing = f"cuda-graph replay, L2 flushed ({FLUSH_MODE}) before every launch"
        gbs = 4 * a * m / (ms * 1e-3) / 1e9
        res[gname] = {"ms": round(ms, 5), "value": m / (ms * 1e-3) / unit_div, "unit": unit,
                      "GBs": round(gbs, 1), "frac": round(gbs / PEAK, 4), "labels_ok": bool(ok),
                      "timing": timing,
                      "geom": {k: v for k, v in g.__dict__.items() if v not in (0, "auto")}}
        print(name, gname, json.dumps(res[gname]), flush=True)
    del xd, out, flush
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--flush", choices=("read", "write"), default="read")
    ap.add_argument("--e2e", action="store_true", help="also time C1 / C3 / C4 end to end from pinned host memory")
    args = ap.parse_args()
    global FLUSH_MODE
    FLUSH_MODE = args.flush
    only = args.only.split(",")
    data_g = ("data", st.GpuGeom(algo="data"))
    spec_g = ("speculative", st.GpuGeom(algo="speculative"))
    spec_g2 = ("speculative-G2", st.GpuGeom(algo="speculative", group_lanes=2))
    spec_g8 = ("speculative-G8", st.GpuGeom(algo="speculative", group_lanes=8))
    spec_g16 = ("speculative-G16", st.GpuGeom(algo="speculative", group_lanes=16))
    data_const = ("data-constant-tree", st.GpuGeom(algo="data", tree_loc="constant"))
    data_glob = ("data-global-tree", st.GpuGeom(algo="data", tree_loc="global"))
    geoms = [data_g, data_const, data_glob, spec_g, spec_g2, spec_g8, spec_g16]
    out = {"peak_GBs": PEAK, "device": torch.cuda.get_device_name(0), "flush": FLUSH_MODE}
    W = bench.WORKLOADS
    for name in ("C1", "C2", "C3"):
        if name not in only:
            continue
        w = W[name]
        tree = st.generate_synthetic_tree(*w["tree"])
        x = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
        div, unit = (w["m"], "frames/s") if name == "C3" else (1.0, "samples/s")
        out[name] = run_tree(name, tree, x, w["labels_fnv"], geoms, args.iters, div, unit)
    if "PAPER" in only or "C1" in only:
        # the paper's own workload (main.cpp:233-246): tree(11,16,19,7,1) with
        # 15 internal nodes -> one speculative window on 16 lanes (Proc. 5)
        tree = st.generate_synthetic_tree(11, 16, 19, 7, 1)
        x = np.tile(st.generate_synthetic_dataset(16384, 19, 2), (4, 1))
        out["paper"] = run_tree("paper", tree, x, 0xc90f17638d0c1525,
                                [data_g, spec_g, ("speculative-G32", st.GpuGeom(algo="speculative", group_lanes=32))],
                                args.iters)
        x = np.tile(x, (256, 1))  # 16.8M records: out of L2, HBM-scale
        out["paper_x256"] = run_tree("paper_x256", tree, x, None,
                                     [data_g, spec_g, ("speculative-G4-windows", st.GpuGeom(algo="speculative", group_lanes=4)),
                                      ("speculative-G2-windows", st.GpuGeom(algo="speculative", group_lanes=2))], args.iters)
    if "C3" in only:
        # video stream: 32 frames (2.1 GB) per launch -> frames/s at HBM scale
        w = W["C3"]
        tree = st.generate_synthetic_tree(*w["tree"])
        frame = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
        x = np.tile(frame, (32, 1))
        r = run_tree("C3x32", tree, x, None, [data_g, spec_g], args.iters, w["m"], "frames/s")
        out["C3_batch32"] = r
    if "C5" in only:
        x = st.generate_synthetic_dataset(15_625_000, 16, 5000)
        sweep = {}
        for d in range(8, 21, 2):
            tree = st.generate_synthetic_tree(d, min(2**d, 4096), 16, 8, 500 + d)
            fnv = W.get(f"C5d{d}", {}).get("labels_fnv")
            r = run_tree(f"C5d{d}", tree, x, fnv, geoms, args.iters)
            best_spec = min((v for k, v in r.items() if k.startswith("spec")), key=lambda v: v["ms"])
            r["spec_over_data_time"] = round(r["speculative"]["ms"] / r["data"]["ms"], 3)
            r["best_spec_over_data_time"] = round(best_spec["ms"] / r["data"]["ms"], 3)
            r["tree"] = {"nodes": tree.size(), "depth": tree.depth()}
            sweep[f"d{d}"] = r
        out["C5"] = sweep
    if "C4" in only:
        trees = [st.generate_synthetic_tree(12, 1024, 64, 8, 401 + t) for t in range(128)]
        x = st.generate_synthetic_dataset(8_000_000, 64, 499)
        f = st.Forest(trees, 8)
        xd = torch.from_numpy(x).cuda()
        lab = torch.empty(len(x), dtype=torch.int32, device="cuda")
        st.eval_forest_device(f, xd, lab)
        torch.cuda.synchronize()
        ok = st.fnv1a64(lab.cpu().numpy()) == 0x1b2543c41e436ce0
        ms = timed(lambda: st.eval_forest_device(f, xd, lab), max(3, args.iters // 4))
        gbs = 4 * 64 * len(x) / (ms * 1e-3) / 1e9
        out["C4"] = {"ms": round(ms, 4), "value": len(x) / (ms * 1e-3), "unit": "samples/s",
                     "GBs": round(gbs, 1), "frac": round(gbs / PEAK, 4), "labels_ok": bool(ok),
                     "trees": 128, "node_visits_per_s_est": len(x) * 128 * 9.09 / (ms * 1e-3)}
        print("C4", json.dumps(out["C4"]), flush=True)
    if "E2E" in only or args.e2e:
        # end to end through the host-buffer API (pinned host records -> H2D ->
        # kernel -> D2H labels, chunked over 3 streams): PCIe-bound
        e2e = {}
        for name in ("C1", "C3"):
            w = W[name]
            tree = st.generate_synthetic_tree(*w["tree"])
            xh = torch.empty((w["m"], w["a"]), dtype=torch.float32, pin_memory=True)
            st.generate_synthetic_dataset(w["m"], w["a"], w["seed"], out=xh.numpy())
            lab = torch.empty(w["m"], dtype=torch.int32, pin_memory=True)
            st.eval_gpu(tree, xh.numpy(), out=lab.numpy().view(np.uint32))
            t0 = time.perf_counter()
            reps = 10
            for _ in range(reps):
                st.eval_gpu(tree, xh.numpy(), out=lab.numpy().view(np.uint32))
            dt = (time.perf_counter() - t0) / reps
            e2e[name] = {"s_per_call": dt, "samples_per_s": w["m"] / dt,
                         "h2d_GBs": 4 * w["a"] * w["m"] / dt / 1e9,
                         "frames_per_s" if name == "C3" else "calls_per_s": 1.0 / dt}
            print("E2E", name, json.dumps(e2e[name]), flush=True)
        trees = [st.generate_synthetic_tree(12, 1024, 64, 8, 401 + t) for t in range(128)]
        f = st.Forest(trees, 8)
        xh = torch.empty((8_000_000, 64), dtype=torch.float32, pin_memory=True)
        st.generate_synthetic_dataset(8_000_000, 64, 499, out=xh.numpy())
        st.eval_forest(f, xh.numpy())
        t0 = time.perf_counter()
        lab = st.eval_forest(f, xh.numpy())
        dt = time.perf_counter() - t0
        e2e["C4"] = {"s_per_call": dt, "samples_per_s": 8_000_000 / dt,
                     "labels_ok": st.fnv1a64(lab) == 0x1b2543c41e436ce0}
        print("E2E C4", json.dumps(e2e["C4"]), flush=True)
        out["e2e"] = e2e
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = "" if args.only == ap.get_default("only") else "_" + args.only.replace(",", "_")
    with open(os.path.join(ROOT, "gpurun_out", f"workloads_{FLUSH_MODE}{tag}.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
