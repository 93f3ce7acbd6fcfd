"""C3 frame rate three ways on one B200, data and speculative decomposition
(writes gpurun_out/frames_C3.json):

  single   one st_eval_device launch per frame (L2 flushed between frames),
  batched  F frames in one launch (m = F x 2,073,600 records),
  stream   the resident frame stream (st_frames_*): frames published into a
           device ring by a producer stream (device-resident records: the
           device-producer case), labels waited for on a consumer stream.

Every frame's labels are checked against the reference hash of the C3 frame
(tests/golden via bench.WORKLOADS).  Times are CUDA events on the streams
that carry the work; frames/s = frames / elapsed.

    python tools/frames_bench.py [--frames 256] [--ring 8] [--pub-batch 1]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402
import workloads  # noqa: E402


def sync(stream, timeout_s=30.0):
    """Host wait for a stream with a deadline (a stream waiting on a frame
    that never completes must not hang the benchmark)."""
    import time

    t0 = time.time()
    while not stream.query():
        if time.time() - t0 > timeout_s:
            raise RuntimeError("frame stream did not complete within the deadline")
        time.sleep(1e-4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=256)
    ap.add_argument("--ring", type=int, default=8)
    ap.add_argument("--pub-batch", type=int, default=1, help="frames per acquire/publish pair")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--algos", default="data,speculative")
    args = ap.parse_args()
    w = bench.WORKLOADS["C3"]
    tree = st.generate_synthetic_tree(*w["tree"])
    frame = st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])
    rec, a = w["m"], w["a"]
    peak, _ = bench.peaks()
    fbytes = rec * a * 4
    res = {"workload": w["desc"], "records_per_frame": rec, "arity": a, "bytes_per_frame": fbytes,
           "peak_gbs": peak}
    dev = torch.device("cuda", 0)
    xd = torch.from_numpy(frame).to(dev)
    out = torch.empty(rec, dtype=torch.int32, device=dev)
    fl = workloads.make_flush()
    for algo in args.algos.split(","):
        g = st.GpuGeom(algo=algo)
        r = res[algo] = {}
        # single launch per frame, L2 flushed before each (graph replay)
        t1 = workloads.graph_time(lambda: st.eval_device(tree, xd, out, g), 20, fl)
        assert st.fnv1a64(out.cpu().numpy()) == w["labels_fnv"]
        r["single"] = {"us_per_frame": t1 * 1e3, "frames_per_s": 1e3 / t1}
        # batched: F frames in one launch
        F = args.batch
        xb = xd.repeat(F, 1)
        ob = torch.empty(rec * F, dtype=torch.int32, device=dev)
        tb = workloads.timed(lambda: st.eval_device(tree, xb, ob, g), 10)
        assert torch.equal(ob.view(F, -1), ob[:rec].expand(F, -1))
        r["batched"] = {"frames_per_launch": F, "us_per_frame": tb * 1e3 / F, "frames_per_s": F * 1e3 / tb}
        del xb, ob
        # resident stream: prefill every ring slot once, then publish frames
        n, ring = args.frames, args.ring
        prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
        outs = torch.empty((ring, rec), dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        with st.FrameStream(tree, rec, a, ring=ring, geom=g, idle_timeout_ms=30000) as fs:
            for k in range(ring):
                x, _ = fs.slot(k)
                with torch.cuda.stream(prod):
                    x.copy_(xd, non_blocking=True)
            sync(prod)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            runs = []
            seq = 0
            for rep in range(3):
                ev0.record(prod)
                for k in range(0, n, args.pub_batch):
                    last = seq + args.pub_batch - 1
                    fs.acquire(last, prod)  # frame last - ring done (and every earlier frame)
                    fs.publish(last, prod)  # the slots' records stay in place (device producer)
                    seq = last + 1
                fs.wait(seq - 1, cons)
                ev1.record(cons)
                sync(cons)
                runs.append(ev0.elapsed_time(ev1))
            # labels of the last ring frames
            for k in range(seq - ring, seq):
                fs.wait(k, cons)
                _, lab = fs.slot(k)
                with torch.cuda.stream(cons):
                    outs[k % ring].copy_(lab, non_blocking=True)
            sync(cons)
            ok = all(st.fnv1a64(outs[q].cpu().numpy()) == w["labels_fnv"] for q in range(ring))
            assert ok, "frame stream labels differ from the reference hash"
            ms = min(runs)
            r["stream"] = {"frames": n, "ring": ring, "pub_batch": args.pub_batch, "ms": runs,
                           "us_per_frame": ms * 1e3 / n, "frames_per_s": n * 1e3 / ms,
                           "hbm_gbs": fbytes * n / (ms * 1e-3) / 1e9,
                           "hbm_frac": fbytes * n / (ms * 1e-3) / 1e9 / peak, "labels_match_reference": ok}
        for k in ("single", "batched"):
            r[k]["hbm_gbs"] = fbytes / (r[k]["us_per_frame"] * 1e-6) / 1e9
            r[k]["hbm_frac"] = r[k]["hbm_gbs"] / peak
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "frames_C3.json"), "w"), indent=1)
    print(json.dumps({k: (v if not isinstance(v, dict) else
                          {kk: {x: y for x, y in vv.items() if x != "ms"} for kk, vv in v.items()})
                      for k, v in res.items()}))


if __name__ == "__main__":
    main()
