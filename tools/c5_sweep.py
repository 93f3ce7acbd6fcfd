"""C5: the 10^9-record sharded sweep over tree depth (BASELINE configs[4],
SURVEY §8d/§8e) at full size.

    64 shards x data(15,625,000, 16, 5000 + s) = 10^9 records (64 GB), resident
    in HBM, split over the GPUs by the Proc. 3 range rule (GPU g owns shards
    [g*64/G, (g+1)*64/G)); tree(D, min(2^D, 4096), 16, 8, 500 + D) for
    D = 8, 10, ..., 20, replicated.  Per depth and algorithm: one launch per
    GPU over its contiguous shard block, all GPUs launched together, time =
    max over GPUs of the CUDA-event time (median of --reps).  No collective:
    the only exchange is the label gather, timed separately (D2H of every
    GPU's labels into one pinned host buffer).  Parity: every shard's
    labels at every depth, both algorithms, against the reference hashes in
    tests/golden/shard_hashes.json (generated from oracle/_ref by
    tests/golden/make_shard_golden.py; shard 0 = SURVEY Appendix A).

Records are generated on the host with the reference generator (one thread
per shard, st_synthetic_dataset releases the GIL) straight into pinned
staging buffers and copied to the owning GPU.

    python tools/c5_sweep.py [--gpus N] [--shards 64] [--reps 5]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

SHARD = 15_625_000
A = 16
GOLD = bench.golden().get("c5", {}).get("depths", {})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--shards", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--depths", default="8,10,12,14,16,18,20")
    args = ap.parse_args()
    G, S = args.gpus, args.shards
    ndev = torch.cuda.device_count()
    dv = lambda g: g % ndev  # noqa: E731  (more shard owners than GPUs: validation runs only)
    peak, _ = bench.peaks()
    own = [(g * S // G, (g + 1) * S // G) for g in range(G)]
    xs, labs, streams = [], [], []
    t_gen = time.perf_counter()
    for g, (lo, hi) in enumerate(own):
        dev = torch.device("cuda", dv(g))
        xs.append(torch.empty(((hi - lo) * SHARD, A), dtype=torch.float32, device=dev))
        labs.append(torch.empty((hi - lo) * SHARD, dtype=torch.int32, device=dev))
        streams.append(torch.cuda.Stream(device=dev))
    # host generation: a ring of pinned staging buffers, one shard each
    ring = [torch.empty((SHARD, A), dtype=torch.float32, pin_memory=True) for _ in range(8)]

    def gen(s, buf):
        st.generate_synthetic_dataset(SHARD, A, 5000 + s, out=buf.numpy())
        return s

    owner = {s: g for g, (lo, hi) in enumerate(own) for s in range(lo, hi)}
    with cf.ThreadPoolExecutor(max_workers=min(len(ring), os.cpu_count() or 1)) as pool:
        pending = {}
        free = list(ring)  # staging buffers not owned by an in-flight shard
        nxt = 0
        while nxt < S or pending:
            while nxt < S and free:
                buf = free.pop()
                pending[pool.submit(gen, nxt, buf)] = (nxt, buf)
                nxt += 1
            done, _ = cf.wait(list(pending), return_when=cf.FIRST_COMPLETED)
            for f in done:
                s, buf = pending.pop(f)
                f.result()
                g = owner[s]
                lo = own[g][0]
                with torch.cuda.device(dv(g)):
                    xs[g][(s - lo) * SHARD:(s - lo + 1) * SHARD].copy_(buf)  # synchronous
                free.append(buf)
    t_gen = time.perf_counter() - t_gen
    print(f"generated {S} shards ({S * SHARD * A * 4 / 1e9:.1f} GB) in {t_gen:.1f} s", flush=True)
    labels_host = torch.empty(S * SHARD, dtype=torch.int32, pin_memory=True)

    out = {"gpus": G, "devices_used": min(G, ndev), "shards": S, "records": S * SHARD, "arity": A, "peak_GBs": peak,
           "device": torch.cuda.get_device_name(0), "generation_s": t_gen, "depths": {}}
    for D in [int(d) for d in args.depths.split(",")]:
        tree = st.generate_synthetic_tree(D, min(2 ** D, 4096), A, 8, 500 + D)
        row = {"tree": {"nodes": tree.size(), "depth": tree.depth()}}
        for algo in ("data", "speculative"):
            geom = st.GpuGeom(algo=algo)

            def launch_all():
                evs = []
                for g in range(G):
                    with torch.cuda.device(dv(g)):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(streams[g])
                        st.eval_device(tree, xs[g], labs[g], geom, stream=streams[g])
                        e1.record(streams[g])
                        evs.append((e0, e1))
                for g in range(G):
                    torch.cuda.synchronize(dv(g))
                return max(a.elapsed_time(b) for a, b in evs) / 1e3

            launch_all()  # warm (device tree / window tables)
            # every shard against the reference hash of that shard and depth
            want = GOLD.get(str(D), {}).get("labels_fnv", [])
            parts = []
            for g, (lo, hi) in enumerate(own):
                host = labs[g].cpu().numpy()
                parts += [(s, host[(s - lo) * SHARD:(s - lo + 1) * SHARD]) for s in range(lo, hi)]
            with cf.ThreadPoolExecutor(max_workers=16) as pool:
                hashes = list(pool.map(lambda p: st.fnv1a64(p[1]), parts))
            ok = [h == int(want[s], 16) if s < len(want) else None for (s, _), h in zip(parts, hashes)]
            del parts
            ts = [launch_all() for _ in range(args.reps)]
            t = statistics.median(ts)
            gbs = S * SHARD * A * 4 / t / 1e9
            row[algo] = {"s": t, "samples_per_s": S * SHARD / t, "GBs": gbs,
                         "frac_of_G_x_peak": gbs / (G * peak),
                         "shards_match_reference": f"{sum(v is True for v in ok)}/{len(ok)}",
                         "all_shards_match_reference": all(v is True for v in ok)}
        # label gather: every GPU's labels into one pinned host buffer
        g0 = time.perf_counter()
        off = 0
        for g in range(G):
            n = labs[g].numel()
            labels_host[off:off + n].copy_(labs[g], non_blocking=True)
            off += n
        for g in range(G):
            torch.cuda.synchronize(dv(g))
        row["label_gather_s"] = time.perf_counter() - g0
        row["spec_over_data_time"] = row["speculative"]["s"] / row["data"]["s"]
        out["depths"][f"d{D}"] = row
        print(f"D={D}", json.dumps(row), flush=True)
    ratios = {k: v["spec_over_data_time"] for k, v in out["depths"].items()}
    out["crossover"] = ("none: speculative is slower at every depth" if all(r > 1 for r in ratios.values())
                        else [k for k, r in ratios.items() if r <= 1])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"c5_sweep_g{G}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
