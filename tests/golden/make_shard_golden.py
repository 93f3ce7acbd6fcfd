"""Per-shard / per-rank reference label hashes for the full-size workloads.

TEST INFRASTRUCTURE.  Runs in the build container only (needs
oracle/_ref/libspectree_ref.so, the reference core compiled unchanged from
/root/reference by `make -C oracle`).  The output, tests/golden/shard_hashes.json,
is committed so the GPU box (no /root/reference) can check every shard of the
10^9-record C5 sweep and every rank of the multi-GPU bench against the
reference itself.

    python tests/golden/make_shard_golden.py [--procs 8]

Contents (all label hashes are FNV-1a-64 over the raw little-endian u32
labels of spectree::eval_serial):

  c5      -- BASELINE configs[4]: shard s = generate_synthetic_dataset(
             15,625,000, 16, 5000 + s) (synthetic.cpp:156-182), s < 64;
             tree(D, min(2^D, 4096), 16, 8, 500 + D) for D = 8, 10, ..., 20.
             Per depth and shard: labels_fnv, and the sum / max of
             traversal_depths (eval_serial.cpp:77-105) so d_mu is pinned too.
  c2_ranks -- bench.py's C2 batch of rank r: tree(24, 256, 32, 8, 201) over
             data(16,000,000, 32, 202 + 1000 r), r < 8.
  c4_ranks -- bench.py's C4 batch of rank r: data(8,000,000, 64, 499 + 1000 r),
             128 trees tree(12, 1024, 64, 8, 401 + t); per-tree labels from the
             reference eval_serial, vote = per-class counts, smallest class id
             on ties (the reference has no forest).
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

C5_SHARD = 15_625_000
C5_SHARDS = 64
C5_A = 16
C5_DEPTHS = (8, 10, 12, 14, 16, 18, 20)


def c5_tree_args(depth):
    return (depth, min(2 ** depth, 4096), C5_A, 8, 500 + depth)


def _c5_shard(s):
    import oracle

    ref, co = oracle.RefOracle(), oracle.COracle()
    x = ref.gen_dataset(C5_SHARD, C5_A, 5000 + s)
    out = {}
    with ref.data(x) as d:
        for D in C5_DEPTHS:
            with ref.tree(ref.gen_tree(*c5_tree_args(D))) as t:
                labels = t.eval_serial(d)
                depths = t.traversal_depths(d)
            out[D] = (co.fnv1a(labels), int(depths.sum(dtype=np.uint64)), int(depths.max()))
    return s, out


def _c2_rank(r):
    import oracle

    ref, co = oracle.RefOracle(), oracle.COracle()
    x = ref.gen_dataset(16_000_000, 32, 202 + 1000 * r)
    with ref.data(x) as d, ref.tree(ref.gen_tree(24, 256, 32, 8, 201)) as t:
        return r, co.fnv1a(t.eval_serial(d))


def _c4_rank(r):
    import oracle

    ref, co = oracle.RefOracle(), oracle.COracle()
    m = 8_000_000
    x = ref.gen_dataset(m, 64, 499 + 1000 * r)
    counts = np.zeros((m, 8), np.uint8)
    rows = np.arange(m)
    with ref.data(x) as d:
        for t in range(128):
            with ref.tree(ref.gen_tree(12, 1024, 64, 8, 401 + t)) as tr:
                counts[rows, tr.eval_serial(d)] += 1
    vote = counts.argmax(axis=1).astype(np.uint32)  # argmax: first (smallest) class among maxima
    return r, co.fnv1a(vote)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--only", choices=["c5", "c2", "c4"], default=None)
    args = ap.parse_args()
    import oracle

    oracle.build()
    path = os.path.join(HERE, "shard_hashes.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    t0 = time.time()
    with mp.get_context("spawn").Pool(args.procs) as pool:
        if args.only in (None, "c2"):
            res = dict(pool.map(_c2_rank, range(8)))
            out["c2_ranks"] = {"tree": [24, 256, 32, 8, 201], "records": 16_000_000, "arity": 32,
                               "seed": "202 + 1000 r",
                               "labels_fnv": [f"0x{res[r]:016x}" for r in range(8)]}
            print(f"c2 ranks done {time.time() - t0:.0f}s", flush=True)
        if args.only in (None, "c4"):
            res = dict(pool.map(_c4_rank, range(8), chunksize=1))
            out["c4_ranks"] = {"trees": "tree(12, 1024, 64, 8, 401 + t), t < 128", "records": 8_000_000,
                               "arity": 64, "seed": "499 + 1000 r",
                               "vote_fnv": [f"0x{res[r]:016x}" for r in range(8)]}
            print(f"c4 ranks done {time.time() - t0:.0f}s", flush=True)
        if args.only in (None, "c5"):
            res = dict(pool.imap_unordered(_c5_shard, range(C5_SHARDS)))
            c5 = {"shard_records": C5_SHARD, "shards": C5_SHARDS, "arity": C5_A, "seed": "5000 + s",
                  "tree": "tree(D, min(2^D, 4096), 16, 8, 500 + D)", "depths": {}}
            for D in C5_DEPTHS:
                c5["depths"][str(D)] = {
                    "labels_fnv": [f"0x{res[s][D][0]:016x}" for s in range(C5_SHARDS)],
                    "depth_sum": [res[s][D][1] for s in range(C5_SHARDS)],
                    "depth_max": [res[s][D][2] for s in range(C5_SHARDS)],
                }
            out["c5"] = c5
            print(f"c5 done {time.time() - t0:.0f}s", flush=True)
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
