"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libspectree_ref.so, built
by `make -C oracle` from the unmodified sources under /root/reference).  The
fixtures are committed so the GPU box (which has no /root/reference) can pin
both the oracle restatement and the CUDA kernels against reference outputs.

    python tests/golden/make_golden.py

Fixtures:
  ref_fuzz.npz      -- the acceptance fuzz recipe (acceptance.cpp:119-143) for
                       seeds 1..60 at 256 records each: tree nodes, records,
                       eval_serial labels, traversal depths, and
                       eval_speculative (mapped, k=1 and k=2, barrier-separated)
                       per-record iterations / doubling steps.
  ref_steplaw.npz   -- criterion 2 workload (acceptance.cpp:173-211): tree
                       (20, 40, 8, 5, 97) on data(10000, 8, 13); labels, depths,
                       k=1 and k=2 stats.
  ref_json.json     -- tree_to_json of the paper-like tree and its round trip.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def fuzz_shape(seed: int):
    """acceptance.cpp:120-128."""
    depth = 1 + seed % 20
    lo = depth + 1
    cap = 1024 if depth >= 10 else (1 << depth)
    hi = min(cap, lo + 19)
    leaves = lo + (seed * 7) % (hi - lo + 1)
    arity = 1 + (seed * 3) % 8
    classes = 2 + seed % 9
    return depth, leaves, arity, classes


def main() -> None:
    oracle.build()
    ref = oracle.RefOracle()
    out = {}
    for seed in range(1, 61):
        depth, leaves, arity, classes = fuzz_shape(seed)
        nodes = ref.gen_tree(depth, leaves, arity, classes, seed)
        x = ref.gen_dataset(256, arity, seed + 5000, gaussian=(seed % 2 == 0))
        with ref.tree(nodes) as t, ref.data(x) as d:
            labels = t.eval_serial(d)
            depths = t.traversal_depths(d)
            internal = max(1, (len(nodes) - 1) // 2)
            _, it1, st1, _ = t.eval_speculative(d, internal, 256, 1, k=1)
            _, it2, st2, _ = t.eval_speculative(d, internal, 256, 1, k=2)
        out[f"s{seed}_nodes"] = nodes.view(np.uint8)
        out[f"s{seed}_x"] = x
        out[f"s{seed}_labels"] = labels
        out[f"s{seed}_depths"] = depths
        out[f"s{seed}_it1"] = it1
        out[f"s{seed}_st1"] = st1
        out[f"s{seed}_it2"] = it2
        out[f"s{seed}_st2"] = st2
    np.savez_compressed(os.path.join(HERE, "ref_fuzz.npz"), **out)

    nodes = ref.gen_tree(20, 40, 8, 5, 97)
    x = ref.gen_dataset(10000, 8, 13)
    with ref.tree(nodes) as t, ref.data(x) as d:
        labels = t.eval_serial(d)
        depths = t.traversal_depths(d)
        internal = (len(nodes) - 1) // 2
        _, it1, st1, _ = t.eval_speculative(d, internal, 625, 16, k=1)
        _, it2, st2, _ = t.eval_speculative(d, internal, 625, 16, k=2)
    np.savez_compressed(os.path.join(HERE, "ref_steplaw.npz"), nodes=nodes.view(np.uint8),
                        labels=labels, depths=depths, it1=it1, st1=st1, it2=it2, st2=st2)

    paper = ref.gen_tree(11, 16, 19, 7, 1)
    text = ref.tree_to_json(paper)
    back = ref.load_tree_json(text)
    with open(os.path.join(HERE, "ref_json.json"), "w") as f:
        json.dump({"paper_tree_json": text,
                   "roundtrip_equal": bool(back.tobytes() == paper.tobytes())}, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
