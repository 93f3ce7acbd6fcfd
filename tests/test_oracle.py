"""Pin the CPU oracle (oracle/st_oracle.c) before trusting it.

1. Appendix A golden hashes (computed in the survey with the reference
   itself) for every canonical workload: tree bytes, dataset checksum, label
   hash, first labels, mean depth.
2. Reference-generated fixtures in tests/golden (make_golden.py): the oracle
   regenerates identical trees/records and reproduces the reference's labels,
   traversal depths and speculative step counters.
3. When oracle/_ref (the reference compiled here) exists: live cross-checks.
4. The exhaustive shape corpus (acceptance.cpp:71-116) against the pure-Python
   conditional-descent oracle (eval_serial.cpp:43-75).
"""
import os
import sys

import numpy as np
import pytest

import support
from paper_1111_1373_b200.tree import encode_breadth_first

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SMALL = ["paper", "fixture", "C1", "C3"]
LARGE = ["C2", "C4t0", "C5d8", "C5d12", "C5d16", "C5d20"]


def _check_workload(co, name):
    tspec, dspec, tile, tree_fnv, ds_ck, lab_fnv, first8, dmu = support.APPENDIX_A[name]
    nodes, x = support.workload(co, name)
    assert co.fnv1a(nodes) == tree_fnv, "tree bytes differ from the reference generator"
    assert co.dataset_checksum(x) == ds_ck, "records differ from the reference generator"
    labels = co.eval_serial(nodes, x)
    assert co.fnv1a(labels) == lab_fnv
    assert labels[:8].tolist() == first8
    depths = co.traversal_depths(nodes, x)
    assert abs(depths.mean() - dmu) < 6e-5


@pytest.mark.parametrize("name", SMALL)
def test_appendix_a_small(co, name):
    _check_workload(co, name)


@pytest.mark.parametrize("name", LARGE)
def test_appendix_a_large(co, name):
    _check_workload(co, name)


def test_c4_forest_chain_hash(co):
    """Forest tree bytes: h = offset; h ^= tree_fnv(t); h *= prime (Appendix A)."""
    h = 0xcbf29ce484222325
    for t in range(128):
        h ^= co.fnv1a(co.gen_tree(12, 1024, 64, 8, 401 + t))
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    assert h == support.C4_FOREST_CHAIN


def test_reference_fuzz_fixtures(co):
    g = np.load(os.path.join(GOLD, "ref_fuzz.npz"))
    for seed in range(1, 61):
        depth, leaves, arity, classes = support.fuzz_shape(seed)
        nodes = co.gen_tree(depth, leaves, arity, classes, seed)
        assert nodes.view(np.uint8).tobytes() == g[f"s{seed}_nodes"].tobytes(), seed
        x = co.gen_dataset(256, arity, seed + 5000, gaussian=(seed % 2 == 0))
        assert np.array_equal(x, g[f"s{seed}_x"]), seed
        assert np.array_equal(co.eval_serial(nodes, x), g[f"s{seed}_labels"]), seed
        assert np.array_equal(co.traversal_depths(nodes, x), g[f"s{seed}_depths"]), seed
        for k in (1, 2):
            lab, it, st = co.eval_speculative(nodes, x, k=k)
            assert np.array_equal(lab, g[f"s{seed}_labels"])
            assert np.array_equal(it, g[f"s{seed}_it{k}"]), (seed, k)
            assert np.array_equal(st, g[f"s{seed}_st{k}"]), (seed, k)


def test_reference_step_law_fixture(co):
    g = np.load(os.path.join(GOLD, "ref_steplaw.npz"))
    nodes = co.gen_tree(20, 40, 8, 5, 97)
    assert nodes.view(np.uint8).tobytes() == g["nodes"].tobytes()
    x = co.gen_dataset(10000, 8, 13)
    lab, it1, st1 = co.eval_speculative(nodes, x, k=1)
    assert np.array_equal(lab, g["labels"])
    assert np.array_equal(st1, g["st1"]) and np.array_equal(it1, g["it1"])
    want = np.array([support.ceil_log2(int(d)) for d in g["depths"]])
    assert np.array_equal(st1, want), "acceptance criterion 2 law"
    _, it2, _ = co.eval_speculative(nodes, x, k=2)
    assert np.array_equal(it2, (want + 1) // 2)


def test_live_reference_cross_check(co, ref):
    rng = np.random.default_rng(7)
    for seed in rng.integers(1, 10**6, size=25):
        seed = int(seed)
        depth, leaves, arity, classes = support.fuzz_shape(seed)
        a = co.gen_tree(depth, leaves, arity, classes, seed)
        b = ref.gen_tree(depth, leaves, arity, classes, seed)
        assert a.tobytes() == b.tobytes()
        for gauss in (False, True):
            xa = co.gen_dataset(500, arity, seed + 1, gauss)
            xb = ref.gen_dataset(500, arity, seed + 1, gauss)
            assert xa.tobytes() == xb.tobytes()
            assert np.array_equal(co.eval_serial(a, xa), ref.eval_serial(b, xb))
    # shuffle order: Fisher-Yates with the hand-rolled bounded draw
    order = co.shuffle_order(100, 5)
    assert sorted(order.tolist()) == list(range(100))


def test_exhaustive_shapes(co):
    """acceptance.cpp:100-116: every full shape up to 8 leaves (626)."""
    count = 0
    for leaves in range(1, 9):
        for shape in support.all_shapes(leaves):
            internal = support.assign_labels(shape)
            x = support.grid_records(internal)
            tree = encode_breadth_first(shape)
            want = support.recursive_oracle(shape, x)
            assert np.array_equal(co.eval_serial(tree.nodes(), x), want)
            lab, _, _ = co.eval_speculative(tree.nodes(), x, k=2)
            assert np.array_equal(lab, want)
            count += 1
    assert count == 626


def test_forest_vote_oracle(co):
    trees = [co.gen_tree(6, 20, 5, 4, 900 + t) for t in range(9)]
    x = co.gen_dataset(400, 5, 3)
    votes = np.stack([co.eval_serial(t, x) for t in trees])
    counts = np.stack([(votes == c).sum(0) for c in range(4)])
    want = counts.argmax(0)  # first max = smallest class id on ties
    assert np.array_equal(co.eval_forest(trees, x, 4), want)


def test_warp_sim_xcheck_profile(co):
    """profiles/r1_warp_sim_xcheck.json (ncu per-SASS-line counts of the data
    and EXACT speculative kernels vs the reference's lockstep warp model,
    tools/warp_sim_xcheck.py): every check is an exact equality, and the
    data-kernel predictions restate from the oracle's traversal depths
    (serialized passes = sum over 32-record warps of the deepest lane)."""
    import json

    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                     "r1_warp_sim_xcheck.json")
    rep = json.load(open(p))
    assert rep["all_equal"]
    sys.path.insert(0, os.path.join(os.path.dirname(p), "..", "tools"))
    import warp_sim_xcheck as xc

    for e in rep["launches"]:
        if e["algo"] != "data":
            continue
        nodes, x = xc.inputs(e["workload"], co.gen_tree, co.gen_dataset)
        d = co.traversal_depths(nodes, x).astype(np.int64).reshape(-1, 32)
        assert int(d.max(axis=1).sum()) == e["warp_sim"]["serialized_passes"] == e["ncu"]["warp_instructions"]
        assert int(d.sum()) == e["warp_sim"]["node_evals"] == e["ncu"]["active_thread_instructions"]
