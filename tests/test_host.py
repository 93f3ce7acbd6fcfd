"""CPU tests of the host side: the C-ABI library loads and exports every symbol
include/spectree_b200.h declares; argument errors surface before any device
work with the reference's messages; the tree model / JSON boundary / config
validation mirror the reference (tree.cpp, io.cpp, eval_*.cpp)."""
import json
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1111_1373_b200 as st
import support
from paper_1111_1373_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spectree_b200.h")
GOLD = os.path.join(ROOT, "tests", "golden")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


# ---------------------------------------------------------------- C ABI ----
def test_header_symbols_exported():
    decl = set(re.findall(r"^(?:int|void|const char\*|uint32_t|uint64_t)\s+(st_[a-z0-9_]+)\(", open(HEADER).read(), re.M))
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = decl - exported
    assert not missing, f"declared but not exported: {missing}"
    assert set(_lib.EXPORTS) == decl


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_struct_sizes():
    import ctypes as C

    assert C.sizeof(_lib.st_geom) == 96
    assert st.NODE_DTYPE.itemsize == 16
    assert [st.NODE_DTYPE.fields[f][1] for f in ("attribute", "threshold", "child", "class_id")] == [0, 4, 8, 12]


def test_version_and_geom_default():
    L = _lib.load()
    assert b"sm_100a" in L.st_version()
    g = _lib.st_geom()
    g.algo = 7
    L.st_geom_default(g)
    assert g.algo == 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback(co):
    nodes = co.gen_tree(11, 16, 19, 7, 1)
    x = co.gen_dataset(64, 19, 2)
    with pytest.raises(st.NoDeviceError):
        st.eval_gpu(nodes, x)
    with pytest.raises(st.NoDeviceError):
        st.eval_data_parallel(nodes, x)
    with pytest.raises(st.NoDeviceError):
        st.eval_forest(st.Forest([nodes], 7), x)
    with pytest.raises(st.NoDeviceError):
        st.FrameStream(co.gen_tree(10, 1024, 16, 8, 101), 4096, 16)


def test_frame_stream_argument_errors_before_device(co):
    """st_frames_open validates before touching a device (same taxonomy as
    st_eval): arity without TMA row-local tiles, empty frames, ring size,
    attribute range, the speculative algorithm."""
    nodes = co.gen_tree(10, 1024, 16, 8, 101)  # reads attributes < 16
    for args, kw, msg in [((4096, 19), {}, "8, 16 or 32 attributes"),
                          ((0, 16), {}, "records per frame"),
                          ((4096, 16), {"ring": 0}, "ring must hold"),
                          ((4096, 8), {}, "reads attribute")]:
        with pytest.raises(st.ArgumentError, match=msg):
            st.FrameStream(nodes, *args, **kw)


def test_argument_errors_before_device(co):
    """check_attribute_range (eval_serial.cpp:10-17) fires before any work."""
    nodes = co.gen_tree(11, 16, 19, 7, 1)  # max attribute 17
    with pytest.raises(st.ArgumentError, match="reads attribute 17 but records have arity 3"):
        st.eval_gpu(nodes, np.zeros((5, 3), np.float32))
    # leaf attribute counts toward max_attribute (tree.cpp:47)
    bad = st.encode_breadth_first(st.make_split(1, 0.5, st.make_leaf(1), st.make_leaf(2)))
    raw = bad.nodes().copy()
    raw[1]["attribute"] = 9
    with pytest.raises(st.ArgumentError, match="reads attribute 9"):
        st.eval_gpu(raw, np.zeros((2, 4), np.float32))


def test_tree_create_rejects_unsafe_links():
    L = _lib.load()
    import ctypes as C

    def create(nodes):
        h = C.c_void_p()
        rc = L.st_tree_create(nodes.ctypes.data_as(C.c_void_p), len(nodes), C.byref(h))
        if rc == 0:
            L.st_tree_destroy(h)
        return rc, _lib.last_error()

    t = st.encode_breadth_first(st.make_split(0, 0.5, st.make_leaf(1), st.make_leaf(2))).nodes().copy()
    assert create(t)[0] == 0
    back = t.copy()
    back[0]["child"] = 0
    rc, msg = create(back)
    assert rc == 2 and "does not point forward" in msg
    oob = t.copy()
    oob[0]["child"] = 2
    rc, msg = create(oob)
    assert rc == 2 and "out of range" in msg
    rc, msg = create(np.zeros(0, dtype=st.NODE_DTYPE))
    assert rc == 2 and "at least one node" in msg


def test_tree_info_windows(co):
    paper = st.tree_info(co.gen_tree(11, 16, 19, 7, 1))
    assert paper["internal"] == 15 and paper["depth"] == 11
    assert paper["spec_windows"] == 1 and paper["spec_group_lanes"] == 16
    c1 = st.tree_info(co.gen_tree(10, 1024, 16, 8, 101))
    assert c1["internal"] == 1023 and c1["compact"] == 1
    # default: 2-level windows of 3 nodes over a complete depth-10 tree
    assert c1["spec_group_lanes"] == 4 and c1["spec_windows"] == 1 + 4 + 16 + 64 + 256
    leaf = st.tree_info(st.EncodedTree(np.array([(0, np.inf, 0, 5)], dtype=st.NODE_DTYPE)))
    assert leaf["spec_windows"] == 0 and leaf["nodes"] == 1


def _windows_python(nodes, G=4, H=2):
    """Independent restatement of st_tree::build_windows' partition: windows
    of <= G internal nodes and <= H levels, breadth-first from each window root,
    window roots discovered breadth-first."""
    import collections

    leaf = lambda i: nodes[i]["class_id"] != st.NO_CLASS  # noqa: E731
    if leaf(0):
        return 0
    win_of_root, order, roots = {0: 0}, [0], collections.deque([0])
    while roots:
        r = roots.popleft()
        mem, q, exits = [], collections.deque([(r, 0)]), []
        while q:
            u, d = q.popleft()
            if len(mem) >= G or d >= H:
                exits.append(u)
                continue
            mem.append(u)
            for c in (int(nodes[u]["child"]), int(nodes[u]["child"]) + 1):
                if not leaf(c):
                    q.append((c, d + 1))
        for u in exits:
            if u not in win_of_root:
                win_of_root[u] = len(order)
                order.append(u)
                roots.append(u)
    return len(order)


def test_window_partition_matches_restatement(co):
    """The speculative window count of the default geometry (3-node, 2-level
    windows for trees with > 32 internal nodes) equals a Python restatement
    of the partition on random balanced and skewed trees."""
    rng = np.random.default_rng(7)
    for k in range(40):
        depth = int(rng.integers(6, 21))
        leaves = int(min(2 ** depth, rng.integers(depth + 1, 3000)))
        nodes = co.gen_tree(depth, leaves, 16, 8, 1000 + k)
        info = st.tree_info(nodes)
        if info["internal"] <= 32:
            continue
        assert info["spec_group_lanes"] == 4
        assert info["spec_windows"] == _windows_python(nodes), (depth, leaves)


# ------------------------------------------------------------ tree model ---
def test_encode_matches_reference_layout(co):
    """encode(decode(t)) reproduces the reference BFS bytes (tree.cpp:72-136)."""
    for seed in (1, 7, 101):
        nodes = co.gen_tree(11, 16, 19, 7, seed) if seed < 100 else co.gen_tree(10, 1024, 16, 8, seed)
        t = st.EncodedTree(nodes)
        assert st.encode_breadth_first(st.decode(t)) == t
        assert st.validate(t) == []


def test_tree_stats_mirror_reference(co):
    nodes = co.gen_tree(24, 256, 32, 8, 201)
    t = st.EncodedTree(nodes)
    assert t.size() == 511 and t.leaf_count() == 256 and t.depth() == 24
    assert t.max_attribute() == 31
    assert np.array_equal(st.processor_node_map(t), np.nonzero(nodes["class_id"] == st.NO_CLASS)[0])


def test_encoder_structure_errors():
    bad = st.LinkedNode(left=st.make_leaf(1))
    with pytest.raises(st.StructureError, match="non-full node"):
        st.encode_breadth_first(bad)
    with pytest.raises(st.StructureError, match="leaf without a class at root"):
        st.encode_breadth_first(st.LinkedNode())
    with pytest.raises(st.ArgumentError):
        st.make_leaf(st.NO_CLASS)


def test_validate_findings():
    t = st.encode_breadth_first(st.make_split(0, 0.5, st.make_leaf(1), st.make_leaf(2)))
    raw = t.nodes().copy()
    raw[1]["threshold"] = 0.0
    raw[2]["child"] = 1
    msgs = [d.message for d in st.validate(st.EncodedTree(raw))]
    assert "leaf threshold is not +inf" in msgs
    assert any("expected self-loop 2" in m for m in msgs)


def test_tree_json_against_reference_fixture(co):
    g = json.load(open(os.path.join(GOLD, "ref_json.json")))
    t = st.load_tree_json_text(g["paper_tree_json"])
    assert t.nodes().tobytes() == co.gen_tree(11, 16, 19, 7, 1).tobytes()
    back = st.load_tree_json_text(st.tree_to_json(t))
    assert back == t


def test_tree_json_matches_live_reference_loader(ref, co):
    text = st.tree_to_json(st.EncodedTree(co.gen_tree(8, 30, 4, 3, 11)))
    assert ref.load_tree_json(text).tobytes() == st.load_tree_json_text(text).nodes().tobytes()


@pytest.mark.parametrize("doc,msg", [
    ("[]", "top level must be an object"),
    ('{"nodes": []}', "missing integer 'version'"),
    ('{"version": 2, "nodes": [1]}', "unsupported schema version 2"),
    ('{"version": 1, "nodes": []}', "'nodes' must be a non-empty array"),
    ('{"version": 1, "nodes": [{"attr": 0, "thr": "-inf", "child": 3, "class": 1}]}',
     "child index 3 out of range"),
    ('{"version": 1, "nodes": [{"attr": 0, "thr": 0.5, "child": 0, "class": 1}]}',
     "leaf thr must be the string"),
    ('{"version": 1, "nodes": [{"attr": -1, "thr": "-inf", "child": 0, "class": 1}]}',
     "attr must be an unsigned 32-bit integer"),
])
def test_tree_json_schema_errors(doc, msg):
    with pytest.raises(st.SchemaError, match=re.escape(msg)):
        st.load_tree_json_text(doc)


# ------------------------------------------------------- config validation ---
def test_validate_data_parallel_messages():
    with pytest.raises(st.ArgumentError, match="workers must be >= 1"):
        st.validate_data_parallel(st.DataParallelConfig(workers=0), 10)
    with pytest.raises(st.ArgumentError, match="chunk must be >= 1"):
        st.validate_data_parallel(st.DataParallelConfig(chunk=0), 10)
    with pytest.raises(st.ArgumentError, match="leaves records unassigned"):
        st.validate_data_parallel(st.DataParallelConfig(workers=3, chunk=3), 10)
    with pytest.raises(st.ArgumentError, match="exact fit requires"):
        st.validate_data_parallel(st.DataParallelConfig(workers=4, chunk=3, exact_fit=True), 10)
    st.validate_data_parallel(st.DataParallelConfig(workers=300, chunk=1), 300)


def test_validate_speculative_messages(co):
    """test_eval_speculative.cpp:266-314."""
    tree = st.EncodedTree(co.gen_tree(4, 7, 2, 3, 2))  # 13 nodes
    good = st.default_speculative(tree, 10, records_per_group=4)
    st.validate_speculative(good, tree, 10, False)
    import dataclasses as dc

    cases = [(dict(group_lanes=0), False, "group_lanes must be >= 1"),
             (dict(group_lanes=5), False, "internal node"),
             (dict(group_lanes=12), True, "one per node"),
             (dict(groups=0), False, "groups must be >= 1"),
             (dict(records_per_group=0), False, "records_per_group must be >= 1"),
             (dict(reductions_per_iteration=0), False, "reductions_per_iteration must be >= 1"),
             (dict(groups=2, records_per_group=4), False, "unassigned")]
    for kw, basic, msg in cases:
        with pytest.raises(st.ArgumentError, match=msg):
            st.validate_speculative(dc.replace(good, **kw), tree, 10, basic)
    st.validate_speculative(dc.replace(good, group_lanes=13), tree, 10, True)


def test_gpu_geometry_argument_errors(co):
    nodes = co.gen_tree(11, 16, 19, 7, 1)
    x = co.gen_dataset(64, 19, 2)
    with pytest.raises(st.ArgumentError):
        st.eval_gpu(nodes, x, st.GpuGeom(algo="bogus"))
    with pytest.raises(st.ArgumentError):
        st.eval_gpu(nodes, x, layout="columnar")


def test_dataset_mirror():
    with pytest.raises(st.ArgumentError, match="arity must be >= 1"):
        st.Dataset(0)
    with pytest.raises(st.ArgumentError, match="multiple of the arity"):
        st.Dataset(3, np.zeros(4, np.float32))
    d = st.Dataset(2, [1, 2, 3, 4])
    assert d.count() == 2 and d.record(1).tolist() == [3, 4]
    assert st.tile_dataset(d, 3).count() == 6
    d.append([5, 6])
    assert d.count() == 3


# --------------------------------------------------- input-side API (L1) ---
@pytest.mark.parametrize("name", ["paper", "fixture", "C1", "C3"])
def test_product_generators_match_reference(co, name):
    """st_synthetic_* == oracle restatement == Appendix A (reference) bytes."""
    tspec, dspec, tile, tree_fnv, ds_ck, *_ = support.APPENDIX_A[name]
    t = st.generate_synthetic_tree(*tspec)
    assert st.fnv1a64(t.nodes()) == tree_fnv
    assert t.nodes().tobytes() == co.gen_tree(*tspec).tobytes()
    x = st.generate_synthetic_dataset(*dspec)
    if tile > 1:
        x = np.tile(x, (tile, 1))
    assert st.dataset_checksum(x) == ds_ck


def test_product_generators_fuzz_and_gaussian(co):
    for seed in range(1, 120, 7):
        spec = support.fuzz_shape(seed)
        assert st.generate_synthetic_tree(*spec, seed).nodes().tobytes() == co.gen_tree(*spec, seed).tobytes()
        for gauss in (False, True):
            a = st.generate_synthetic_dataset(300, spec[2], seed, gauss)
            assert a.tobytes() == co.gen_dataset(300, spec[2], seed, gauss).tobytes()
    with pytest.raises(st.ArgumentError, match="exceeds 2\\^depth"):
        st.generate_synthetic_tree(3, 9, 2, 2, 1)
    with pytest.raises(st.ArgumentError, match="need at least depth \\+ 1 leaves"):
        st.generate_synthetic_tree(5, 3, 2, 2, 1)


def test_cli_cpu_strategies_and_exit_codes(tmp_path):
    """tools/spectree_b200_cli (the reference CLI's verify/bench with GPU names,
    built against the reference sources into oracle/_ref): CPU strategies run
    here; a GPU strategy without a device exits 3 (Error, no CPU fallback);
    an unknown strategy exits 2 (ArgumentError) -- main.cpp:37-40, 703-712."""
    import subprocess

    cli = os.path.join(ROOT, "oracle", "_ref", "spectree_b200_cli")
    if not os.path.exists(cli):
        pytest.skip("oracle/_ref/spectree_b200_cli not built (needs /root/reference)")
    t, d = str(tmp_path / "t.json"), str(tmp_path / "d.strec")
    r = subprocess.run([cli, "gen", "--records", "2000", "--out-tree", t, "--out-data", d],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([cli, "verify", "--tree", t, "--data", d, "--strategy", "serial", "--strategy", "data",
                        "--strategy", "spec", "--strategy", "spec-basic"], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.count(": OK (2000 records)") == 4, r.stdout + r.stderr
    r = subprocess.run([cli, "bench", "--tree", t, "--data", d, "--strategy", "serial", "--strategy", "data",
                        "--iterations", "3", "--warmup", "1", "--format", "json"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    import json as _json
    rep = _json.loads(r.stdout)
    assert rep["version"] == 1 and [s["name"] for s in rep["strategies"]] == ["serial", "data"]
    assert rep["strategies"][1]["inner_us"]["iterations"] == 3
    import torch

    if not torch.cuda.is_available():
        r = subprocess.run([cli, "verify", "--tree", t, "--data", d, "--strategy", "gpu-data"],
                           capture_output=True, text=True)
        assert r.returncode == 3 and "no CUDA device" in r.stderr
    r = subprocess.run([cli, "verify", "--tree", t, "--data", d, "--strategy", "nope"],
                       capture_output=True, text=True)
    assert r.returncode == 2
    r = subprocess.run([cli, "verify", "--tree", t], capture_output=True, text=True)
    assert r.returncode == 2 and "--data is required" in r.stderr
