"""GPU tests for the §8f rows: the reference bench flow with GPU strategies
(st_eval_timed, bench_flow, the C++ CLI over include/spectree_b200_bench.hpp)
and the streaming record-file evaluator (st_eval_file), all against the
oracle's eval_serial labels."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_1111_1373_b200 as st
from paper_1111_1373_b200 import bench_flow
from paper_1111_1373_b200.errors import ArgumentError

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "oracle", "_ref", "spectree_b200_cli")


def test_eval_timed_phases(cuda, co):
    nodes = co.gen_tree(10, 1024, 16, 8, 101)
    x = co.gen_dataset(200_000, 16, 102)
    want = co.eval_serial(nodes, x)
    for algo in ("data", "speculative"):
        got, t = bench_flow.eval_timed(nodes, x, st.GpuGeom(algo=algo))
        assert np.array_equal(got, want), algo
        assert t["inner_us"] > 0 and t["h2d_us"] > 0 and t["d2h_us"] > 0 and t["alloc_us"] > 0
        assert t["outer_us"] >= t["inner_us"] + t["h2d_us"]


def test_run_bench_gpu_strategies(cuda, co):
    nodes = co.gen_tree(11, 16, 19, 7, 1)
    x = np.tile(co.gen_dataset(16384, 19, 2), (4, 1))
    want = co.eval_serial(nodes, x)
    reps = bench_flow.run_bench(nodes, x, iterations=5, warmup=2, expected=want)
    assert [r.strategy.value for r in reps] == ["gpu-data", "gpu-spec"]
    for r in reps:
        assert r.mismatches == 0 and r.outer.iterations == 5 and r.inner.mean_us > 0
    with pytest.raises(ArgumentError):
        bench_flow.run_bench(nodes, x, iterations=0)


@pytest.mark.parametrize("layout,width", [("aos", 4), ("soa", 4), ("aos", 1)])
def test_eval_file_streaming(cuda, co, tmp_path, layout, width):
    """> 64 MB of records -> several pinned chunks through the 3-buffer pipeline."""
    nodes = co.gen_tree(24, 256, 32, 8, 201)
    x = co.gen_dataset(700_001, 32, 202)  # 89.6 MB, ragged last chunk
    want = co.eval_serial(nodes, x)
    src, dst = str(tmp_path / "d.strec"), str(tmp_path / "l.stlab")
    st.save_dataset_bin(src, x, layout=layout, checksum=False)
    for algo in ("data", "speculative"):
        n = st.eval_file(nodes, src, dst, st.GpuGeom(algo=algo), width=width)
        assert n == len(x)
        assert os.path.getsize(dst) == 32 + n * width
        assert np.array_equal(st.load_labels_bin(dst), want), (layout, width, algo)


def test_eval_file_errors(cuda, co, tmp_path):
    nodes = co.gen_tree(11, 16, 19, 7, 1)
    src = str(tmp_path / "d.strec")
    st.save_dataset_bin(src, co.gen_dataset(100, 8, 2))  # arity 8 < max attribute 18
    with pytest.raises(ArgumentError):
        st.eval_file(nodes, src, str(tmp_path / "l.stlab"))
    big = np.array([(0, np.inf, 0, 300)], dtype=st.NODE_DTYPE)  # class 300 does not fit u8
    st.save_dataset_bin(src, co.gen_dataset(10, 2, 2))
    with pytest.raises(ArgumentError):
        st.eval_file(big, src, str(tmp_path / "l.stlab"), width=1)
    empty = str(tmp_path / "e.strec")
    st.save_dataset_bin(empty, np.zeros((0, 19), np.float32))
    assert st.eval_file(nodes, empty, str(tmp_path / "e.stlab")) == 0
    assert st.load_labels_bin(str(tmp_path / "e.stlab")).size == 0


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        pytest.skip("oracle/_ref/spectree_b200_cli not built (needs /root/reference at build time)")
    return CLI


def test_cli_verify_bench_classify(cuda, co, cli, tmp_path):
    t, d = str(tmp_path / "t.json"), str(tmp_path / "d.strec")
    r = subprocess.run([cli, "gen", "--depth", "12", "--leaves", "2048", "--arity", "8", "--classes", "8",
                        "--seed", "301", "--records", "300000", "--data-seed", "302",
                        "--out-tree", t, "--out-data", d], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([cli, "verify", "--tree", t, "--data", d, "--strategy", "serial",
                        "--strategy", "gpu-data", "--strategy", "gpu-spec"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu-data: OK (300000 records)" in r.stdout and "gpu-spec: OK" in r.stdout
    r = subprocess.run([cli, "bench", "--tree", t, "--data", d, "--strategy", "serial", "--strategy", "gpu-data",
                        "--strategy", "gpu-spec", "--iterations", "5", "--warmup", "1", "--format", "json"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    rep = json.loads(r.stdout)
    assert rep["version"] == 1 and rep["verification"]["all_match"]
    names = [s["name"] for s in rep["strategies"]]
    assert names == ["serial", "gpu-data", "gpu-spec"]
    g = rep["strategies"][1]
    assert g["inner_us"]["mean_us"] > 0 and g["alloc_us"]["iterations"] == 5 and g["gpu"]["h2d_mean_us"] > 0
    lab = str(tmp_path / "l.stlab")
    r = subprocess.run([cli, "classify", "--tree", t, "--data", d, "--out", lab, "--width", "1"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    nodes = co.gen_tree(12, 2048, 8, 8, 301)
    assert np.array_equal(st.load_labels_bin(lab), co.eval_serial(nodes, co.gen_dataset(300000, 8, 302)))
    r = subprocess.run([cli, "verify", "--tree", t, "--data", d, "--strategy", "gpu-bogus"],
                       capture_output=True, text=True)
    assert r.returncode == 2


@pytest.mark.parametrize("slots", [1, 3, 7])
def test_spec_ring_shallow_ring_stress(cuda, co, slots):
    """k_spec_ring with a ring shallower than the warp count: tickets run up to
    several generations ahead of a slow warp on a deep record (skewed depth-24
    tree), which a parity-only slot wait would mistake for a completed refill.
    Labels must stay exact for any ring depth."""
    import torch

    nodes = co.gen_tree(24, 256, 32, 8, 201)
    x = co.gen_dataset(400_000, 32, 202)
    want = co.eval_serial(nodes, x)
    xd = torch.from_numpy(x).cuda()
    for sr, var in ((1, ()), (2, ()), (2, ("spec_branch",)), (2, ("spec_select",)), (2, ("spec_fixed",)), (1, ())):
        out = torch.empty(len(x), dtype=torch.int32, device="cuda")
        st.eval_device(nodes, xd, out, st.GpuGeom(algo="speculative", pipeline=2, samples_per_thread=sr,
                                                  ring_slots=slots, variant=var))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want)


def _c_eval(tree, buf, m, a, ld, layout, timed=False):
    """st_eval / st_eval_timed straight through the C ABI on a host buffer."""
    import ctypes as C
    from paper_1111_1373_b200 import _lib
    L = _lib.load()
    out = np.empty(m, np.uint32)
    g = st.GpuGeom().to_c()
    h = tree.handle()
    ptr = C.c_void_p(buf.ctypes.data)
    lay = _lib.ST_LAYOUT_SOA if layout == "soa" else _lib.ST_LAYOUT_AOS
    if timed:
        t = _lib.st_timing()
        rc = L.st_eval_timed(h.h, ptr, m, a, ld, lay, C.byref(g), out.ctypes.data_as(C.c_void_p), C.byref(t))
    else:
        rc = L.st_eval(h.h, ptr, m, a, ld, lay, C.byref(g), out.ctypes.data_as(C.c_void_p), None)
    assert rc == 0, _lib.last_error()
    return out


def _host_layout_cases(co, timed):
    """Pageable host records packed into pinned staging by the host copy pool
    (several 64 MB chunks, ragged tail): dense / strided AoS, SoA with a
    leading dimension, unaligned base, and the same from pinned memory."""
    import torch
    nodes = co.gen_tree(10, 1000, 64, 8, 77)
    tree = st.EncodedTree(nodes)
    m, a = 600_001, 64  # 154 MB: 3 chunks of 262,144 records
    x = co.gen_dataset(m, a, 78)
    want = co.eval_serial(nodes, x)
    assert np.array_equal(_c_eval(tree, x, m, a, a, "aos", timed), want)
    wide = np.zeros((m, a + 5), np.float32)
    wide[:, :a] = x
    assert np.array_equal(_c_eval(tree, wide, m, a, a + 5, "aos", timed), want)
    del wide
    soa = np.zeros((a, m + 7), np.float32)
    soa[:, :m] = x.T
    assert np.array_equal(_c_eval(tree, soa, m, a, m + 7, "soa", timed), want)
    del soa
    raw = np.zeros(m * a + 1, np.float32)
    raw[1:] = x.reshape(-1)
    assert np.array_equal(_c_eval(tree, raw[1:], m, a, a, "aos", timed), want)
    del raw
    pinned = torch.from_numpy(x).pin_memory().numpy()
    assert np.array_equal(_c_eval(tree, pinned, m, a, a, "aos", timed), want)


@pytest.mark.parametrize("timed", [False, True])
def test_pageable_staging_layouts(cuda, co, timed):
    _host_layout_cases(co, timed)


def test_pageable_staging_thread_counts(cuda, tmp_path):
    """The copy pool's split is exact for any worker count (the pool size is
    fixed per process: run in subprocesses)."""
    code = ("import sys; sys.path.insert(0, 'tests'); import oracle, test_gpu_flow as t; "
            "co = oracle.COracle(); t._host_layout_cases(co, False); t._host_layout_cases(co, True)")
    for n in ("1", "3"):
        env = dict(os.environ, ST_HOST_COPY_THREADS=n)
        r = subprocess.run(["python", "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, (n, r.stdout[-2000:], r.stderr[-2000:])
