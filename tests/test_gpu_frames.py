"""Resident frame stream (st_frames_*): every frame's labels equal the
oracle's eval_serial on the same records, through the host push/pop path and
the stream-ordered device-producer protocol; ring reuse, ordering rules,
argument errors and the idle-timeout stop.

No device-wide synchronisation while a stream is open (it would wait for the
resident grid): these tests synchronise streams only."""
import time

import numpy as np
import pytest
import torch

import paper_1111_1373_b200 as st

pytestmark = pytest.mark.gpu


def _frames(co, n, records, a, seed):
    return [co.gen_dataset(records, a, seed + k, gaussian=(k % 2 == 1)) for k in range(n)]


@pytest.mark.parametrize("depth,leaves,a,records,ring,geom", [
    (12, 2048, 8, 65536, 3, None),                         # C3-shaped tree, transposed tiles
    (10, 1024, 16, 32768, 1, None),                        # C1-shaped, one slot
    (24, 256, 32, 16384, 2, None),                         # skewed C2-shaped tree
    (12, 2048, 8, 32768, 2, st.GpuGeom(algo="data", record_regs=1)),   # records from registers
    (16, 4096, 16, 16384, 4, st.GpuGeom(algo="data", tree_loc="global")),
])
def test_frames_push_pop(cuda, co, depth, leaves, a, records, ring, geom):
    nodes = co.gen_tree(depth, leaves, a, 8, 700 + depth)
    frames = _frames(co, 2 * ring + 3, records, a, 900 + a)
    want = [co.eval_serial(nodes, f) for f in frames]
    with st.FrameStream(nodes, records, a, ring=ring, geom=geom, idle_timeout_ms=20000) as fs:
        pending = []
        for k, f in enumerate(frames):
            if len(pending) == ring:  # pop before publishing frame seq + ring
                s = pending.pop(0)
                assert np.array_equal(fs.pop(s), want[s]), (s, depth, a)
            pending.append(fs.push(f))
            assert pending[-1] == k
        for s in pending:
            assert np.array_equal(fs.pop(s), want[s]), (s, depth, a)
        assert fs.status() == (len(frames), False)


@pytest.mark.parametrize("depth,leaves,a,records,ring,geom", [
    (12, 2048, 8, 120 * 500, 3, None),                     # C3-shaped tree: lane triples, 120-record slots
    (12, 4096, 16, 80 * 400, 2, None),                     # lane triples, 80-record slots
    (24, 256, 32, 32 * 1000, 2, None),                     # skewed tree, 4-lane groups (early exit)
    (12, 2048, 8, 80 * 300, 1, st.GpuGeom(algo="speculative", slot_records=2)),
    (14, 4096, 8, 32 * 900, 4, st.GpuGeom(algo="speculative", variant=("spec_quad",))),
])
def test_frames_speculative(cuda, co, depth, leaves, a, records, ring, geom):
    """The speculative ring as a resident frame stream (deferred slot
    hand-over across frame boundaries): every frame = the oracle."""
    g = geom or st.GpuGeom(algo="speculative")
    nodes = co.gen_tree(depth, leaves, a, 8, 800 + depth)
    frames = _frames(co, 2 * ring + 3, records, a, 950 + a)
    want = [co.eval_serial(nodes, f) for f in frames]
    with st.FrameStream(nodes, records, a, ring=ring, geom=g, idle_timeout_ms=20000) as fs:
        pending = []
        for k, f in enumerate(frames):
            if len(pending) == ring:
                s0 = pending.pop(0)
                assert np.array_equal(fs.pop(s0), want[s0]), (s0, depth, a)
            pending.append(fs.push(f))
        for s0 in pending:
            assert np.array_equal(fs.pop(s0), want[s0]), (s0, depth, a)
    with pytest.raises(st.ArgumentError):  # one-window trees (<= 32 internal nodes) have no window loop
        st.FrameStream(co.gen_tree(5, 16, a, 8, 1), records, a, geom=g)


def test_frames_back_to_back_streams(cuda, co):
    """Streams opened one after another over a plain node array, the
    variable rebound while the next grid is resident: close() drops the
    tree, so its cudaFree does not stall behind the next stream (which would
    run into the idle timeout)."""
    nodes = co.gen_tree(12, 2048, 8, 8, 301)
    for algo in ("data", "speculative", "data", "speculative"):
        rec = 128 * 64 if algo == "data" else 120 * 64
        frames = _frames(co, 3, rec, 8, 77)
        with st.FrameStream(nodes, rec, 8, ring=2, geom=st.GpuGeom(algo=algo), idle_timeout_ms=5000) as fs:
            s0, s1 = fs.push(frames[0]), fs.push(frames[1])
            assert np.array_equal(fs.pop(s0), co.eval_serial(nodes, frames[0])), algo
            s2 = fs.push(frames[2])
            assert np.array_equal(fs.pop(s1), co.eval_serial(nodes, frames[1])), algo
            assert np.array_equal(fs.pop(s2), co.eval_serial(nodes, frames[2])), algo


def test_frames_device_producer(cuda, co):
    """Stream-ordered protocol: a torch stream writes each frame into its
    slot, publishes it; another stream waits for the labels and copies them."""
    records, a, ring, n = 65536, 8, 3, 10
    nodes = co.gen_tree(12, 2048, a, 8, 301)
    frames = _frames(co, n, records, a, 302)
    want = [co.eval_serial(nodes, f) for f in frames]
    src = [torch.from_numpy(f).to(cuda) for f in frames]  # allocated before the stream opens
    outs = [torch.empty(records, dtype=torch.int32, device=cuda) for _ in range(n)]
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    # max_ctas leaves SMs free for work beside the resident grid
    with st.FrameStream(nodes, records, a, ring=ring, max_ctas=120, idle_timeout_ms=20000) as fs:
        for k in range(n):
            x, lab = fs.slot(k)
            fs.acquire(k, prod)
            with torch.cuda.stream(prod):
                x.copy_(src[k], non_blocking=True)
            fs.publish(k, prod)
            fs.wait(k, cons)
            with torch.cuda.stream(cons):
                outs[k].copy_(lab, non_blocking=True)
            # the slot is reused by frame k + ring: the copy-out must precede
            # that frame's records (the producer stream waits on the consumer)
            prod.wait_stream(cons)
        for strm in (cons, prod):
            t0 = time.time()
            while not strm.query():  # a deadline instead of a blocking synchronize
                assert time.time() - t0 < 30, "frame stream did not complete"
                time.sleep(1e-4)
    for k in range(n):
        assert np.array_equal(outs[k].cpu().numpy().view(np.uint32), want[k]), k


def test_frames_rules(cuda, co):
    nodes = co.gen_tree(10, 1024, 16, 8, 101)
    with pytest.raises(st.ArgumentError):
        st.FrameStream(nodes, 1000, 16)                    # not whole tiles
    with pytest.raises(st.ArgumentError):
        st.FrameStream(nodes, 4096, 19)                    # arity without row-local tiles
    with pytest.raises(st.ArgumentError):
        st.FrameStream(nodes, 4096, 8)                     # tree reads attribute >= 8
    with pytest.raises(st.ArgumentError):
        st.FrameStream(nodes, 4096, 16, ring=0)
    x = co.gen_dataset(4096, 16, 5)
    want = co.eval_serial(nodes, x)
    with st.FrameStream(nodes, 4096, 16, ring=2, idle_timeout_ms=20000) as fs:
        with pytest.raises(st.ArgumentError):
            fs.pop(0)                                      # not published
        for _ in range(3):
            fs.push(x)
        with pytest.raises(st.ArgumentError):
            fs.publish(1)                                  # already published
        with pytest.raises(st.ArgumentError):
            fs.pop(0)                                      # overwritten by frame 2
        assert np.array_equal(fs.pop(2), want)
    with pytest.raises(st.ArgumentError):
        fs.push(x)                                         # closed


def test_frames_idle_timeout(cuda, co):
    """A resident grid that sees no frame for idle_timeout_ms stops itself;
    the stream then reports it and refuses to hang."""
    nodes = co.gen_tree(10, 1024, 16, 8, 101)
    x = co.gen_dataset(4096, 16, 5)
    fs = st.FrameStream(nodes, 4096, 16, ring=2, idle_timeout_ms=200)
    try:
        time.sleep(0.8)
        assert fs.status()[1] is True
        seq = fs.push(x)
        with pytest.raises(st.CudaError):
            fs.pop(seq)
    finally:
        fs.close()
    # the device is usable afterwards
    out = st.eval_gpu(nodes, x, st.GpuGeom(algo="data"))
    assert np.array_equal(out, co.eval_serial(nodes, x))
