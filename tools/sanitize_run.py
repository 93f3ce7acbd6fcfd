"""One small launch of every kernel family (data: shared/global/constant tree,
S = 1/2/4; speculative: ring (lane triples, 4-lane groups, stream loops),
one-window ballot / jump, per-warp, EXACT shfl, EXACT CTA; forest; with
--frames the resident frame stream), labels
checked against the C oracle -- the target for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (checker only)
import paper_1111_1373_b200 as st  # noqa: E402

co = oracle.COracle()
args = [a for a in sys.argv[1:] if not a.startswith("--")]
m = int(args[0]) if args else 20_000
bad = 0
if "--frames" in sys.argv:
    # the resident frame stream: 3 frames through a 2-slot ring, labels vs the oracle
    nodes = co.gen_tree(12, 2048, 8, 8, 301)
    frames = [co.gen_dataset(7680, 8, 50 + k) for k in range(3)]  # whole 128- and 120-record tiles
    for algo in ("data", "speculative"):
        print("frames", algo, flush=True)
        with st.FrameStream(nodes, 7680, 8, ring=2, geom=st.GpuGeom(algo=algo), idle_timeout_ms=1200000) as fs:
            seqs = []
            for k, f in enumerate(frames):
                if len(seqs) == 2:
                    s0 = seqs.pop(0)
                    bad += not np.array_equal(fs.pop(s0), co.eval_serial(nodes, frames[s0]))
                seqs.append(fs.push(f))
            for s0 in seqs:
                bad += not np.array_equal(fs.pop(s0), co.eval_serial(nodes, frames[s0]))
    print("sanitize_run frames:", "ok" if bad == 0 else f"{bad} mismatches")
    sys.exit(1 if bad else 0)
cases = [((24, 256, 32, 8, 201), 32), ((12, 2048, 8, 8, 301), 8), ((10, 1024, 16, 8, 101), 16),
         ((11, 16, 19, 7, 1), 19), ((12, 1024, 64, 8, 401), 64)]
for targs, a in cases:
    nodes = co.gen_tree(*targs)
    x = co.gen_dataset(m + 7, a, 5)  # ragged tail tile
    want = co.eval_serial(nodes, x)
    xd = torch.from_numpy(x).cuda()
    geoms = [st.GpuGeom(algo="data", tree_loc=tl, samples_per_thread=s)
             for tl in ("shared", "global", "constant") for s in (1, 2, 4)]
    geoms += [st.GpuGeom(algo="data", record_regs=1, samples_per_thread=s) for s in (1, 2)]
    geoms += [st.GpuGeom(algo="data", record_regs=3, samples_per_thread=s, stages=n) for s in (1, 4) for n in (1, 2)]
    geoms += [st.GpuGeom(algo="speculative", pipeline=p, group_lanes=g) for p in (1, 2) for g in (0, 2, 8)]
    geoms += [st.GpuGeom(algo="speculative", samples_per_thread=2, group_lanes=g) for g in (2, 4)]
    # the fixed-trip loop on lane triples (default) and 4-lane groups, the round-2 stream loops
    geoms += [st.GpuGeom(algo="speculative", variant=v)
              for v in ((), ("spec_quad",), ("spec_pred",), ("spec_branch",))]
    for g in geoms:
        out = torch.empty(len(x), dtype=torch.int32, device="cuda")
        st.eval_device(nodes, xd, out, g)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        if not np.array_equal(got, want):
            bad += 1
            print("MISMATCH", targs, g)
    # one-window trees: the pointer-jumping variant of the one-window path too
    out = torch.empty(len(x), dtype=torch.int32, device="cuda")
    st.eval_device(nodes, xd, out, st.GpuGeom(algo="speculative", variant=("spec_jump",)))
    torch.cuda.synchronize()
    if not np.array_equal(out.cpu().numpy().view(np.uint32), want):
        bad += 1
        print("MISMATCH one-window jump", targs)
    it = torch.empty(len(x), dtype=torch.int32, device="cuda")
    sp = torch.empty(len(x), dtype=torch.int32, device="cuda")
    out = torch.empty(len(x), dtype=torch.int32, device="cuda")
    st.eval_device(nodes, xd, out, st.GpuGeom(algo="speculative", reductions=2), stats=(it, sp))
    torch.cuda.synchronize()
    if not np.array_equal(out.cpu().numpy().view(np.uint32), want):
        bad += 1
        print("MISMATCH exact", targs)
trees = [co.gen_tree(10, 512, 64, 8, 401 + t) for t in range(6)]
x = co.gen_dataset(m + 5, 64, 9)
f = st.Forest(trees, 8)
out = torch.empty(len(x), dtype=torch.int32, device="cuda")
st.eval_forest_device(f, torch.from_numpy(x).cuda(), out)
torch.cuda.synchronize()
if not np.array_equal(out.cpu().numpy().view(np.uint32), co.eval_forest(trees, x, 8)):
    bad += 1
    print("MISMATCH forest")
print("sanitize_run:", "ok" if bad == 0 else f"{bad} mismatches")
sys.exit(1 if bad else 0)
