"""A/B several builds of the library on one box (development aid): every
build runs in its own subprocess, rounds alternate between builds.

    python tools/ab_libs.py W1,W2 ALGO lib_a.so lib_b.so ... [--rounds=3] [--geom='dict(...)']

Prints, per workload and build, the CUDA-event us per launch (min, median)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
sys.path.insert(0, {root!r})
import paper_1111_1373_b200._lib as L
L.LIB_PATH = {lib!r}
import torch
import bench
import paper_1111_1373_b200 as st
out = {{}}
for name in {names!r}:
    w = bench.WORKLOADS[name]
    tree = st.generate_synthetic_tree(*w["tree"])
    x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
    lab = torch.empty(w["m"], dtype=torch.int32, device="cuda")
    g = st.GpuGeom(algo={algo!r}, **{geom})
    st.eval_device(tree, x, lab, g)
    torch.cuda.synchronize()
    want = bench.golden_labels(w, 0)
    assert want is None or st.fnv1a64(lab.cpu().numpy()) == want, name
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            st.eval_device(tree, x, lab, g)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 20 * 1e3)
    out[name] = ts
print("RESULT" + json.dumps(out))
'''


def main():
    names = sys.argv[1].split(",")
    algo = sys.argv[2]
    libs = [a for a in sys.argv[3:] if not a.startswith("--")]
    rounds = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--rounds=")), 3))
    geom = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--geom=")), "dict()")
    res = {lib: {n: [] for n in names} for lib in libs}
    for _ in range(rounds):
        for lib in libs:
            code = CHILD.format(root=ROOT, lib=os.path.abspath(lib), names=names, algo=algo, geom=geom)
            p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")]
            if not line:
                print(lib, "failed:", p.stderr[-800:], flush=True)
                continue
            for n, ts in json.loads(line[0][6:]).items():
                res[lib][n] += ts
    for n in names:
        print(n, {os.path.basename(lib): (round(min(v[n]), 2), round(sorted(v[n])[len(v[n]) // 2], 2))
                  for lib, v in res.items() if v[n]}, "us (min, median)", flush=True)


if __name__ == "__main__":
    main()
