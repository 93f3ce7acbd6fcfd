"""A/B library builds on the paper workload (tree(11,16,19,7,1) on 1024
copies of data(16384,19,2)), speculative and data (development aid):
    python tools/ab_paper_libs.py lib_a.so lib_b.so ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys
sys.path.insert(0, {root!r})
import paper_1111_1373_b200._lib as L
L.LIB_PATH = {lib!r}
import numpy as np, torch
import paper_1111_1373_b200 as st
tree = st.generate_synthetic_tree(11, 16, 19, 7, 1)
x = torch.from_numpy(np.tile(st.generate_synthetic_dataset(16384, 19, 2), (1024, 1))).cuda()
lab = torch.empty(len(x), dtype=torch.int32, device="cuda")
out = {{}}
for algo in ("data", "speculative"):
    g = st.GpuGeom(algo=algo)
    ts = []
    for _ in range(5):
        st.eval_device(tree, x, lab, g)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            st.eval_device(tree, x, lab, g)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 20 * 1e3)
    out[algo] = (min(ts), sorted(ts)[2])
print("RESULT" + json.dumps(out))
'''
res = {}
for _ in range(2):
    for lib in sys.argv[1:]:
        p = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, lib=os.path.abspath(lib))],
                           capture_output=True, text=True)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")]
        if line:
            for k, v in json.loads(line[0][6:]).items():
                res.setdefault((os.path.basename(lib), k), []).append(v)
        else:
            print(lib, p.stderr[-500:])
for (lib, k), v in sorted(res.items()):
    print(lib, k, [tuple(round(t, 1) for t in x) for x in v], "us (min, median)")
