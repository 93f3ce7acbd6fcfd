"""A/B library builds on the C4 forest (development aid): each build in its
own process, rounds alternate; geometries as st_geom dicts.

    python tools/ab_forest_libs.py lib_a.so lib_b.so [--geoms='[dict(), dict(forest_chains=4)]']
"""
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
import torch
import paper_1111_1373_b200 as st
m = 8_000_000
trees = [st.generate_synthetic_tree(12, 1024, 64, 8, 401 + t) for t in range(128)]
x = torch.from_numpy(st.generate_synthetic_dataset(m, 64, 499)).cuda()
f = st.Forest(trees, 8)
lab = torch.empty(m, dtype=torch.int32, device="cuda")
out = {{}}
for gs in {geoms!r}:
    g = st.GpuGeom(**eval(gs))
    st.eval_forest_device(f, x, lab, g)
    torch.cuda.synchronize()
    ok = st.fnv1a64(lab.cpu().numpy()) == 0x1b2543c41e436ce0
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            st.eval_forest_device(f, x, lab, g)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 5)
    out[gs] = (min(ts), ok)
print("RESULT" + json.dumps(out))
'''


def main():
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    geoms = eval(next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--geoms=")), "['dict()']"))
    res = {}
    for _ in range(2):
        for lib in libs:
            code = CHILD.format(root=ROOT, lib=os.path.abspath(lib), geoms=geoms)
            p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")]
            if not line:
                print(lib, "failed:", p.stderr[-600:], flush=True)
                continue
            for g, (t, ok) in json.loads(line[0][6:]).items():
                k = (os.path.basename(lib), g)
                res[k] = min(res.get(k, (1e9, ok))[0], t), ok
    for (lib, g), (t, ok) in sorted(res.items()):
        print(f"{lib:28s} {g:50s} {t:.3f} ms ok={ok}", flush=True)


if __name__ == "__main__":
    main()
