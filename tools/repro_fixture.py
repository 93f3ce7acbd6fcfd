import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1111_1373_b200 as st
g = np.load("tests/golden/ref_fuzz.npz")
seeds = [int(a) for a in sys.argv[1:]] or range(1, 61)
for seed in seeds:
    nodes = g[f"s{seed}_nodes"].view(st.NODE_DTYPE); x = g[f"s{seed}_x"]
    for algo in ("data", "speculative"):
        try:
            got = st.eval_gpu(nodes, x, st.GpuGeom(algo=algo))
            print(seed, algo, x.shape, "ok" if np.array_equal(got, g[f"s{seed}_labels"]) else "MISMATCH", flush=True)
        except Exception as e:
            print(seed, algo, x.shape, "ERR", e, flush=True); sys.exit(1)
