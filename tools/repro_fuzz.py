import sys, os, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle, paper_1111_1373_b200 as st, support
from paper_1111_1373_b200 import _lib
co = oracle.COracle()
DG = [st.GpuGeom(algo="data"), st.GpuGeom(algo="data", samples_per_thread=1), st.GpuGeom(algo="data", tree_loc="global"), st.GpuGeom(algo="data", tree_loc="constant")]
SG = [st.GpuGeom(algo="speculative"), st.GpuGeom(algo="speculative", group_lanes=4), st.GpuGeom(algo="speculative", group_lanes=8), st.GpuGeom(algo="speculative", group_lanes=32), st.GpuGeom(algo="speculative", group_lanes=16, window_levels=8), st.GpuGeom(algo="speculative", reductions=2)]
bad = 0
for seed in range(1, 60):
    spec = support.fuzz_shape(seed)
    nodes = co.gen_tree(*spec, seed)
    x = co.gen_dataset(1000, spec[2], seed + 5000, gaussian=(seed % 2 == 0))
    want = co.eval_serial(nodes, x)
    for gi, g in enumerate(DG + SG):
        try:
            got = st.eval_gpu(nodes, x, g)
            ok = np.array_equal(got, want)
        except Exception as e:
            ok = repr(e)
        if ok is not True:
            bad += 1
            if bad < 25: print("seed", seed, spec, "geom", gi, g, "->", ok, flush=True)
print("bad", bad)
