import os, sys, threading, traceback
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_1111_1373_b200 as st
import torch
torch.cuda.init()
print("mem", [x / 2**30 for x in torch.cuda.mem_get_info()])
tree = st.generate_synthetic_tree(10, 1024, 16, 8, 101)
xs = [st.generate_synthetic_dataset(20000, 16, s) for s in range(8)]
errs = []
def work(i):
    try:
        for g in (st.GpuGeom(algo="data"), st.GpuGeom(algo="speculative")):
            st.eval_gpu(tree, xs[i], g)
    except Exception as e:
        errs.append((i, repr(e)))
for fresh in (True, False):
    if fresh:
        tree = st.generate_synthetic_tree(10, 1024, 16, 8, 101)  # new handle, no device replica yet
    th = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    [t.start() for t in th]; [t.join() for t in th]
    print("fresh" if fresh else "warm", "errors:", errs[:3], flush=True)
    errs.clear()
