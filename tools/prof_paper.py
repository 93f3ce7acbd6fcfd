"""The paper's workload at scale -- tree(11,16,19,7,1) on 256 copies of
data(16384,19,2) x 4 (16.8 M records) -- a few launches of one algorithm, as
an ncu target:  ncu -k regex:k_spec -s 2 -c 1 python tools/prof_paper.py speculative"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_1373_b200 as st  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "speculative"
tree = st.generate_synthetic_tree(11, 16, 19, 7, 1)
x = np.tile(st.generate_synthetic_dataset(16384, 19, 2), (4 * 256, 1))
xd = torch.from_numpy(x).cuda()
out = torch.empty(len(x), dtype=torch.int32, device="cuda")
for _ in range(4):
    st.eval_device(tree, xd, out, st.GpuGeom(algo=algo))
torch.cuda.synchronize()
print("paper x256", algo, len(x))
