import os, sys
sys.path.insert(0, os.getcwd())
import paper_1111_1373_b200 as st, torch
trees = [st.generate_synthetic_tree(12, 1024, 64, 8, 401 + t) for t in range(128)]
x = st.generate_synthetic_dataset(int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 64, 499)
f = st.Forest(trees, 8)
xd = torch.from_numpy(x).cuda(); lab = torch.empty(len(x), dtype=torch.int32, device="cuda")
for _ in range(2):
    st.eval_forest_device(f, xd, lab)
torch.cuda.synchronize()
print("ok")
