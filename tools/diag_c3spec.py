"""Diagnose: C3-tree speculative labels through the host pipeline vs the device path."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, paper_1111_1373_b200 as st
co = oracle.COracle()
nodes = co.gen_tree(12, 2048, 8, 8, 301)
x = co.gen_dataset(9_000_000, 8, 302)
want = co.eval_serial(nodes, x)
tree = st.EncodedTree(nodes)
def rep(tag, got, w):
    bad = np.nonzero(got != w)[0]
    print(tag, "mismatches", len(bad), "first", bad[:8].tolist(), "last", bad[-4:].tolist() if len(bad) else [],
          "chunks", sorted(set((bad // 2097152).tolist())) if len(bad) else [], flush=True)
for name, var in (("default", ()), ("fixed", ("spec_fixed",)), ("pred", ("spec_pred",)), ("branch", ("spec_branch",)), ("select", ("spec_select",))):
    g = st.GpuGeom(algo="speculative", variant=var)
    rep("host " + name, st.eval_gpu(nodes, x, g), want)
    for m in (2_073_600, 2_097_152, 9_000_000):
        xd = torch.from_numpy(x[:m]).cuda()
        out = torch.zeros(m, dtype=torch.int32, device="cuda")
        st.eval_device(tree, xd, out, g)
        torch.cuda.synchronize()
        rep(f"dev{m} " + name, out.cpu().numpy().view(np.uint32), want[:m])
# concurrent device launches on 3 streams
g = st.GpuGeom(algo="speculative")
ss = [torch.cuda.Stream() for _ in range(3)]
xs = [torch.from_numpy(x[i * 2097152:(i + 1) * 2097152]).cuda() for i in range(3)]
outs = [torch.zeros(2097152, dtype=torch.int32, device="cuda") for _ in range(3)]
for i in range(3):
    st.eval_device(tree, xs[i], outs[i], g, stream=ss[i])
torch.cuda.synchronize()
for i in range(3):
    rep(f"conc{i}", outs[i].cpu().numpy().view(np.uint32), want[i * 2097152:(i + 1) * 2097152])
