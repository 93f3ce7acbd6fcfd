"""A/B two builds of the library on one box (development aid):
    python tools/ab_lib.py <lib.so> [workload]   -> CUDA-event ms for data / spec G=2,4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1111_1373_b200._lib as L  # noqa: E402

L.LIB_PATH = os.path.abspath(sys.argv[1])
import ctypes as C  # noqa: E402


class _Tolerant(C.CDLL):  # older builds lack newer symbols: give them dummies
    def __getattr__(self, name):
        try:
            return super().__getattr__(name)
        except AttributeError:
            f = lambda *a: 0  # noqa: E731
            setattr(self, name, f)
            return f


_orig = C.CDLL
C.CDLL = _Tolerant
L.load()
C.CDLL = _orig
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1111_1373_b200 as st  # noqa: E402

w = bench.WORKLOADS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
tree = st.generate_synthetic_tree(*w["tree"])
x = torch.from_numpy(st.generate_synthetic_dataset(w["m"], w["a"], w["seed"])).cuda()
out = torch.empty(w["m"], dtype=torch.int32, device="cuda")
for name, g in [("data", st.GpuGeom(algo="data")), ("spec-G2", st.GpuGeom(algo="speculative", group_lanes=2)),
                ("spec-G4", st.GpuGeom(algo="speculative", group_lanes=4))]:
    ts = []
    for rep in range(3):
        for _ in range(3):
            st.eval_device(tree, x, out, g)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            st.eval_device(tree, x, out, g)
        b.record()
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b) / 20, 4))
    ok = st.fnv1a64(out.cpu().numpy()) == w["labels_fnv"]
    print(os.path.basename(sys.argv[1]), name, ts, "labels_ok", ok, flush=True)
