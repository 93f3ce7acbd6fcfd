"""TEST INFRASTRUCTURE ONLY: the CPU oracle for parity checks.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package.  The product path
(``paper_1111_1373_b200``) never does.

Two back ends:

* ``C`` -- ``_build/libst_oracle.so``, a plain-C restatement of the reference
  algorithms (``st_oracle.c``, every function cites reference file:line).
  Always built (``make -C oracle``); travels to the GPU box.
* ``Ref`` -- ``_ref/libspectree_ref.so``, the UNMODIFIED reference core compiled
  from /root/reference by ``oracle/Makefile`` plus the ``ref_shim.cpp`` C-ABI.
  Built here when /root/reference exists; the prebuilt .so travels to the box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB_PATH = os.path.join(HERE, "_build", "libst_oracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libspectree_ref.so")

NODE_DTYPE = np.dtype(
    [("attribute", "<u4"), ("threshold", "<f4"), ("child", "<u4"), ("class_id", "<u4")]
)
NO_CLASS = 0xFFFFFFFF

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build() -> None:
    """Build both oracle libraries (the reference one only if its sources exist)."""
    subprocess.run(["make", "-s", "-j4", "-C", HERE], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _nodes_ptr(nodes: np.ndarray):
    assert nodes.dtype == NODE_DTYPE and nodes.flags.c_contiguous
    return nodes.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class COracle:
    def __init__(self, path: str = C_LIB_PATH):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.or_gen_tree.restype = C.c_uint32
        L.or_gen_tree.argtypes = [C.c_uint32] * 4 + [C.c_uint64, C.POINTER(C.c_void_p)]
        L.or_free.argtypes = [C.c_void_p]
        L.or_gen_dataset.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, _f32p]
        L.or_shuffle_order.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        L.or_fnv1a.restype = C.c_uint64
        L.or_fnv1a.argtypes = [C.c_void_p, C.c_uint64]
        L.or_dataset_checksum.restype = C.c_uint64
        L.or_dataset_checksum.argtypes = [_f32p, C.c_uint64, C.c_uint32]
        L.or_max_attribute.restype = C.c_uint32
        L.or_max_attribute.argtypes = [C.c_void_p, C.c_uint32]
        for name in ("or_eval_serial", "or_traversal_depths"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [C.c_void_p, C.c_uint32, _f32p, C.c_uint64, C.c_uint32, _u32p]
        L.or_eval_speculative.restype = C.c_int
        L.or_eval_speculative.argtypes = [C.c_void_p, C.c_uint32, _f32p, C.c_uint64,
                                          C.c_uint32, C.c_uint32, _u32p, C.c_void_p,
                                          C.c_void_p]
        L.or_eval_forest.restype = C.c_int
        L.or_eval_forest.argtypes = [C.c_void_p, _u64p, C.c_uint32, _f32p, C.c_uint64,
                                     C.c_uint32, C.c_uint32, _u32p]
        self.L = L

    def gen_tree(self, depth, leaves, arity, classes, seed) -> np.ndarray:
        p = C.c_void_p()
        n = self.L.or_gen_tree(depth, leaves, arity, classes, seed, C.byref(p))
        if n == 0:
            raise OracleError(2, "infeasible synthetic tree shape")
        buf = (C.c_char * (16 * n)).from_address(p.value)
        out = np.frombuffer(bytes(buf), dtype=NODE_DTYPE).copy()
        self.L.or_free(p)
        return out

    def gen_dataset(self, count, arity, seed, gaussian=False) -> np.ndarray:
        out = np.empty(count * arity, dtype=np.float32)
        self.L.or_gen_dataset(count, arity, seed, int(bool(gaussian)), out)
        return out.reshape(count, arity)

    def shuffle_order(self, count, seed) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        self.L.or_shuffle_order(count, seed, out)
        return out

    def fnv1a(self, arr: np.ndarray) -> int:
        a = np.ascontiguousarray(arr)
        return int(self.L.or_fnv1a(a.ctypes.data_as(C.c_void_p), a.nbytes))

    def dataset_checksum(self, x: np.ndarray) -> int:
        x = np.ascontiguousarray(x, dtype=np.float32)
        return int(self.L.or_dataset_checksum(x.reshape(-1), x.shape[0], x.shape[1]))

    def max_attribute(self, nodes) -> int:
        return int(self.L.or_max_attribute(_nodes_ptr(nodes), len(nodes)))

    def _x(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        return x.reshape(-1), x.shape[0], x.shape[1]

    def eval_serial(self, nodes, x) -> np.ndarray:
        xf, m, a = self._x(x)
        out = np.empty(m, dtype=np.uint32)
        rc = self.L.or_eval_serial(_nodes_ptr(nodes), len(nodes), xf, m, a, out)
        if rc:
            raise OracleError(rc, "attribute out of range")
        return out

    def traversal_depths(self, nodes, x) -> np.ndarray:
        xf, m, a = self._x(x)
        out = np.empty(m, dtype=np.uint32)
        rc = self.L.or_traversal_depths(_nodes_ptr(nodes), len(nodes), xf, m, a, out)
        if rc:
            raise OracleError(rc, "attribute out of range")
        return out

    def eval_speculative(self, nodes, x, k=1):
        xf, m, a = self._x(x)
        out = np.empty(m, dtype=np.uint32)
        it = np.empty(m, dtype=np.uint32)
        st = np.empty(m, dtype=np.uint32)
        rc = self.L.or_eval_speculative(_nodes_ptr(nodes), len(nodes), xf, m, a, k, out,
                                        it.ctypes.data_as(C.c_void_p),
                                        st.ctypes.data_as(C.c_void_p))
        if rc:
            raise OracleError(rc, "bad speculative geometry or attribute range")
        return out, it, st

    def eval_forest(self, trees, x, n_classes) -> np.ndarray:
        nodes = np.ascontiguousarray(np.concatenate(trees))
        offs = np.zeros(len(trees) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(t) for t in trees])
        xf, m, a = self._x(x)
        out = np.empty(m, dtype=np.uint32)
        rc = self.L.or_eval_forest(_nodes_ptr(nodes), offs, len(trees), xf, m, a,
                                   n_classes, out)
        if rc:
            raise OracleError(rc, "bad forest")
        return out


# --------------------------------------------------------------------------
# compiled reference (oracle/_ref)
# --------------------------------------------------------------------------
def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


class RefOracle:
    """ctypes view of the reference core compiled by oracle/Makefile."""

    def __init__(self, path: str = REF_LIB_PATH):
        L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen_tree.restype = C.c_int
        L.ref_gen_tree.argtypes = [C.c_uint32] * 4 + [C.c_uint64, vp, C.c_uint32,
                                                      C.POINTER(C.c_uint32)]
        L.ref_gen_dataset.restype = C.c_int
        L.ref_gen_dataset.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, _f32p]
        L.ref_dataset_checksum.restype = C.c_uint64
        L.ref_dataset_checksum.argtypes = [_f32p, C.c_uint64, C.c_uint32]
        L.ref_tree_create.restype = C.c_int
        L.ref_tree_create.argtypes = [vp, C.c_uint32, C.POINTER(vp)]
        L.ref_tree_destroy.argtypes = [vp]
        for n in ("ref_tree_depth", "ref_tree_max_attribute", "ref_tree_leaf_count",
                  "ref_tree_validate"):
            getattr(L, n).restype = C.c_uint32
            getattr(L, n).argtypes = [vp]
        L.ref_data_create.restype = C.c_int
        L.ref_data_create.argtypes = [vp, C.c_uint64, C.c_uint32, C.POINTER(vp)]
        L.ref_data_destroy.argtypes = [vp]
        L.ref_eval_serial.restype = C.c_int
        L.ref_eval_serial.argtypes = [vp, vp, vp]
        L.ref_eval_data_parallel.restype = C.c_int
        L.ref_eval_data_parallel.argtypes = [vp, vp, C.c_uint32, C.c_uint32, C.c_int,
                                             C.c_uint32, vp]
        L.ref_eval_speculative.restype = C.c_int
        L.ref_eval_speculative.argtypes = [vp, vp] + [C.c_uint32] * 4 + [C.c_int, C.c_int,
                                                                         C.c_uint32, vp, vp,
                                                                         vp, vp]
        L.ref_traversal_depths.restype = C.c_int
        L.ref_traversal_depths.argtypes = [vp, vp, vp]
        L.ref_simulate_data_parallel.restype = C.c_int
        L.ref_simulate_data_parallel.argtypes = [vp, vp, C.c_uint32, C.c_int, C.c_uint32, C.c_uint32, vp]
        L.ref_simulate_speculative.restype = C.c_int
        L.ref_simulate_speculative.argtypes = [vp, vp, C.c_uint32, C.c_int] + [C.c_uint32] * 4 + [C.c_int, vp]
        L.ref_load_tree_json.restype = C.c_int
        L.ref_load_tree_json.argtypes = [C.c_char_p, vp, C.c_uint32, C.POINTER(C.c_uint32)]
        L.ref_tree_to_json.restype = C.c_uint64
        L.ref_tree_to_json.argtypes = [vp, C.c_uint32, C.c_char_p, C.c_uint64]
        self.L = L

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def gen_tree(self, depth, leaves, arity, classes, seed) -> np.ndarray:
        n = C.c_uint32()
        self._check(self.L.ref_gen_tree(depth, leaves, arity, classes, seed, None, 0,
                                        C.byref(n)))
        out = np.empty(n.value, dtype=NODE_DTYPE)
        self._check(self.L.ref_gen_tree(depth, leaves, arity, classes, seed,
                                        out.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
        return out

    def gen_dataset(self, count, arity, seed, gaussian=False) -> np.ndarray:
        out = np.empty(count * arity, dtype=np.float32)
        self._check(self.L.ref_gen_dataset(count, arity, seed, int(bool(gaussian)), out))
        return out.reshape(count, arity)

    def dataset_checksum(self, x) -> int:
        x = np.ascontiguousarray(x, dtype=np.float32)
        return int(self.L.ref_dataset_checksum(x.reshape(-1), x.shape[0], x.shape[1]))

    def tree(self, nodes) -> "RefTree":
        return RefTree(self, nodes)

    def data(self, x) -> "RefData":
        return RefData(self, x)

    def load_tree_json(self, text: str) -> np.ndarray:
        n = C.c_uint32()
        b = text.encode()
        self._check(self.L.ref_load_tree_json(b, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=NODE_DTYPE)
        self._check(self.L.ref_load_tree_json(b, out.ctypes.data_as(C.c_void_p), n.value,
                                              C.byref(n)))
        return out

    def tree_to_json(self, nodes) -> str:
        n = self.L.ref_tree_to_json(_nodes_ptr(nodes), len(nodes), None, 0)
        buf = C.create_string_buffer(n + 1)
        self.L.ref_tree_to_json(_nodes_ptr(nodes), len(nodes), buf, n + 1)
        return buf.value.decode()

    # one-shot conveniences
    def eval_serial(self, nodes, x):
        with self.tree(nodes) as t, self.data(x) as d:
            return t.eval_serial(d)


class RefTree:
    def __init__(self, ref: RefOracle, nodes: np.ndarray):
        self.ref = ref
        self.nodes = np.ascontiguousarray(nodes)
        self.h = C.c_void_p()
        ref._check(ref.L.ref_tree_create(_nodes_ptr(self.nodes), len(self.nodes),
                                         C.byref(self.h)))

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def close(self):
        if self.h:
            self.ref.L.ref_tree_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def depth(self):
        return int(self.ref.L.ref_tree_depth(self.h))

    @property
    def max_attribute(self):
        return int(self.ref.L.ref_tree_max_attribute(self.h))

    def validate_findings(self):
        return int(self.ref.L.ref_tree_validate(self.h))

    def eval_serial(self, d: "RefData") -> np.ndarray:
        out = np.empty(d.m, dtype=np.uint32)
        self.ref._check(self.ref.L.ref_eval_serial(self.h, d.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def eval_data_parallel(self, d, workers, chunk, exact_fit=False, os_threads=0):
        out = np.empty(d.m, dtype=np.uint32)
        self.ref._check(self.ref.L.ref_eval_data_parallel(
            self.h, d.h, workers, chunk, int(exact_fit), os_threads,
            out.ctypes.data_as(C.c_void_p)))
        return out

    def eval_speculative(self, d, group_lanes, groups, records_per_group, k=2,
                         compound=False, basic=False, os_threads=0):
        out = np.empty(d.m, dtype=np.uint32)
        it = np.empty(d.m, dtype=np.uint32)
        st = np.empty(d.m, dtype=np.uint32)
        bar = C.c_uint64()
        self.ref._check(self.ref.L.ref_eval_speculative(
            self.h, d.h, group_lanes, groups, records_per_group, k, int(compound),
            int(basic), os_threads, out.ctypes.data_as(C.c_void_p),
            it.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p), C.byref(bar)))
        return out, it, st, bar.value

    METRICS = ("divergent_branches", "serialized_passes", "barriers", "node_evals",
               "reduction_iterations", "lane_idle_slots")

    def simulate_data_parallel(self, d, workers, chunk, warp_width=32, half_warp=True) -> dict:
        """warp_sim.cpp:30-99 (reference lockstep model) -> ExecMetrics dict."""
        out = (C.c_uint64 * 6)()
        self.ref._check(self.ref.L.ref_simulate_data_parallel(self.h, d.h, warp_width, int(half_warp),
                                                              workers, chunk, out))
        return dict(zip(self.METRICS, [int(v) for v in out]))

    def simulate_speculative(self, d, group_lanes, groups, records_per_group, k=1, basic=False,
                             warp_width=32, half_warp=True) -> dict:
        """warp_sim.cpp:156-274 (reference lockstep model) -> ExecMetrics dict."""
        out = (C.c_uint64 * 6)()
        self.ref._check(self.ref.L.ref_simulate_speculative(self.h, d.h, warp_width, int(half_warp),
                                                            group_lanes, groups, records_per_group, k,
                                                            int(basic), out))
        return dict(zip(self.METRICS, [int(v) for v in out]))

    def traversal_depths(self, d):
        out = np.empty(d.m, dtype=np.uint32)
        self.ref._check(self.ref.L.ref_traversal_depths(self.h, d.h,
                                                        out.ctypes.data_as(C.c_void_p)))
        return out


class RefData:
    def __init__(self, ref: RefOracle, x: np.ndarray):
        self.ref = ref
        x = np.ascontiguousarray(x, dtype=np.float32)
        self.m, self.a = x.shape
        self.h = C.c_void_p()
        ref._check(ref.L.ref_data_create(x.ctypes.data_as(C.c_void_p), self.m, self.a,
                                         C.byref(self.h)))

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def close(self):
        if self.h:
            self.ref.L.ref_data_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
