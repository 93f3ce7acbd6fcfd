"""Evaluators: the reference's evaluate API, executed by the sm_100a kernels.

Mirrors (names, config fields, validation messages, error classes):
  * ``eval_data_parallel`` + ``DataParallelConfig`` + ``validate_data_parallel``
    (core/include/spectree/eval_data_parallel.hpp:13-33, src :13-88)
  * ``eval_speculative`` / ``eval_speculative_basic`` + ``SpeculativeConfig`` +
    ``SpeculativeStats`` + ``validate_speculative``
    (core/include/spectree/eval_speculative.hpp:23-106, src :69-273)
  * ``check_attribute_range`` (eval_serial.cpp:10-17)

Everything evaluates on the GPU through the C ABI (include/spectree_b200.h).
The CPU geometry fields of the reference configs (workers, chunk, groups,
records_per_group, os_threads) are validated exactly as the reference does
and then have no effect, just as ``os_threads`` never changes results in the
reference (eval_data_parallel.hpp:26-30).  GPU geometry lives in ``GpuGeom``.
There is no CPU fallback: without the CUDA library or a device every call
raises.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import st_geom, st_stats, st_tree_info
from .dataset import Dataset
from .errors import ArgumentError, raise_for
from .tree import NODE_DTYPE, NO_CLASS, EncodedTree

_ALGOS = {"auto": _lib.ST_ALGO_AUTO, "data": _lib.ST_ALGO_DATA,
          "speculative": _lib.ST_ALGO_SPECULATIVE, "spec": _lib.ST_ALGO_SPECULATIVE}
_TREE_LOCS = {"auto": _lib.ST_TREE_AUTO, "shared": _lib.ST_TREE_SHARED,
              "constant": _lib.ST_TREE_CONSTANT, "global": _lib.ST_TREE_GLOBAL}
# st_geom.variant flags (spectree_b200.h st_variant): implementation variants
# the tuned defaults were measured against; labels never depend on them.
VARIANTS = {"no_fold": _lib.ST_VAR_NO_FOLD, "tree_loop": _lib.ST_VAR_TREE_LOOP,
            "spec_general": _lib.ST_VAR_SPEC_GENERAL, "spec_jump": _lib.ST_VAR_SPEC_JUMP,
            "spec_wide": _lib.ST_VAR_SPEC_WIDE, "spec_select": _lib.ST_VAR_SPEC_SELECT,
            "spec_pred": _lib.ST_VAR_SPEC_PRED, "spec_branch": _lib.ST_VAR_SPEC_BRANCH,
            "spec_fixed": _lib.ST_VAR_SPEC_FIXED, "spec_quad": _lib.ST_VAR_SPEC_QUAD}


def _check(rc: int) -> None:
    if rc:
        raise_for(rc, _lib.last_error())


@dataclass
class GpuGeom:
    """GPU geometry (st_geom).  Zero means "choose automatically"."""

    algo: str = "auto"
    tree_loc: str = "auto"          # data kernel: shared | constant | global
    samples_per_thread: int = 0     # data kernel ILP
    group_lanes: int = 0            # speculative lanes per record group (pow2 <= 32)
    window_levels: int = 0          # speculative window height
    reductions: int = 0             # 0 = fixed per-window doublings; k = check root every k
    blocks_per_sm: int = 0
    stages: int = 0                 # TMA record-pipeline stages per warp
    warps_per_cta: int = 0          # CTA width (warps)
    pipeline: int = 0               # 0 auto, 1 per-warp TMA ring, 2 CTA-shared ring (spec)
    record_regs: int = 0            # data, 8/16-attribute records: 0 auto (3 for 8), 1 registers, 2 shared tile, 3 transposed tile
    variant: tuple = ()             # names from VARIANTS (A/B implementation variants)
    ring_slots: int = 0             # speculative ring: cap on tile slots (stress tests)
    slot_records: int = 0           # speculative ring: records per slot / 32 (1 or 2)
    fold_min: int = 0               # data: fold trees with >= this many nodes (0 = 2047)
    pdl: int = 0                    # data: 0 auto, 1 early trigger, 2 at exit, 3 off
    forest_chains: int = 0          # forest: trees per lane at once (1-4)
    forest_slots: int = 0           # forest: tree ring slots

    def to_c(self) -> st_geom:
        g = st_geom()
        if self.algo not in _ALGOS:
            raise ArgumentError(f"unknown algorithm '{self.algo}'")
        if self.tree_loc not in _TREE_LOCS:
            raise ArgumentError(f"unknown tree location '{self.tree_loc}'")
        g.algo = _ALGOS[self.algo]
        g.tree_loc = _TREE_LOCS[self.tree_loc]
        g.samples_per_thread = self.samples_per_thread
        g.group_lanes = self.group_lanes
        g.window_levels = self.window_levels
        g.reductions = self.reductions
        g.blocks_per_sm = self.blocks_per_sm
        g.stages = self.stages
        g.warps_per_cta = self.warps_per_cta
        g.pipeline = self.pipeline
        g.record_regs = self.record_regs
        names = (self.variant,) if isinstance(self.variant, str) else tuple(self.variant)
        flags = 0
        for n in names:
            if n not in VARIANTS:
                raise ArgumentError(f"unknown variant '{n}' (known: {', '.join(sorted(VARIANTS))})")
            flags |= VARIANTS[n]
        g.variant = flags
        g.ring_slots = self.ring_slots
        g.slot_records = self.slot_records
        g.fold_min = self.fold_min
        g.pdl = self.pdl
        g.forest_chains = self.forest_chains
        g.forest_slots = self.forest_slots
        return g


class _TreeHandle:
    def __init__(self, nodes: np.ndarray):
        self.L = _lib.load()
        self.nodes = np.ascontiguousarray(nodes, dtype=NODE_DTYPE)
        self.h = C.c_void_p()
        _check(self.L.st_tree_create(self.nodes.ctypes.data_as(C.c_void_p), len(self.nodes),
                                     C.byref(self.h)))

    def info(self) -> st_tree_info:
        inf = st_tree_info()
        _check(self.L.st_tree_get_info(self.h, C.byref(inf)))
        return inf

    def __del__(self):
        try:
            if self.h:
                self.L.st_tree_destroy(self.h)
        except Exception:
            pass


def _as_tree(tree) -> EncodedTree:
    if isinstance(tree, EncodedTree):
        return tree
    return EncodedTree(tree)


def _as_data(dataset) -> Dataset:
    if isinstance(dataset, Dataset):
        return dataset
    return Dataset.from_array(dataset)


def check_attribute_range(tree: EncodedTree, dataset: Dataset) -> None:
    """eval_serial.cpp:10-17 -- before any work."""
    if tree.max_attribute() >= dataset.arity():
        raise ArgumentError(f"tree reads attribute {tree.max_attribute()} but records have "
                            f"arity {dataset.arity()}")


def _u32_out(out, m, what="out"):
    if out is None:
        return np.empty(m, dtype=np.uint32)
    if out.dtype != np.uint32 or out.size != m or not out.flags.c_contiguous:
        raise ArgumentError(f"{what} must be a contiguous uint32 array of one entry per record")
    return out


def traversal_depths(tree, dataset, geom: Optional[GpuGeom] = None,
                     labels_out: Optional[np.ndarray] = None) -> np.ndarray:
    """Per-record traversal depth -- edges from the root to the leaf reached
    (reference traversal_depths, eval_serial.cpp:77-105) -- computed on the GPU
    by the data kernel beside the labels (``st_eval_depths``)."""
    tree = _as_tree(tree)
    dataset = _as_data(dataset)
    check_attribute_range(tree, dataset)
    m = dataset.count()
    depths = np.empty(m, dtype=np.uint32)
    labels = _u32_out(labels_out, m, "labels_out")
    g = (geom or GpuGeom()).to_c()
    x = dataset.values()
    L = _lib.load()
    h = tree.handle()
    _check(L.st_eval_depths(h.h, x.ctypes.data_as(C.c_void_p) if m else None, m, dataset.arity(), 0,
                            _lib.ST_LAYOUT_AOS, C.byref(g), labels.ctypes.data_as(C.c_void_p) if m else None,
                            depths.ctypes.data_as(C.c_void_p) if m else None))
    return depths


def mean_traversal_depth(tree, dataset, geom: Optional[GpuGeom] = None) -> float:
    """eval_serial.cpp:99-110: mean of traversal_depths; an empty dataset
    raises ArgumentError, as in the reference."""
    dataset = _as_data(dataset)
    if dataset.count() == 0:
        raise ArgumentError("mean traversal depth of an empty dataset")
    d = traversal_depths(tree, dataset, geom)
    return float(d.sum(dtype=np.uint64)) / len(d)


def eval_gpu(tree, dataset, geom: Optional[GpuGeom] = None, stats: Optional["SpeculativeStats"] = None,
             layout: str = "aos", out: Optional[np.ndarray] = None) -> np.ndarray:
    """Host-buffer evaluation through ``st_eval`` (H2D + kernel + D2H).
    ``out`` may be a preallocated (e.g. pinned) uint32 buffer of m labels."""
    tree = _as_tree(tree)
    dataset = _as_data(dataset)
    check_attribute_range(tree, dataset)
    m = dataset.count()
    out = _u32_out(out, m)
    g = (geom or GpuGeom()).to_c()
    x = dataset.values()
    if layout == "soa":
        x = np.ascontiguousarray(x.T)
        lay = _lib.ST_LAYOUT_SOA
    elif layout == "aos":
        lay = _lib.ST_LAYOUT_AOS
    else:
        raise ArgumentError(f"unknown layout '{layout}'")
    sp = None
    if stats is not None:
        stats.iterations = np.zeros(m, dtype=np.uint32)
        stats.doubling_steps = np.zeros(m, dtype=np.uint32)
        sp = st_stats(stats.iterations.ctypes.data_as(C.c_void_p),
                      stats.doubling_steps.ctypes.data_as(C.c_void_p))
    L = _lib.load()
    h = tree.handle()  # keep the native tree alive for the whole call
    _check(L.st_eval(h.h, x.ctypes.data_as(C.c_void_p) if m else None, m,
                     dataset.arity(), 0, lay, C.byref(g), out.ctypes.data_as(C.c_void_p) if m else None,
                     C.byref(sp) if sp is not None else None))
    if stats is not None:
        stats.barriers = int(m + int(stats.doubling_steps.sum(dtype=np.uint64)))
    return out


# --------------------------------------------------------------------------
# Data decomposition (Algorithm 1)
# --------------------------------------------------------------------------
@dataclass
class DataParallelConfig:
    """eval_data_parallel.hpp:13-19 (+ GPU geometry)."""

    workers: int = 1
    chunk: int = 1
    exact_fit: bool = False
    os_threads: int = 0
    gpu: GpuGeom = field(default_factory=GpuGeom)


def validate_data_parallel(config: DataParallelConfig, record_count: int) -> None:
    """eval_data_parallel.cpp:13-33."""
    if config.workers == 0:
        raise ArgumentError("data-parallel workers must be >= 1")
    if config.chunk == 0:
        raise ArgumentError("data-parallel chunk must be >= 1")
    capacity = int(config.workers) * int(config.chunk)
    if capacity < record_count:
        raise ArgumentError(f"workers * chunk = {capacity} leaves records unassigned (dataset has "
                            f"{record_count})")
    if config.exact_fit and capacity != record_count:
        raise ArgumentError(f"exact fit requires workers * chunk == {record_count}, got {capacity}")


def default_data_parallel(records: int, workers: int = 148) -> DataParallelConfig:
    """resolve_data (main.cpp:89-101): one even chunk per worker."""
    return DataParallelConfig(workers=workers, chunk=max(1, -(-records // workers)))


def eval_data_parallel(tree, dataset, config: Optional[DataParallelConfig] = None) -> np.ndarray:
    tree = _as_tree(tree)
    dataset = _as_data(dataset)
    if config is None:
        config = default_data_parallel(dataset.count())
    validate_data_parallel(config, dataset.count())
    check_attribute_range(tree, dataset)
    geom = GpuGeom(**{**config.gpu.__dict__, "algo": "data"})
    return eval_gpu(tree, dataset, geom)


# --------------------------------------------------------------------------
# Speculative decomposition (Algorithm 2)
# --------------------------------------------------------------------------
class ReductionMode(enum.Enum):
    """eval_speculative.hpp:23."""

    barrier_separated = 0
    compound_in_place = 1


@dataclass
class SpeculativeConfig:
    """eval_speculative.hpp:25-32 (+ GPU geometry)."""

    group_lanes: int = 0
    groups: int = 0
    records_per_group: int = 1
    reductions_per_iteration: int = 2
    mode: ReductionMode = ReductionMode.barrier_separated
    os_threads: int = 0
    gpu: GpuGeom = field(default_factory=GpuGeom)


@dataclass
class SpeculativeStats:
    """eval_speculative.hpp:73-77."""

    iterations: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    doubling_steps: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    barriers: int = 0


def validate_speculative(config: SpeculativeConfig, tree: EncodedTree, record_count: int,
                         basic_lanes: bool) -> None:
    """eval_speculative.cpp:69-107."""
    if config.group_lanes == 0:
        raise ArgumentError("speculative group_lanes must be >= 1")
    if basic_lanes:
        if config.group_lanes != tree.size():
            raise ArgumentError(f"all-lanes kernel requires group_lanes == {tree.size()} (one per "
                                f"node), got {config.group_lanes}")
    else:
        internal = (tree.size() - 1) // 2
        if config.group_lanes < internal:
            raise ArgumentError(f"mapped kernel requires group_lanes >= {internal} (one per "
                                f"internal node), got {config.group_lanes}")
    if config.groups == 0:
        raise ArgumentError("speculative groups must be >= 1")
    if config.records_per_group == 0:
        raise ArgumentError("speculative records_per_group must be >= 1")
    if config.reductions_per_iteration == 0:
        raise ArgumentError("reductions_per_iteration must be >= 1")
    capacity = int(config.groups) * int(config.records_per_group)
    if capacity < record_count:
        raise ArgumentError(f"groups * records_per_group = {capacity} leaves records unassigned "
                            f"(dataset has {record_count})")


def default_speculative(tree: EncodedTree, records: int, records_per_group: int = 32,
                        reductions: int = 2) -> SpeculativeConfig:
    """resolve_speculative (main.cpp:103-123): p = (N-1)/2, m = 32, k = 2."""
    return SpeculativeConfig(group_lanes=max(1, (tree.size() - 1) // 2),
                             records_per_group=records_per_group,
                             groups=max(1, -(-records // records_per_group)),
                             reductions_per_iteration=reductions)


def _spec_geom(tree: EncodedTree, config: SpeculativeConfig, stats) -> GpuGeom:
    g = GpuGeom(**{**config.gpu.__dict__, "algo": "speculative"})
    internal = len(tree.internal_indices())
    if g.group_lanes == 0 and internal <= 32:
        # mapped lanes in one warp-shuffle group: the paper's Proc. 5 shape
        gl = 1
        while gl < max(1, internal):
            gl *= 2
        g.group_lanes = gl
    if stats is not None and g.reductions == 0:
        # barrier-separated law: check the root after every k doublings
        g.reductions = config.reductions_per_iteration
    return g


def _run_speculative(tree, dataset, config, stats, basic):
    tree = _as_tree(tree)
    dataset = _as_data(dataset)
    if config is None:
        config = default_speculative(tree, dataset.count())
        if basic:
            config.group_lanes = tree.size()
            config.reductions_per_iteration = 1
    validate_speculative(config, tree, dataset.count(), basic)
    check_attribute_range(tree, dataset)
    geom = _spec_geom(tree, config, stats)
    if basic and stats is not None:
        geom.reductions = 1  # all-lanes kernel: one doubling per iteration (cpp:157-168)
    return eval_gpu(tree, dataset, geom, stats)


def eval_speculative(tree, dataset, config: Optional[SpeculativeConfig] = None,
                     stats: Optional[SpeculativeStats] = None) -> np.ndarray:
    """Mapped-lane speculative kernel (eval_speculative.cpp:267-273)."""
    return _run_speculative(tree, dataset, config, stats, basic=False)


def eval_speculative_basic(tree, dataset, config: Optional[SpeculativeConfig] = None,
                           stats: Optional[SpeculativeStats] = None) -> np.ndarray:
    """All-lanes variant (eval_speculative.cpp:261-266).  Leaves are fixpoints,
    so the GPU evaluates the internal lanes only; labels are identical."""
    return _run_speculative(tree, dataset, config, stats, basic=True)


# --------------------------------------------------------------------------
# Device-resident entry points (torch tensors; inputs already in HBM)
# --------------------------------------------------------------------------
def _stream_handle(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _device_records(x, layout: str):
    """(m, a, ld, st_layout) of a float32 CUDA tensor on the current device
    (AoS x is (m, a), SoA x is (a, m)); raises ArgumentError otherwise."""
    import torch

    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ArgumentError("expected a CUDA tensor of records")
    if x.dtype != torch.float32:
        raise ArgumentError(f"records must be float32, got {x.dtype}")
    if x.dim() != 2:
        raise ArgumentError(f"records must be a 2-D tensor, got shape {tuple(x.shape)}")
    if x.device.index != torch.cuda.current_device():
        raise ArgumentError(f"records live on {x.device}, the current device is "
                            f"cuda:{torch.cuda.current_device()}")
    # strides of size-1 dimensions carry no information (torch reports 1)
    if layout == "aos":
        m, a = x.shape
        ld = x.stride(0) if m > 1 else a
        if x.stride(1) != 1 and a > 1:
            raise ArgumentError("AoS tensor must have unit attribute stride")
        return m, a, ld, _lib.ST_LAYOUT_AOS
    if layout == "soa":
        a, m = x.shape
        ld = x.stride(0) if a > 1 else m
        if x.stride(1) != 1 and m > 1:
            raise ArgumentError("SoA tensor must have unit record stride")
        return m, a, ld, _lib.ST_LAYOUT_SOA
    raise ArgumentError(f"unknown layout '{layout}'")


def _device_u32(t, m: int, what: str, device) -> C.c_void_p:
    """Pointer of a CUDA tensor of >= m contiguous 4-byte integers on `device`."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ArgumentError(f"{what} must be a CUDA tensor")
    if t.dtype not in (torch.int32, torch.uint32):
        raise ArgumentError(f"{what} must be int32 or uint32, got {t.dtype}")
    if not t.is_contiguous():
        raise ArgumentError(f"{what} must be contiguous")
    if t.numel() < m:
        raise ArgumentError(f"{what} holds {t.numel()} elements, need {m}")
    if t.device != device:
        raise ArgumentError(f"{what} lives on {t.device}, the records on {device}")
    return C.c_void_p(t.data_ptr())


def eval_device(tree, x, labels, geom: Optional[GpuGeom] = None, layout: str = "aos",
                stream=None, stats=None) -> None:
    """Enqueue one evaluation of device tensor ``x`` into device tensor
    ``labels`` (uint32/int32, m elements) on ``stream``.  AoS x is (m, a);
    SoA x is (a, m); both float32 on the current device.  ``stats`` =
    (iterations, doubling_steps) tensors for the speculative counters.
    Asynchronous."""
    tree = _as_tree(tree)
    m, a, ld, lay = _device_records(x, layout)
    lp = _device_u32(labels, m, "labels", x.device)
    g = (geom or GpuGeom()).to_c()
    sp = None
    if stats is not None:
        sp = st_stats(_device_u32(stats[0], m, "stats[0] (iterations)", x.device),
                      _device_u32(stats[1], m, "stats[1] (doubling_steps)", x.device))
    L = _lib.load()
    h = tree.handle()
    _check(L.st_eval_device(h.h, C.c_void_p(x.data_ptr()), m, a, ld, lay, C.byref(g), lp,
                            C.byref(sp) if sp is not None else None, _stream_handle(stream)))


def eval_depths_device(tree, x, labels, depths, geom: Optional[GpuGeom] = None, layout: str = "aos",
                       stream=None) -> None:
    """Device-resident labels + traversal depths (``st_eval_depths_device``)."""
    tree = _as_tree(tree)
    m, a, ld, lay = _device_records(x, layout)
    lp = _device_u32(labels, m, "labels", x.device)
    dp = _device_u32(depths, m, "depths", x.device)
    g = (geom or GpuGeom()).to_c()
    L = _lib.load()
    h = tree.handle()
    _check(L.st_eval_depths_device(h.h, C.c_void_p(x.data_ptr()), m, a, ld, lay, C.byref(g), lp, dp,
                                   _stream_handle(stream)))


def eval_sharded(tree, dataset, devices: Sequence[int], geom: Optional[GpuGeom] = None) -> np.ndarray:
    """Sample-sharded evaluation over several local GPUs (st_eval_sharded)."""
    tree = _as_tree(tree)
    dataset = _as_data(dataset)
    check_attribute_range(tree, dataset)
    m = dataset.count()
    out = np.empty(m, dtype=np.uint32)
    devs = (C.c_int * len(devices))(*devices)
    g = (geom or GpuGeom()).to_c()
    x = dataset.values()
    L = _lib.load()
    h = tree.handle()
    _check(L.st_eval_sharded(h.h, x.ctypes.data_as(C.c_void_p) if m else None, m,
                             dataset.arity(), 0, _lib.ST_LAYOUT_AOS, C.byref(g), devs, len(devices),
                             out.ctypes.data_as(C.c_void_p) if m else None))
    return out


def last_launch_count() -> int:
    return int(_lib.load().st_last_launch_count())


def tree_info(tree) -> dict:
    inf = _as_tree(tree).handle().info()
    return {k: getattr(inf, k) for k, _ in st_tree_info._fields_}


# --------------------------------------------------------------------------
# Random forest
# --------------------------------------------------------------------------
class Forest:
    """T trees with a per-record majority vote (smallest class id on ties)."""

    def __init__(self, trees: Sequence, n_classes: int):
        self.trees = [_as_tree(t) for t in trees]
        self.n_classes = int(n_classes)
        self.max_attribute = max(t.max_attribute() for t in self.trees) if self.trees else 0
        self.L = _lib.load()
        arrs = [t.nodes() for t in self.trees]
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        sizes = (C.c_uint32 * len(arrs))(*[len(a) for a in arrs])
        self.h = C.c_void_p()
        _check(self.L.st_forest_create(ptrs, sizes, len(arrs), self.n_classes, C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                self.L.st_forest_destroy(self.h)
        except Exception:
            pass


def eval_forest(forest: Forest, dataset, geom: Optional[GpuGeom] = None,
                out: Optional[np.ndarray] = None) -> np.ndarray:
    dataset = _as_data(dataset)
    if forest.max_attribute >= dataset.arity():
        raise ArgumentError(f"tree reads attribute {forest.max_attribute} but records have arity "
                            f"{dataset.arity()}")
    m = dataset.count()
    out = _u32_out(out, m)
    g = (geom or GpuGeom()).to_c()
    x = dataset.values()
    _check(forest.L.st_forest_eval(forest.h, x.ctypes.data_as(C.c_void_p) if m else None, m,
                                   dataset.arity(), 0, _lib.ST_LAYOUT_AOS, C.byref(g),
                                   out.ctypes.data_as(C.c_void_p) if m else None))
    return out


def eval_forest_device(forest: Forest, x, labels, geom: Optional[GpuGeom] = None, stream=None) -> None:
    """Enqueue the forest vote of AoS float32 device tensor ``x`` (m, a) into
    ``labels`` (m int32/uint32) on ``stream``."""
    m, a, ld, lay = _device_records(x, "aos")
    lp = _device_u32(labels, m, "labels", x.device)
    g = (geom or GpuGeom()).to_c()
    _check(forest.L.st_forest_eval_device(forest.h, C.c_void_p(x.data_ptr()), m, a, ld, lay, C.byref(g),
                                          lp, _stream_handle(stream)))
