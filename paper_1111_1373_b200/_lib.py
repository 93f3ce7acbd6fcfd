"""ctypes binding of the C ABI in include/spectree_b200.h.

The shared library is built in-tree (``__graft_entry__.build()`` /
``python -m paper_1111_1373_b200.build``).  There is no CPU fallback: if the
library is missing, importing the evaluators raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspectree_b200.so")

# st_status (spectree_b200.h)
ST_OK = 0
ST_ERR_ARGUMENT = 2
ST_ERR_IO = 3
ST_ERR_CUDA = 4
ST_ERR_NO_DEVICE = 5

ST_LAYOUT_AOS = 0
ST_LAYOUT_SOA = 1
ST_ALGO_AUTO = 0
ST_ALGO_DATA = 1
ST_ALGO_SPECULATIVE = 2
ST_TREE_AUTO = 0
ST_TREE_SHARED = 1
ST_TREE_CONSTANT = 2
ST_TREE_GLOBAL = 3


class st_geom(C.Structure):
    _fields_ = [
        ("algo", C.c_uint32),
        ("tree_loc", C.c_uint32),
        ("samples_per_thread", C.c_uint32),
        ("group_lanes", C.c_uint32),
        ("window_levels", C.c_uint32),
        ("reductions", C.c_uint32),
        ("blocks_per_sm", C.c_uint32),
        ("stages", C.c_uint32),
        ("warps_per_cta", C.c_uint32),
        ("pipeline", C.c_uint32),
        ("record_regs", C.c_uint32),
        ("variant", C.c_uint32),
        ("ring_slots", C.c_uint32),
        ("slot_records", C.c_uint32),
        ("fold_min", C.c_uint32),
        ("pdl", C.c_uint32),
        ("forest_chains", C.c_uint32),
        ("forest_slots", C.c_uint32),
        ("reserved", C.c_uint32 * 6),
    ]


# st_variant flags (st_geom.variant)
ST_VAR_NO_FOLD = 1
ST_VAR_TREE_LOOP = 2
ST_VAR_SPEC_GENERAL = 4
ST_VAR_SPEC_JUMP = 8
ST_VAR_SPEC_WIDE = 16
ST_VAR_SPEC_SELECT = 32
ST_VAR_SPEC_PRED = 64
ST_VAR_SPEC_BRANCH = 128
ST_VAR_SPEC_FIXED = 256
ST_VAR_SPEC_QUAD = 512


class st_stats(C.Structure):
    _fields_ = [("iterations", C.c_void_p), ("doubling_steps", C.c_void_p)]


class st_tree_info(C.Structure):
    _fields_ = [
        ("nodes", C.c_uint32),
        ("leaves", C.c_uint32),
        ("internal", C.c_uint32),
        ("depth", C.c_uint32),
        ("max_attribute", C.c_uint32),
        ("compact", C.c_uint32),
        ("spec_windows", C.c_uint32),
        ("spec_group_lanes", C.c_uint32),
        ("max_class", C.c_uint32),
    ]


class st_timing(C.Structure):
    _fields_ = [("outer_us", C.c_double), ("inner_us", C.c_double), ("alloc_us", C.c_double),
                ("h2d_us", C.c_double), ("d2h_us", C.c_double)]


class st_dataset_info(C.Structure):
    _fields_ = [("count", C.c_uint64), ("arity", C.c_uint32), ("layout", C.c_uint32),
                ("has_checksum", C.c_uint32), ("checksum", C.c_uint64), ("data_offset", C.c_uint64)]


# Every symbol declared in include/spectree_b200.h (checked by tests).
EXPORTS = (
    "st_last_error", "st_version", "st_device_count", "st_geom_default",
    "st_tree_create", "st_tree_destroy", "st_tree_get_info",
    "st_forest_create", "st_forest_destroy",
    "st_eval", "st_eval_device", "st_eval_sharded",
    "st_forest_eval", "st_forest_eval_device", "st_last_launch_count",
    "st_synthetic_tree", "st_synthetic_dataset", "st_dataset_checksum", "st_fnv1a64",
    "st_eval_timed", "st_dataset_save", "st_dataset_info_read", "st_dataset_load",
    "st_labels_save", "st_labels_load", "st_eval_file",
    "st_eval_depths", "st_eval_depths_device",
    "st_frames_open", "st_frames_slot", "st_frames_acquire", "st_frames_publish", "st_frames_wait",
    "st_frames_push", "st_frames_pop", "st_frames_status", "st_frames_close",
)

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"spectree_b200 CUDA library not found at {LIB_PATH}; run "
            "`python -m paper_1111_1373_b200.build` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    L.st_last_error.restype = C.c_char_p
    L.st_version.restype = C.c_char_p
    L.st_device_count.restype = i32
    L.st_device_count.argtypes = [C.POINTER(i32)]
    L.st_geom_default.argtypes = [C.POINTER(st_geom)]
    L.st_tree_create.restype = i32
    L.st_tree_create.argtypes = [vp, u32, C.POINTER(vp)]
    L.st_tree_destroy.argtypes = [vp]
    L.st_tree_get_info.restype = i32
    L.st_tree_get_info.argtypes = [vp, C.POINTER(st_tree_info)]
    L.st_forest_create.restype = i32
    L.st_forest_create.argtypes = [C.POINTER(vp), C.POINTER(u32), u32, u32, C.POINTER(vp)]
    L.st_forest_destroy.argtypes = [vp]
    L.st_eval.restype = i32
    L.st_eval.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp,
                          C.POINTER(st_stats)]
    L.st_eval_device.restype = i32
    L.st_eval_device.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp,
                                 C.POINTER(st_stats), vp]
    L.st_eval_sharded.restype = i32
    L.st_eval_sharded.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom),
                                  C.POINTER(i32), i32, vp]
    L.st_forest_eval.restype = i32
    L.st_forest_eval.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp]
    L.st_forest_eval_device.restype = i32
    L.st_forest_eval_device.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp, vp]
    L.st_eval_depths.restype = i32
    L.st_eval_depths.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp, vp]
    L.st_eval_depths_device.restype = i32
    L.st_eval_depths_device.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp, vp, vp]
    L.st_last_launch_count.restype = u32
    L.st_synthetic_tree.restype = i32
    L.st_synthetic_tree.argtypes = [u32, u32, u32, u32, u64, vp, u32, C.POINTER(u32)]
    L.st_synthetic_dataset.restype = i32
    L.st_synthetic_dataset.argtypes = [u64, u32, u64, i32, vp]
    L.st_dataset_checksum.restype = u64
    L.st_dataset_checksum.argtypes = [vp, u64, u32]
    L.st_fnv1a64.restype = u64
    L.st_fnv1a64.argtypes = [vp, u64]
    cp = C.c_char_p
    L.st_eval_timed.restype = i32
    L.st_eval_timed.argtypes = [vp, vp, u64, u32, u64, i32, C.POINTER(st_geom), vp,
                                C.POINTER(st_timing)]
    L.st_dataset_save.restype = i32
    L.st_dataset_save.argtypes = [cp, vp, u64, u32, i32, i32]
    L.st_dataset_info_read.restype = i32
    L.st_dataset_info_read.argtypes = [cp, C.POINTER(st_dataset_info)]
    L.st_dataset_load.restype = i32
    L.st_dataset_load.argtypes = [cp, u64, u64, vp, i32]
    L.st_labels_save.restype = i32
    L.st_labels_save.argtypes = [cp, vp, u64, u32]
    L.st_labels_load.restype = i32
    L.st_labels_load.argtypes = [cp, vp, u64, C.POINTER(u64), C.POINTER(u32)]
    L.st_eval_file.restype = i32
    L.st_eval_file.argtypes = [vp, cp, C.POINTER(st_geom), cp, u32, C.POINTER(u64)]
    L.st_frames_open.restype = i32
    L.st_frames_open.argtypes = [vp, u64, u32, u32, C.POINTER(st_geom), u32, u32, C.POINTER(vp)]
    L.st_frames_slot.restype = i32
    L.st_frames_slot.argtypes = [vp, u64, C.POINTER(vp), C.POINTER(vp)]
    for fn in (L.st_frames_acquire, L.st_frames_publish, L.st_frames_wait):
        fn.restype = i32
        fn.argtypes = [vp, u64, vp]
    L.st_frames_push.restype = i32
    L.st_frames_push.argtypes = [vp, vp, C.POINTER(u64)]
    L.st_frames_pop.restype = i32
    L.st_frames_pop.argtypes = [vp, u64, vp]
    L.st_frames_status.restype = i32
    L.st_frames_status.argtypes = [vp, C.POINTER(u64), C.POINTER(u32)]
    L.st_frames_close.restype = i32
    L.st_frames_close.argtypes = [vp]
    _lib = L
    return L


def last_error() -> str:
    return load().st_last_error().decode(errors="replace")
