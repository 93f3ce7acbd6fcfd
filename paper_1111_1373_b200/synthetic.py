"""Canonical synthetic inputs (reference synthetic.hpp:18-30) via the native
library: same seed -> byte-identical trees and records to the reference."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .errors import raise_for
from .tree import NODE_DTYPE, EncodedTree


def generate_synthetic_tree(depth: int, leaf_count: int, arity: int, class_count: int,
                            seed: int) -> EncodedTree:
    L = _lib.load()
    n = C.c_uint32()
    rc = L.st_synthetic_tree(depth, leaf_count, arity, class_count, seed, None, 0, C.byref(n))
    raise_for(rc, _lib.last_error())
    out = np.empty(n.value, dtype=NODE_DTYPE)
    rc = L.st_synthetic_tree(depth, leaf_count, arity, class_count, seed,
                             out.ctypes.data_as(C.c_void_p), n.value, C.byref(n))
    raise_for(rc, _lib.last_error())
    return EncodedTree(out)


def generate_synthetic_dataset(count: int, arity: int, seed: int, gaussian: bool = False,
                               out: Optional[np.ndarray] = None) -> np.ndarray:
    """(count, arity) float32.  ``out`` may be a preallocated C-contiguous
    float32 buffer (e.g. a pinned-host tensor's numpy view)."""
    if out is None:
        out = np.empty((count, arity), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size == count * arity
    rc = _lib.load().st_synthetic_dataset(count, arity, seed, int(bool(gaussian)),
                                          out.ctypes.data_as(C.c_void_p))
    raise_for(rc, _lib.last_error())
    return out.reshape(count, arity)


def dataset_checksum(x: np.ndarray) -> int:
    x = np.ascontiguousarray(x, dtype=np.float32)
    return int(_lib.load().st_dataset_checksum(x.ctypes.data_as(C.c_void_p), x.shape[0], x.shape[1]))


def fnv1a64(arr: np.ndarray) -> int:
    a = np.ascontiguousarray(arr)
    return int(_lib.load().st_fnv1a64(a.ctypes.data_as(C.c_void_p), a.nbytes))
