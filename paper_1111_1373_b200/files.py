"""Record / label files at scale over the C ABI.

The reference loads datasets only from CSV (io.cpp:80-117) and writes
assignments as text (io.cpp:274-283); both are parse-bound far below what one
B200 classifies.  This module mirrors the raw binary formats specified in
include/spectree_b200.h (``STREC001`` float32 records, AoS or SoA, with the
reference ``dataset_checksum`` in the header; ``STLAB001`` u32 or u8 labels)
and the streaming evaluator ``st_eval_file`` that pushes a file of any size
through the GPU in pinned 64 MB chunks.  Errors follow the reference
taxonomy: malformed files raise ``IoError`` (exit code 3), bad arguments
``ArgumentError``.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .dataset import Dataset
from .errors import ArgumentError, raise_for
from .evaluate import GpuGeom, _as_data, _as_tree

_LAYOUTS = {"aos": _lib.ST_LAYOUT_AOS, "soa": _lib.ST_LAYOUT_SOA}


def _check(rc: int) -> None:
    if rc:
        raise_for(rc, _lib.last_error())


def save_dataset_bin(path: str, dataset, layout: str = "aos", checksum: bool = True) -> None:
    """Write ``dataset`` as a STREC001 file (``layout`` = file layout)."""
    if layout not in _LAYOUTS:
        raise ArgumentError(f"unknown layout '{layout}'")
    d = _as_data(dataset)
    x = d.values() if layout == "aos" else np.ascontiguousarray(d.values().T)
    _check(_lib.load().st_dataset_save(path.encode(), x.ctypes.data_as(C.c_void_p) if x.size else None,
                                       d.count(), d.arity(), _LAYOUTS[layout], int(checksum)))


def dataset_info(path: str) -> dict:
    inf = _lib.st_dataset_info()
    _check(_lib.load().st_dataset_info_read(path.encode(), C.byref(inf)))
    return {"count": int(inf.count), "arity": int(inf.arity),
            "layout": "aos" if inf.layout == _lib.ST_LAYOUT_AOS else "soa",
            "checksum": int(inf.checksum) if inf.has_checksum else None,
            "data_offset": int(inf.data_offset)}


def load_dataset_bin(path: str, first: int = 0, count: Optional[int] = None,
                     verify: bool = False) -> Dataset:
    """Records ``[first, first+count)`` of a STREC001 file as a (AoS) Dataset;
    ``verify`` re-checks the header checksum over the whole file first."""
    info = dataset_info(path)
    if count is None:
        count = max(0, info["count"] - first)
    out = np.empty((count, info["arity"]), dtype=np.float32)
    _check(_lib.load().st_dataset_load(path.encode(), first, count,
                                       out.ctypes.data_as(C.c_void_p) if out.size else None,
                                       int(verify)))
    return Dataset(info["arity"], out)


def save_labels_bin(path: str, labels, width: int = 4) -> None:
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    _check(_lib.load().st_labels_save(path.encode(), lab.ctypes.data_as(C.c_void_p) if lab.size else None,
                                      lab.size, width))


def load_labels_bin(path: str) -> np.ndarray:
    L = _lib.load()
    n, w = C.c_uint64(), C.c_uint32()
    _check(L.st_labels_load(path.encode(), None, 0, C.byref(n), C.byref(w)))
    out = np.empty(n.value, dtype=np.uint32)
    _check(L.st_labels_load(path.encode(), out.ctypes.data_as(C.c_void_p) if out.size else None,
                            n.value, C.byref(n), C.byref(w)))
    return out


def eval_file(tree, data_path: str, labels_path: str, geom: Optional[GpuGeom] = None,
              width: int = 4) -> int:
    """Stream a STREC001 file through the GPU into a STLAB001 label file
    (``width`` 1 = u8 labels, narrowed on the device).  Returns the record
    count.  The file never has to fit in host memory."""
    tree = _as_tree(tree)
    g = (geom or GpuGeom()).to_c()
    n = C.c_uint64()
    h = tree.handle()
    _check(_lib.load().st_eval_file(h.h, data_path.encode(), C.byref(g), labels_path.encode(),
                                    width, C.byref(n)))
    return int(n.value)
