"""Record table mirroring the reference Dataset (core/include/spectree/dataset.hpp).

Row-major (AoS) float32, ``record(i) = values + i*arity`` (dataset.hpp:20-22),
``arity >= 1`` (dataset.cpp:10-14).  ``ClassAssignment`` is a uint32 numpy
array, one class per record, positionally aligned (dataset.hpp:35-36).
"""
from __future__ import annotations

import numpy as np

from .errors import ArgumentError

ClassAssignment = np.ndarray  # uint32[count]


class Dataset:
    def __init__(self, arity: int, values=None):
        if arity == 0:
            raise ArgumentError("dataset arity must be >= 1")
        self._arity = int(arity)
        if values is None:
            values = np.zeros((0, arity), dtype=np.float32)
        v = np.asarray(values, dtype=np.float32)
        if v.ndim == 1:
            if v.size % arity != 0:
                raise ArgumentError("value count is not a multiple of the arity")
            v = v.reshape(-1, arity)
        if v.ndim != 2 or v.shape[1] != arity:
            raise ArgumentError("record arity mismatch")
        self._values = np.ascontiguousarray(v)

    @classmethod
    def from_array(cls, x) -> "Dataset":
        x = np.asarray(x, dtype=np.float32)
        return cls(x.shape[1], x)

    def arity(self) -> int:
        return self._arity

    def count(self) -> int:
        return int(self._values.shape[0])

    def record(self, i: int) -> np.ndarray:
        return self._values[i]

    def values(self) -> np.ndarray:
        """(count, arity) float32, C-contiguous."""
        return self._values

    def append(self, record) -> None:
        r = np.asarray(record, dtype=np.float32).reshape(1, -1)
        if r.shape[1] != self._arity:
            raise ArgumentError("record arity mismatch")
        self._values = np.ascontiguousarray(np.concatenate([self._values, r]))

    def __len__(self) -> int:
        return self.count()


def tile_dataset(dataset: Dataset, factor: int) -> Dataset:
    """Concatenate ``factor`` copies (dataset.cpp:35-46)."""
    if factor == 0:
        raise ArgumentError("tile factor must be >= 1")
    return Dataset(dataset.arity(), np.tile(dataset.values(), (factor, 1)))
