"""Resident frame-stream evaluation (``st_frames_*``, include/spectree_b200.h).

One data-decomposition grid (or, with ``GpuGeom(algo="speculative")``, the
speculative ring) stays resident on the GPU and classifies frame 0, 1, 2, ...
as they are published into a device ring of frame slots -- the C3
per-pixel segmentation workload at video rate without a launch, a tree
staging or a pipeline ramp-up per frame.  Labels equal ``eval_gpu``'s for
every frame (the reference's ``eval_serial``, eval_serial.cpp:33-41).

Host producers::

    with FrameStream(tree, records=1920 * 1080, arity=8, ring=4) as fs:
        seq = fs.push(frame)          # (records, 8) float32
        labels = fs.pop(seq)          # (records,) uint32

While a stream is open its grid stays resident: device-wide synchronisation
(``torch.cuda.synchronize()``, ``cudaFree`` -- including a tree or forest
being destroyed) waits until ``close()``.  Synchronise streams instead.

Device producers (stream-ordered, no SM time for the synchronisation)::

    x, lab = fs.slot(seq)             # device tensors viewing the slot
    fs.acquire(seq, s)                # s waits until the slot is free
    ... write x on s ...
    fs.publish(seq, s)                # frame seq is ready after s's work
    fs.wait(seq, s2)                  # s2 waits for frame seq's labels
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .evaluate import GpuGeom, _as_tree, _check, _stream_handle
from .errors import ArgumentError


class FrameStream:
    def __init__(self, tree, records: int, arity: int, ring: int = 4, geom: Optional[GpuGeom] = None,
                 max_ctas: int = 0, idle_timeout_ms: int = 0):
        self.tree = _as_tree(tree)
        self.records, self.arity, self.ring = int(records), int(arity), int(ring)
        L = _lib.load()
        h = C.c_void_p()
        g = (geom or GpuGeom(algo="data")).to_c()
        _check(L.st_frames_open(self.tree.handle().h, self.records, self.arity, self.ring, C.byref(g),
                                int(max_ctas), int(idle_timeout_ms), C.byref(h)))
        self._h = h

    # ---- host producers ---------------------------------------------------
    def push(self, frame: np.ndarray) -> int:
        """Copy one frame of records into the next slot and publish it;
        blocks while the slot still holds an unfinished frame.  Returns the
        frame's sequence number."""
        x = np.ascontiguousarray(frame, dtype=np.float32)
        if x.shape != (self.records, self.arity):
            raise ArgumentError(f"frame must be ({self.records}, {self.arity}) float32, got {x.shape}")
        seq = C.c_uint64()
        _check(_lib.load().st_frames_push(self._live(), x.ctypes.data_as(C.c_void_p), C.byref(seq)))
        return seq.value

    def pop(self, seq: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Wait for frame ``seq`` and copy its labels out."""
        if out is None:
            out = np.empty(self.records, dtype=np.uint32)
        if out.dtype != np.uint32 or out.size != self.records or not out.flags.c_contiguous:
            raise ArgumentError("out must be a contiguous uint32 array of one frame's records")
        _check(_lib.load().st_frames_pop(self._live(), int(seq), out.ctypes.data_as(C.c_void_p)))
        return out

    # ---- device producers -------------------------------------------------
    def slot_ptrs(self, seq: int):
        """Device pointers (records, labels) of frame ``seq``'s slot."""
        xp, lp = C.c_void_p(), C.c_void_p()
        _check(_lib.load().st_frames_slot(self._live(), int(seq), C.byref(xp), C.byref(lp)))
        return xp.value, lp.value

    def slot(self, seq: int):
        """(records, labels) torch tensors viewing frame ``seq``'s slot."""
        import torch

        xp, lp = self.slot_ptrs(seq)
        dev = torch.cuda.current_device()
        x = _view(xp, (self.records, self.arity), torch.float32, dev)
        lab = _view(lp, (self.records,), torch.int32, dev)
        return x, lab

    def acquire(self, seq: int, stream=None) -> None:
        _check(_lib.load().st_frames_acquire(self._live(), int(seq), _stream_handle(stream)))

    def publish(self, seq: int, stream=None) -> None:
        _check(_lib.load().st_frames_publish(self._live(), int(seq), _stream_handle(stream)))

    def wait(self, seq: int, stream=None) -> None:
        _check(_lib.load().st_frames_wait(self._live(), int(seq), _stream_handle(stream)))

    def status(self):
        """(frames published, stopped by its idle timeout)."""
        pub, stop = C.c_uint64(), C.c_uint32()
        _check(_lib.load().st_frames_status(self._live(), C.byref(pub), C.byref(stop)))
        return pub.value, bool(stop.value)

    def close(self) -> None:
        """Walk every published frame, stop the resident grid, free the ring.
        The tree reference is dropped here too: a tree destroyed later (its
        device tables freed by cudaFree, which waits for every resident grid)
        could otherwise stall behind the next frame stream."""
        if self._h is not None:
            h, self._h = self._h, None
            try:
                _check(_lib.load().st_frames_close(h))
            finally:
                self.tree = None

    def _live(self):
        if self._h is None:
            raise ArgumentError("frame stream is closed")
        return self._h

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _view(ptr: int, shape, dtype, device: int):
    """A torch tensor over device memory owned by the frame stream."""
    import torch

    class _Cai:
        def __init__(self):
            typestr = {torch.float32: "<f4", torch.int32: "<i4"}[dtype]
            self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                             "version": 3, "strides": None}

    return torch.as_tensor(_Cai(), device=f"cuda:{device}")
