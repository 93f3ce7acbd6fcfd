"""The reference verify/bench flow with the GPU strategies.

Mirrors core/include/spectree/bench.hpp for the strategies that run here:
``gpu-data`` (Algorithm 1) and ``gpu-spec`` (Algorithm 2).  Timing windows
keep the reference's meaning (bench.hpp:50-56, bench.cpp:228-262): "outer" is
one whole host round trip (device allocation, records H2D, kernel, labels
D2H, release), "inner" the kernel alone (CUDA events), "alloc" the device
allocation + release -- the paper's Table 1 columns.  Each iteration is one
``st_eval_timed`` call.  The CPU strategies (serial, data, spec, spec-basic)
are the reference's own C++ evaluators; the C++ flow that runs them beside
these is include/spectree_b200_bench.hpp.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ArgumentError, raise_for
from .evaluate import (DataParallelConfig, GpuGeom, SpeculativeConfig, _as_data, _as_tree,
                       check_attribute_range, default_data_parallel, default_speculative,
                       validate_data_parallel, validate_speculative)


class Strategy(enum.Enum):
    gpu_data = "gpu-data"
    gpu_spec = "gpu-spec"


def strategy_name(s: Strategy) -> str:
    return s.value


def strategy_from_name(name: str) -> Optional[Strategy]:
    for s in Strategy:
        if s.value == name:
            return s
    return None


@dataclass
class TimingStats:
    """bench.hpp:22-30; population stddev (bench.cpp:128-151)."""

    mean_us: float = 0.0
    min_us: float = 0.0
    max_us: float = 0.0
    stddev_us: float = 0.0
    iterations: int = 0


def summarize(samples_us: Sequence[float]) -> TimingStats:
    s = TimingStats()
    if len(samples_us) == 0:
        return s
    a = np.asarray(samples_us, dtype=np.float64)
    s.iterations = int(a.size)
    s.min_us, s.max_us = float(a.min()), float(a.max())
    s.mean_us = float(a.sum() / a.size)
    s.stddev_us = float(math.sqrt(((a - s.mean_us) ** 2).sum() / a.size))
    return s


@dataclass
class StrategyReport:
    strategy: Strategy
    outer: TimingStats
    inner: TimingStats
    alloc: TimingStats
    h2d_mean_us: float
    d2h_mean_us: float
    labels: np.ndarray = field(repr=False, default=None)
    mismatches: Optional[int] = None  # against `expected` when given


def eval_timed(tree, dataset, geom: Optional[GpuGeom] = None):
    """One unpipelined round trip through ``st_eval_timed``: returns
    (labels, {outer_us, inner_us, alloc_us, h2d_us, d2h_us})."""
    tree = _as_tree(tree)
    d = _as_data(dataset)
    check_attribute_range(tree, d)
    m = d.count()
    out = np.empty(m, dtype=np.uint32)
    t = _lib.st_timing()
    g = (geom or GpuGeom()).to_c()
    x = d.values()
    h = tree.handle()
    rc = _lib.load().st_eval_timed(h.h, x.ctypes.data_as(C.c_void_p) if m else None, m, d.arity(), 0,
                                   _lib.ST_LAYOUT_AOS, C.byref(g),
                                   out.ctypes.data_as(C.c_void_p) if m else None, C.byref(t))
    if rc:
        raise_for(rc, _lib.last_error())
    return out, {k: float(getattr(t, k)) for k, _ in _lib.st_timing._fields_}


def run_bench(tree, dataset, strategies: Sequence[Strategy] = (Strategy.gpu_data, Strategy.gpu_spec),
              iterations: int = 100, warmup: int = 10,
              data_parallel: Optional[DataParallelConfig] = None,
              speculative: Optional[SpeculativeConfig] = None,
              expected: Optional[np.ndarray] = None) -> List[StrategyReport]:
    """bench.cpp:168-281 for the GPU strategies: geometry validated before any
    clock starts, warm-up excluded, labels checked against ``expected``
    (e.g. the reference's eval_serial output) when given."""
    tree = _as_tree(tree)
    d = _as_data(dataset)
    if iterations == 0:
        raise ArgumentError("bench iterations must be >= 1")
    if not strategies:
        raise ArgumentError("bench requires at least one strategy")
    check_attribute_range(tree, d)
    dp = data_parallel or default_data_parallel(d.count())
    sp = speculative or default_speculative(tree, d.count())
    for s in strategies:
        if s is Strategy.gpu_data:
            validate_data_parallel(dp, d.count())
        elif s is Strategy.gpu_spec:
            validate_speculative(sp, tree, d.count(), False)
        else:
            raise ArgumentError(f"unknown strategy '{s}'")
    reports = []
    for s in strategies:
        geom = GpuGeom(**{**(dp.gpu if s is Strategy.gpu_data else sp.gpu).__dict__,
                          "algo": "data" if s is Strategy.gpu_data else "speculative"})
        outer, inner, alloc, h2d, d2h = [], [], [], [], []
        last = None
        for i in range(warmup + iterations):
            last, t = eval_timed(tree, d, geom)
            if i >= warmup:
                outer.append(t["outer_us"])
                inner.append(t["inner_us"])
                alloc.append(t["alloc_us"])
                h2d.append(t["h2d_us"])
                d2h.append(t["d2h_us"])
        r = StrategyReport(s, summarize(outer), summarize(inner), summarize(alloc),
                           float(np.mean(h2d)), float(np.mean(d2h)), last)
        if expected is not None:
            r.mismatches = int((np.asarray(expected, dtype=np.uint32) != last).sum())
        reports.append(r)
    return reports
