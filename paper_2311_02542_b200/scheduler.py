"""Throughput-proportional row scheduler (proj/include/lumi/scheduler.h, proj/src/scheduler.cpp).

The arithmetic (largest-remainder rounding, dampened shares, p99 statistics) runs in the
native library (lumi_equal_assignment / lumi_assign_rows / lumi_next_assignment /
lumi_aggregate_stats); this module keeps the reference's types and `run_frame`, whose
workers are host threads driving one GPU (or one CUDA stream) each.  The multi-process
one-rank-per-GPU driver is in multigpu.py.
"""
from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import Error, check


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class RowRange:
    begin: int = 0
    end: int = 0

    def count(self) -> int:
        return self.end - self.begin


@dataclass
class WorkerAssignment:
    """scheduler.h:22-35."""

    ranges: List[RowRange] = field(default_factory=list)
    shares: List[float] = field(default_factory=list)
    height: int = 0

    def valid(self) -> bool:
        if not self.ranges or self.ranges[0].begin != 0 or self.ranges[-1].end != self.height:
            return False
        for i, r in enumerate(self.ranges):
            if r.count() < 0:
                return False
            if i and r.begin != self.ranges[i - 1].end:
                return False
        return True

    def rows(self) -> np.ndarray:
        return np.array([r.count() for r in self.ranges], np.int32)


def _from_rows(rows: np.ndarray, shares: np.ndarray, height: int) -> WorkerAssignment:
    a = WorkerAssignment(height=height)
    at = 0
    for r, s in zip(rows.tolist(), shares.tolist()):
        a.ranges.append(RowRange(at, at + r))
        a.shares.append(s)
        at += r
    return a


def equal_assignment(height: int, workers: int) -> WorkerAssignment:
    rows = np.zeros(max(workers, 1), np.int32)
    shares = np.zeros(max(workers, 1))
    check(_abi.lib().lumi_equal_assignment(height, workers, _p(rows), _p(shares)))
    return _from_rows(rows, shares, height)


def assign_rows(height: int, throughputs: Sequence[float], prev: WorkerAssignment,
                dampening: float) -> WorkerAssignment:
    n = len(throughputs)
    if len(prev.ranges) != n:
        raise Error("assign_rows: worker count changed")
    tp = np.ascontiguousarray(throughputs, np.float64)
    ps = np.ascontiguousarray(prev.shares, np.float64)
    rows = np.zeros(max(n, 1), np.int32)
    shares = np.zeros(max(n, 1))
    check(_abi.lib().lumi_assign_rows(height, n, _p(tp), _p(ps), float(dampening), _p(rows),
                                      _p(shares)))
    return _from_rows(rows[:n], shares[:n], height)


@dataclass
class FrameStats:
    """scheduler.h:44-50."""

    wall_ms: float = 0.0
    rays: int = 0
    worker_ms: List[float] = field(default_factory=list)
    worker_rays: List[int] = field(default_factory=list)

    def fps(self) -> float:
        return 1000.0 / self.wall_ms if self.wall_ms > 0 else 0.0


@dataclass
class StatsSummary:
    mean_fps: float = 0.0
    std_fps: float = 0.0
    p99_fps: float = 0.0


def aggregate_stats(frames: Sequence[FrameStats]) -> StatsSummary:
    ms = np.ascontiguousarray([f.wall_ms for f in frames], np.float64)
    if ms.size == 0:
        raise Error("aggregate_stats: no frames")
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    check(_abi.lib().lumi_aggregate_stats(_p(ms), int(ms.size), C.byref(a), C.byref(b),
                                          C.byref(c)))
    return StatsSummary(a.value, b.value, c.value)


def next_assignment(current: WorkerAssignment, stats: FrameStats,
                    dampening: float) -> WorkerAssignment:
    """scheduler.cpp:154-162: throughput_k = max(rays_k, 1) / (max(ms_k, 1e-6) / 1000)."""
    tp = [max(float(r), 1.0) / (max(ms, 1e-6) / 1000.0)
          for r, ms in zip(stats.worker_rays, stats.worker_ms)]
    return assign_rows(current.height, tp, current, dampening)


def run_frame(assignment: WorkerAssignment, width: int, work: Callable[[int, RowRange], None],
              simulated_ms: Optional[Sequence[float]] = None) -> FrameStats:
    """scheduler.cpp:114-152: one thread per worker on disjoint row ranges; worker
    exceptions are re-raised as Error("run_frame: worker i failed: ...")."""
    if not assignment.valid():
        raise Error("run_frame: invalid assignment")
    n = len(assignment.ranges)
    st = FrameStats(worker_ms=[0.0] * n, worker_rays=[0] * n)
    errors: List[Optional[str]] = [None] * n

    def body(i: int) -> None:
        t0 = time.perf_counter()
        try:
            work(i, assignment.ranges[i])
        except Exception as e:  # noqa: BLE001 - mirrors catch (const std::exception&)
            errors[i] = str(e)
        st.worker_ms[i] = (time.perf_counter() - t0) * 1000.0

    t0 = time.perf_counter()
    threads = [threading.Thread(target=body, args=(i,)) for i in range(n)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for i, e in enumerate(errors):
        if e is not None:
            raise Error(f"run_frame: worker {i} failed: {e}")
    st.wall_ms = (time.perf_counter() - t0) * 1000.0
    if simulated_ms is not None:
        st.worker_ms = list(simulated_ms)
        st.wall_ms = max(simulated_ms)
    st.worker_rays = [assignment.ranges[i].count() * width for i in range(n)]
    st.rays = assignment.height * width
    return st
