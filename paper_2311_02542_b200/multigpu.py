"""Stereo eyebuffer frames across GPUs: one process per GPU (torch.distributed for the
plumbing), rows of the stacked dual-eye image split by the paper's dynamic,
throughput-proportional scheduler (proj/src/scheduler.cpp:68-87, 154-162; §5), and
finished bands gathered to rank 0 over NVLink with NCCL point-to-point transfers (the bands
are unequal, so an all-gather does not fit).

With world size 1 the same driver renders the whole frame on one GPU with no collective.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np

from . import _abi, scenes
from .renderer import CameraModel, DeviceModel, RenderOptions
from .scheduler import FrameStats, WorkerAssignment, equal_assignment, next_assignment


def eye_bands(begin: int, end: int, eye_size: int):
    """Splits stacked-image rows [begin, end) at the eye seam: yields (eye, cam_b, cam_e)."""
    for eye in (0, 1):
        lo, hi = max(begin, eye * eye_size), min(end, (eye + 1) * eye_size)
        if lo < hi:
            yield eye, lo - eye * eye_size, hi - eye * eye_size


def gather_bands(dist, img, assign: WorkerAssignment, rank: int, world: int) -> None:
    """Rank r > 0 sends rows [begin, end) of its band of the planar [C, H, W] image to rank 0
    (one contiguous slab per plane), batched point-to-point; bands are unequal, so an
    all-gather does not fit.  Works for CUDA tensors over NCCL and CPU tensors over gloo."""
    if world == 1:
        return
    ops = []
    planes = img.shape[0]
    if rank == 0:
        for r in range(1, world):
            rr = assign.ranges[r]
            if rr.count() > 0:
                for c in range(planes):
                    ops.append(dist.P2POp(dist.irecv, img[c, rr.begin:rr.end], r))
    else:
        rr = assign.ranges[rank]
        if rr.count() > 0:
            for c in range(planes):
                ops.append(dist.P2POp(dist.isend, img[c, rr.begin:rr.end].contiguous(), 0))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def exchange_ms(torch, dist, ms_local: float, world: int, device) -> List[float]:
    """All ranks learn every rank's band time (the reference measures per worker,
    scheduler.cpp:124-142)."""
    if world == 1:
        return [ms_local]
    t = torch.tensor([ms_local], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def rebalance(assign: WorkerAssignment, ms: List[float], width: int,
              dampening: float) -> (FrameStats, WorkerAssignment):
    """FrameStats of the finished frame and the next assignment (scheduler.cpp:154-162);
    deterministic, so every rank computes the same partition."""
    st = FrameStats(wall_ms=max(ms), rays=assign.height * width, worker_ms=list(ms),
                    worker_rays=[r.count() * width for r in assign.ranges])
    nxt = next_assignment(assign, st, dampening) if len(ms) > 1 else assign
    return st, nxt


class StereoFrameDriver:
    """Renders dual `eye_size`^2 eyebuffers stacked into one [3, 2*eye_size, eye_size]
    planar frame.  Each rank renders its scheduler band; rank 0 receives the others."""

    def __init__(self, torch, model: DeviceModel, eye_size: int, opts: RenderOptions,
                 rank: int = 0, world: int = 1, dampening: float = 0.5, gather: bool = True,
                 dist=None, counters: bool = False):
        self.torch, self.dm, self.S, self.opts = torch, model, int(eye_size), opts
        self.rank, self.world, self.damp, self.gather, self.dist = rank, world, dampening, gather, dist
        self.H, self.W = 2 * self.S, self.S
        self.assign: WorkerAssignment = equal_assignment(self.H, world)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.rgb = torch.zeros((3, self.H, self.W), dtype=torch.float32, device=dev)
        self.stats = torch.zeros(4, dtype=torch.int64, device=dev) if counters else None
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self.launches = 0
        self.history: List[FrameStats] = []

    def cameras(self, frame: int) -> List[CameraModel]:
        rot, origin = scenes.head_pose(frame)
        return [CameraModel.from_spec(c) for c in scenes.eye_cameras(self.S, rot, origin)]

    def _target(self, eye: int) -> _abi.FrameTarget:
        t = _abi.FrameTarget()
        t.rgb = self.rgb.data_ptr()
        t.work_stats = self.stats.data_ptr() if self.stats is not None else None
        t.width, t.height, t.row_offset = self.W, self.H, eye * self.S
        return t

    def render_local(self, frame: int) -> None:
        """Enqueues this rank's band on the current stream (no host sync)."""
        stream = self.torch.cuda.current_stream().cuda_stream
        band = self.assign.ranges[self.rank]
        cams = self.cameras(frame)
        self.ev0.record()
        for eye, b, e in eye_bands(band.begin, band.end, self.S):
            self.dm.render_rows_async(cams[eye], self.opts, b, e, self._target(eye), stream)
            self.launches += 1 if self.dm.kernel == "simt" else 2  # march pass + render
        self.ev1.record()

    def gather_bands(self) -> None:
        if self.gather:
            gather_bands(self.dist, self.rgb, self.assign, self.rank, self.world)

    def rebalance(self) -> FrameStats:
        """Per-rank render time of the frame just finished -> next assignment."""
        self.ev1.synchronize()
        ms = exchange_ms(self.torch, self.dist, float(self.ev0.elapsed_time(self.ev1)),
                         self.world, self.rgb.device)
        st, self.assign = rebalance(self.assign, ms, self.W, self.damp)
        self.history.append(st)
        return st

    def frame(self, frame: int) -> FrameStats:
        self.render_local(frame)
        self.gather_bands()
        return self.rebalance()

    def counters(self) -> Optional[np.ndarray]:
        return None if self.stats is None else self.stats.cpu().numpy()
