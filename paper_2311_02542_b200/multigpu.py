"""Stereo eyebuffer frames across GPUs: one process per GPU (torch.distributed for the
plumbing), rows of the stacked dual-eye image split by the paper's dynamic,
throughput-proportional scheduler (proj/src/scheduler.cpp:68-87, 154-162; §5), and
the bands gathered to rank 0 over NVLink one of two ways:

* ``gather="p2p"`` (default): rank 0's two frame buffers (frames alternate between them) are
  mapped into every rank through CUDA IPC handles (`lumi_ipc_export` / `lumi_ipc_open`), and
  each rank's render kernel stores its band's pixels straight into rank 0's memory as it
  renders -- the gather IS the kernel's epilogue, there is no separate transfer.  The per-frame
  exchange of band times (which every rank waits on after its own kernel finished) orders
  those stores before rank 0 reads the frame; alternating buffers keep a fast rank's next
  frame off the buffer rank 0 may still be copying out.
* ``gather="nccl"``: finished bands are sent to rank 0 with batched NCCL point-to-point
  transfers (the bands are unequal, so an all-gather does not fit).

With world size 1 the same driver renders the whole frame on one GPU with no collective.

`NativeFrameDriver` is the single-process form behind the C ABI (lumi_frame_driver_*): one
host thread per GPU inside liblumi_cuda.so, exactly the reference's run_frame shape
(scheduler.cpp:114-162), for callers of the drop-in that do not run one process per GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _abi, scenes
from .renderer import CameraModel, DeviceModel, RenderOptions
from .scheduler import (FrameStats, WorkerAssignment, _from_rows, equal_assignment,
                        next_assignment)


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
    out = torch.empty(world, dtype=torch.float64, device=device)
    try:
        # one collective into one tensor, one device-to-host read: the exchange sits between
        # two frames on every rank, so its latency is paid once per frame at any N
        dist.all_gather_into_tensor(out, t)
    except (RuntimeError, NotImplementedError):  # backends without the tensor form
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        out = torch.cat(parts)
    return out.cpu().tolist()


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
                 rank: int = 0, world: int = 1, dampening: float = 0.5, gather="p2p",
                 dist=None, counters: bool = False):
        self.torch, self.dm, self.S, self.opts = torch, model, int(eye_size), opts
        if gather is True:
            gather = "p2p"
        if gather not in (False, None, "p2p", "nccl"):
            raise ValueError(f"gather must be 'p2p', 'nccl' or False, got {gather!r}")
        self.rank, self.world, self.damp, self.dist = rank, world, dampening, dist
        self.gather = gather if world > 1 else None
        self.H, self.W = 2 * self.S, self.S
        self.assign: WorkerAssignment = equal_assignment(self.H, world)
        self.dev = dev = torch.device("cuda", torch.cuda.current_device())
        # frames alternate between two buffers; with the p2p gather rank 0's are the targets of
        # every rank's kernel (ranks > 0 map them and keep no frame of their own)
        nbuf = 2 if self.gather == "p2p" else 1
        self.frames = [torch.zeros((3, self.H, self.W), dtype=torch.float32, device=dev)
                       for _ in range(nbuf if rank == 0 or self.gather != "p2p" else 0)]
        self._targets_ptr = [f.data_ptr() for f in self.frames]
        self._peer = []
        if self.gather == "p2p":
            self._map_rank0_frames(dev.index)
        self.rgb = self.frames[0] if self.frames else None
        self.stats = torch.zeros(4, dtype=torch.int64, device=dev) if counters else None
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self._pending = []  # world 1, frame(sync=False): (ev0, ev1) of frames not yet collected
        self.launches = 0
        self.history: List[FrameStats] = []

    def _map_rank0_frames(self, device: int) -> None:
        import ctypes as C
        L = _abi.lib()
        handles = None
        if self.rank == 0:
            handles = []
            for f in self.frames:
                h = (C.c_uint8 * 64)()
                off = C.c_uint64()
                _abi.check(L.lumi_ipc_export(C.c_void_p(f.data_ptr()), h, C.byref(off)))
                handles.append((bytes(h), off.value))
        box = [handles]
        self.dist.broadcast_object_list(box, src=0)
        if self.rank != 0:
            for h, off in box[0]:
                p = C.c_void_p()
                hb = (C.c_uint8 * 64).from_buffer_copy(h)
                _abi.check(L.lumi_ipc_open(device, hb, C.c_uint64(off), C.byref(p)))
                self._peer.append(p.value)
            self._targets_ptr = list(self._peer)

    def close(self) -> None:
        """Unmaps rank 0's frames (p2p gather); rank 0 must keep its buffers alive until every
        rank has closed, so callers end with a barrier."""
        if self._peer:
            self.torch.cuda.synchronize()
            for p in self._peer:
                _abi.check(_abi.lib().lumi_ipc_close(self.torch.cuda.current_device(), p))
            self._peer = []
            self._targets_ptr = []

    def frame_buffer(self, frame: int):
        """Rank 0's [3, H, W] buffer holding `frame` (None on ranks > 0 with the p2p gather)."""
        return self.frames[frame % len(self.frames)] if self.frames else None

    def cameras(self, frame: int) -> List[CameraModel]:
        rot, origin = scenes.head_pose(frame)
        return [CameraModel.from_spec(c) for c in scenes.eye_cameras(self.S, rot, origin)]

    def _target(self, eye: int, frame: int) -> _abi.FrameTarget:
        t = _abi.FrameTarget()
        t.rgb = self._targets_ptr[frame % len(self._targets_ptr)]
        t.work_stats = self.stats.data_ptr() if self.stats is not None else None
        t.width, t.height, t.row_offset = self.W, self.H, eye * self.S
        return t

    def render_local(self, frame: int) -> None:
        """Enqueues this rank's band on the current stream (no host sync)."""
        if self._pending:  # this frame gets its own events; the pending ones keep theirs
            self.ev0 = self.torch.cuda.Event(enable_timing=True)
            self.ev1 = self.torch.cuda.Event(enable_timing=True)
        stream = self.torch.cuda.current_stream().cuda_stream
        band = self.assign.ranges[self.rank]
        cams = self.cameras(frame)
        if self.frames:
            self.rgb = self.frame_buffer(frame)
        self.ev0.record()
        for eye, b, e in eye_bands(band.begin, band.end, self.S):
            self.dm.render_rows_async(cams[eye], self.opts, b, e, self._target(eye, frame), stream)
            self.launches += 1 if self.dm.kernel == "simt" else 2  # march pass + render
        self.ev1.record()

    def gather_bands(self) -> None:
        if self.gather == "nccl":
            gather_bands(self.dist, self.rgb, self.assign, self.rank, self.world)

    def rebalance(self) -> FrameStats:
        """Per-rank render time of the frame just finished -> next assignment."""
        self.ev1.synchronize()
        dev = "cpu" if self.world > 1 and self.dist.get_backend() == "gloo" else self.dev
        ms = exchange_ms(self.torch, self.dist, float(self.ev0.elapsed_time(self.ev1)),
                         self.world, dev)
        st, self.assign = rebalance(self.assign, ms, self.W, self.damp)
        self.history.append(st)
        return st

    def frame(self, frame: int, sync: bool = True) -> Optional[FrameStats]:
        """One frame: render this rank's band, gather, rebalance from the band times (the
        reference's run_frame + next_assignment, scheduler.cpp:114-162).  With one GPU the
        assignment never changes (next_assignment of a single worker is the identity), so
        `sync=False` only enqueues the frame -- frames run back to back on the device and
        `collect()` returns their FrameStats once."""
        if not sync and self.world == 1:
            self.render_local(frame)
            self._pending.append((self.ev0, self.ev1))
            return None
        self.render_local(frame)
        self.gather_bands()
        return self.rebalance()

    def collect(self) -> List[FrameStats]:
        """FrameStats of the frames enqueued with frame(sync=False), in order (one host sync)."""
        if not self._pending:
            return []
        self._pending[-1][1].synchronize()
        out = []
        for e0, e1 in self._pending:
            ms = float(e0.elapsed_time(e1))
            st, self.assign = rebalance(self.assign, [ms], self.W, self.damp)
            self.history.append(st)
            out.append(st)
        self._pending = []
        return out

    def counters(self) -> Optional[np.ndarray]:
        return None if self.stats is None else self.stats.cpu().numpy()


class NativeFrameDriver:
    """run_frame + next_assignment inside the native library (lumi_frame_driver_*): worker i
    renders with models[i] (one replica per GPU; a model may repeat to run several workers on
    one GPU), one host thread per worker, every band stored straight into the device frame
    target (over NVLink peer access from other GPUs).  `render` returns the FrameStats of the
    frame and moves the assignment for the next one."""

    def __init__(self, models: Sequence[DeviceModel], eye_size: int, eyes: int = 2,
                 dampening: float = 0.5, width: Optional[int] = None):
        L = _abi.lib()
        self.models = list(models)  # keeps the replicas alive
        self.n = len(self.models)
        self.W = int(width or eye_size)
        self.S, self.eyes = int(eye_size), int(eyes)
        self.H = self.S * self.eyes
        arr = (C.c_void_p * self.n)(*[m.h.value for m in self.models])
        h = C.c_void_p()
        _abi.check(L.lumi_frame_driver_create(arr, self.n, self.W, self.S, self.eyes,
                                              float(dampening), C.byref(h)))
        self.h = h

    def assignment(self) -> WorkerAssignment:
        import numpy as np
        rows = np.zeros(self.n, np.int32)
        shares = np.zeros(self.n, np.float64)
        _abi.check(_abi.lib().lumi_frame_driver_assignment(self.h, rows.ctypes.data,
                                                           shares.ctypes.data))
        return _from_rows(rows, shares, self.H)

    def set_assignment(self, rows: Sequence[int]) -> None:
        import numpy as np
        r = np.ascontiguousarray(rows, np.int32)
        _abi.check(_abi.lib().lumi_frame_driver_set_assignment(self.h, r.ctypes.data))

    def render(self, cams: Sequence[CameraModel], opts: RenderOptions,
               target: _abi.FrameTarget) -> FrameStats:
        import numpy as np
        cd = (_abi.CameraDesc * self.eyes)(*[c.desc() for c in cams])
        od = opts.desc()
        wall = C.c_double()
        ms = np.zeros(self.n, np.float64)
        rays = np.zeros(self.n, np.int64)
        rows_before = self.assignment()
        _abi.check(_abi.lib().lumi_frame_driver_render(self.h, cd, C.byref(od), C.byref(target),
                                                       C.byref(wall), ms.ctypes.data,
                                                       rays.ctypes.data))
        return FrameStats(wall_ms=float(wall.value), rays=rows_before.height * self.W,
                          worker_ms=ms.tolist(), worker_rays=rays.tolist())

    def close(self) -> None:
        if getattr(self, "h", None):
            _abi.lib().lumi_frame_driver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
