"""Host-side mirror of the reference renderer/model API over the sm_100a C ABI.

Names, argument meaning and error behaviour follow proj/include/lumi/{grid,field,camera,
occupancy,renderer}.h so code (and tests) written against the reference read the same:

    field = RadianceField(FieldConfig(grid=HashGridConfig(table_size=1 << 19)))
    field.init_random(1234)
    out = Image(cam.width, cam.height, 3)
    render_rows(field, grid, cam, RenderOptions(), 0, cam.height, out, None, None, stats)

The device work happens in liblumi_cuda.so (paper_2311_02542_b200/csrc); this module only
marshals descriptors and owns device-model caching.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import itertools
import os
import math
import threading
import weakref
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import Error, check

__all__ = [
    "Error", "HashGridConfig", "ColorSpaceMode", "FieldConfig", "RadianceField", "OccupancyGrid",
    "ContractionMode", "CameraModel", "RenderOptions", "RowStats", "Image", "DeviceModel",
    "render_rows", "lod_levels_of", "device_info",
]


def _p(a) -> Optional[int]:
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# Content versions come from ONE process-wide counter, so a new object never repeats a version a
# dead object (whose id() Python may reuse) had: a cached device copy can only match the object
# and the edit it was made from.
_versions = itertools.count(1)


@dataclass
class HashGridConfig:
    """proj/include/lumi/grid.h:18-29 (note the reference default table_size = 2^15)."""

    levels: int = 16
    features_per_level: int = 2
    base_resolution: int = 128
    per_level_scale: float = 1.4
    table_size: int = 1 << 15

    def resolution(self, level: int) -> int:
        return int(math.floor(self.base_resolution * math.pow(self.per_level_scale, level)))

    def feature_dim(self) -> int:
        return self.levels * self.features_per_level


class ColorSpaceMode(enum.IntEnum):
    kPq = 0
    kLinear = 1


@dataclass
class FieldConfig:
    """proj/include/lumi/field.h:22-27."""

    grid: HashGridConfig = dc_field(default_factory=HashGridConfig)
    hidden_width: int = 64
    bottleneck: int = 16
    color_space: ColorSpaceMode = ColorSpaceMode.kPq

    def desc(self) -> _abi.FieldDesc:
        g = self.grid
        return _abi.FieldDesc(g.levels, g.features_per_level, g.base_resolution, self.hidden_width,
                              float(g.per_level_scale), int(g.table_size), self.bottleneck,
                              int(self.color_space), 0)


def layout_of(cfg: FieldConfig) -> _abi.GridLayout:
    lay = _abi.GridLayout()
    d = cfg.desc()
    check(_abi.lib().lumi_field_layout(C.byref(d), C.byref(lay)))
    return lay


class RadianceField:
    """Host parameters of RadianceField<float> (field.h:65-209) in the reference layout:
    one float grid table (grid.h:58-74) and per-net flattened weights-then-bias
    (network.h:144-151)."""

    Scalar = np.float32
    kShDim = 16

    def __init__(self, cfg: FieldConfig = None):
        self.cfg = cfg or FieldConfig()
        self.layout = layout_of(self.cfg)
        self.grid_params = np.zeros(self.layout.total_floats, np.float32)
        self.density_params = np.zeros(self.layout.density_params, np.float32)
        self.color_params = np.zeros(self.layout.color_params, np.float32)
        self.version = next(_versions)

    def config(self) -> FieldConfig:
        return self.cfg

    def _synth(self, seed: int, amp: float) -> None:
        d = self.cfg.desc()
        check(_abi.lib().lumi_synth_params(C.byref(d), int(seed), float(amp), _p(self.grid_params),
                                           _p(self.density_params), _p(self.color_params)))
        self.version = next(_versions)

    def init_random(self, seed: int) -> None:
        """RadianceField::init_random (field.h:88-93), bit-identical pcg32 stream."""
        self._synth(seed, 0.0)

    @classmethod
    def synthetic(cls, cfg: FieldConfig, seed: int, amplitude: float) -> "RadianceField":
        """init_random(seed) then grid <- Rng(seed+1).uniform(-a, a) (trainer.cpp:257-259)."""
        f = cls(cfg)
        f._synth(seed, amplitude)
        return f

    def level_is_dense(self, level: int) -> bool:
        return bool(self.layout.dense[level])

    def parameter_count(self) -> int:
        return int(self.grid_params.size)

    def touch(self) -> None:
        """Call after editing parameters in place so cached device copies refresh."""
        self.version = next(_versions)


class OccupancyGrid:
    """Binary occupancy over the contracted domain [-2,2]^3 (occupancy.h:32-100): one byte per
    voxel, index (iz*res+iy)*res+ix, default all occupied (occupancy.cpp:13-20)."""

    kMaxResolution = 1024

    def __init__(self, resolution: int = 128, bits: Optional[np.ndarray] = None):
        if not (0 < resolution <= self.kMaxResolution):
            raise Error("occupancy: bad resolution")
        self.res = int(resolution)
        n = self.res ** 3
        if bits is None:
            self.bits = np.ones(n, np.uint8)
        else:
            bits = np.ascontiguousarray(bits, dtype=np.uint8).reshape(-1)
            if bits.size != n:
                raise Error("occupancy: bit count does not match resolution")
            self.bits = (bits != 0).astype(np.uint8)
        self.version = next(_versions)

    def resolution(self) -> int:
        return self.res

    def voxel_count(self) -> int:
        return self.res ** 3

    def voxel_index(self, c) -> int:
        """occupancy.cpp:22-29."""
        u, v, w = ((c[0] + 2.0) * 0.25, (c[1] + 2.0) * 0.25, (c[2] + 2.0) * 0.25)
        if u < 0 or u > 1 or v < 0 or v > 1 or w < 0 or w > 1:
            return -1
        r = self.res
        ix, iy, iz = (min(int(u * r), r - 1), min(int(v * r), r - 1), min(int(w * r), r - 1))
        return (iz * r + iy) * r + ix

    def is_occupied(self, c) -> bool:
        i = self.voxel_index(c)
        return i >= 0 and bool(self.bits[i])

    def occupied_bit(self, index: int) -> bool:
        return bool(self.bits[index])

    def occupied_count(self) -> int:
        return int(self.bits.sum())

    def touch(self) -> None:
        self.version = next(_versions)


class ContractionMode(enum.IntEnum):
    kNone = 0
    kLInfCubic = 1


@dataclass
class CameraModel:
    """proj/include/lumi/camera.h:15-23 (pose row-major world <- camera)."""

    rot: Sequence[float] = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
    origin: Sequence[float] = (0.0, 0.0, 0.0)
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    t_near: float = 0.05
    t_far: float = 10.0

    def desc(self) -> _abi.CameraDesc:
        c = _abi.CameraDesc()
        c.rot[:] = [float(v) for v in self.rot]
        c.origin[:] = [float(v) for v in self.origin]
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.t_near, c.t_far = float(self.t_near), float(self.t_far)
        return c

    @classmethod
    def from_spec(cls, spec) -> "CameraModel":
        return cls(tuple(spec.rot), tuple(spec.origin), spec.fx, spec.fy, spec.cx, spec.cy,
                   spec.width, spec.height, spec.t_near, spec.t_far)


@dataclass
class RenderOptions:
    """proj/include/lumi/renderer.h:22-30."""

    samples_per_ray: int = 256
    lod_bias: float = 0.0
    lod_enabled: bool = True
    termination_transmittance: float = 1e-4
    background: Sequence[float] = (0.0, 0.0, 0.0)
    contraction: ContractionMode = ContractionMode.kLInfCubic
    chunk_size: int = 32

    def desc(self) -> _abi.RenderOptionsDesc:
        o = _abi.RenderOptionsDesc()
        o.samples_per_ray = int(self.samples_per_ray)
        o.lod_enabled = 1 if self.lod_enabled else 0
        o.lod_bias = float(self.lod_bias)
        o.termination_transmittance = float(self.termination_transmittance)
        o.background[:] = [float(v) for v in self.background]
        o.contraction = int(self.contraction)
        o.chunk_size = int(self.chunk_size)
        return o


@dataclass
class RowStats:
    """proj/include/lumi/renderer.h:241-246."""

    row: int = 0
    ms: float = 0.0
    rays: int = 0
    evals: int = 0


class Image:
    """Planar channel-major float image (image.h:16-35): data[c, y, x]."""

    def __init__(self, width: int, height: int, channels: int, fill: float = 0.0):
        self.width, self.height, self.channels = int(width), int(height), int(channels)
        self.data = np.full((self.channels, self.height, self.width), fill, np.float32)

    def at(self, x: int, y: int, c: int) -> float:
        return float(self.data[c, y, x])


def device_info(device: int = 0) -> str:
    buf = C.create_string_buffer(256)
    check(_abi.lib().lumi_device_info(device, buf, 256))
    return buf.value.decode()


class DeviceModel:
    """A field + occupancy grid resident on one B200 (LumiModel*)."""

    def __init__(self, field: RadianceField, grid: OccupancyGrid, device: int = 0):
        self.device = device
        self.cfg = field.cfg
        h = C.c_void_p()
        d = field.cfg.desc()
        check(_abi.lib().lumi_model_create(device, C.byref(d), _p(field.grid_params),
                                           _p(field.density_params), _p(field.color_params),
                                           _p(grid.bits), grid.res, C.byref(h)))
        self.h = h
        self.field_version = field.version
        self.grid_version = grid.version
        self.kernel = os.environ.get("LUMI_KERNEL", "ws")
        self._lock = threading.Lock()

    def set_kernel(self, kernel: str) -> None:
        """'ws' (the warp-specialised tcgen05 packet kernel, default) or 'simt' (fp32
        CUDA-core cross-check with bit-exact features)."""
        k = {"tc": _abi.LUMI_KERNEL_TC, "simt": _abi.LUMI_KERNEL_SIMT,
             "packet": _abi.LUMI_KERNEL_PACKET, "ws": _abi.LUMI_KERNEL_WS}[kernel]
        check(_abi.lib().lumi_model_set_kernel(self.h, k))
        self.kernel = kernel

    def set_timing(self, enable: bool) -> None:
        """Record CUDA events around each launch's march pass and render kernel."""
        check(_abi.lib().lumi_model_set_timing(self.h, 1 if enable else 0))

    def take_timing(self):
        """(march_ms, render_ms, launches) summed since the last call (synchronises)."""
        a, b, n = C.c_double(), C.c_double(), C.c_int()
        check(_abi.lib().lumi_model_take_timing(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return float(a.value), float(b.value), int(n.value)

    def set_occupancy(self, grid: OccupancyGrid) -> None:
        check(_abi.lib().lumi_model_set_occupancy(self.h, _p(grid.bits), grid.res))
        self.grid_version = grid.version

    def close(self) -> None:
        if getattr(self, "h", None):
            _abi.lib().lumi_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def nbytes(self) -> int:
        v = C.c_uint64()
        check(_abi.lib().lumi_model_bytes(self.h, C.byref(v)))
        return int(v.value)

    # -- rendering -------------------------------------------------------------------
    def render_rows(self, cam: CameraModel, opts: RenderOptions, row_begin: int, row_end: int,
                    out: np.ndarray, depth: Optional[np.ndarray] = None,
                    opacity: Optional[np.ndarray] = None,
                    stats: Optional[List[RowStats]] = None) -> None:
        """Synchronous, host buffers (renderer.h:252-278 semantics)."""
        W, H = cam.width, cam.height
        for name, a, shape in (("out", out, (3, H, W)), ("depth", depth, (H, W)),
                               ("opacity", opacity, (H, W))):
            if a is not None and (a.dtype != np.float32 or a.size != int(np.prod(shape)) or
                                  not a.flags.c_contiguous):
                raise Error(f"render_rows: {name} must be a contiguous float32 image of {shape}")
        rows = max(row_end - row_begin, 0)
        st = (_abi.RowStatsDesc * max(rows, 1))()
        cd, od = cam.desc(), opts.desc()
        check(_abi.lib().lumi_render_rows(self.h, C.byref(cd), C.byref(od), row_begin, row_end,
                                          _p(out), _p(depth), _p(opacity),
                                          st if stats is not None else None))
        if stats is not None:
            for i in range(rows):
                stats.append(RowStats(st[i].row, st[i].ms, st[i].rays, st[i].evals))

    def render_rows_async(self, cam: CameraModel, opts: RenderOptions, row_begin: int,
                          row_end: int, target: _abi.FrameTarget, stream: int = 0) -> None:
        """Device-resident variant: `target` holds device pointers; enqueued on `stream`."""
        cd, od = cam.desc(), opts.desc()
        check(_abi.lib().lumi_render_rows_async(self.h, C.byref(cd), C.byref(od), row_begin,
                                                row_end, C.byref(target), C.c_void_p(stream)))

    def march_kept_async(self, cam: CameraModel, opts: RenderOptions, row_begin: int,
                         row_end: int, mask_ptr: int, counts_ptr: int, stream: int = 0) -> None:
        cd, od = cam.desc(), opts.desc()
        check(_abi.lib().lumi_march_kept_async(self.h, C.byref(cd), C.byref(od), row_begin,
                                               row_end, C.c_void_p(mask_ptr),
                                               C.c_void_p(counts_ptr), C.c_void_p(stream)))

    def mlp_batch_async(self, features_ptr: int, dirs_ptr: int, n: int, out_ptr: int,
                        stream: int = 0) -> None:
        """The renderer's tcgen05 MLP alone: device features [n][32] fp16 and directions
        [n][3] fp32 -> out [n][4] fp32 (sigma, r, g, b) (field.h:114-136)."""
        check(_abi.lib().lumi_mlp_batch_async(self.h, C.c_void_p(features_ptr),
                                              C.c_void_p(dirs_ptr), int(n),
                                              C.c_void_p(out_ptr), C.c_void_p(stream)))

    def encode_async(self, n: int, pos_ptr: int, lod_ptr: int, out_ptr: int, stream: int = 0) -> None:
        """MultiResHashGrid::encode (grid.h:90-114) through the production gather: contracted
        positions [n][3] fp32 and LOD fl [n] (w_l = clamp(fl - l, 0, 1)) -> [n][2*levels]."""
        check(_abi.lib().lumi_encode_async(self.h, int(n), C.c_void_p(pos_ptr), C.c_void_p(lod_ptr),
                                           C.c_void_p(out_ptr), C.c_void_p(stream)))

    def gather_bench_async(self, n: int, coherent: bool, out_ptr: int, stream: int = 0) -> None:
        """The renderer's hash-grid gather alone over n points x all levels (benchmark)."""
        check(_abi.lib().lumi_gather_bench_async(self.h, int(n), 1 if coherent else 0,
                                                 C.c_void_p(out_ptr), C.c_void_p(stream)))

    def bake_occupancy(self, cams: Sequence[CameraModel], samples_per_ray: int,
                       points_per_axis: int, resolution: int, alpha: float,
                       want_probe: bool = False):
        """OccupancyGrid::probe + prune on the GPU (occupancy.cpp:97-154)."""
        arr = (_abi.CameraDesc * max(len(cams), 1))(*[c.desc() for c in cams])
        n = resolution ** 3
        occ = np.zeros(n, np.uint8)
        pm = np.zeros(n, np.float32) if want_probe else None
        check(_abi.lib().lumi_bake_occupancy(self.h, arr, len(cams), samples_per_ray,
                                             points_per_axis, resolution, float(alpha), _p(occ),
                                             _p(pm)))
        grid = OccupancyGrid(resolution, occ)
        return (grid, pm) if want_probe else grid


_cache_lock = threading.Lock()
# field -> grid -> device -> DeviceModel; both levels are weak, so a dead field or grid drops
# its device copies (and their device memory)
_model_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


class _Lease:
    """A render's hold on a cached DeviceModel: a model replaced while renders still use it is
    closed by the last of them, never under a running render."""

    def __init__(self, m: DeviceModel):
        self.m = m

    def __enter__(self) -> DeviceModel:
        return self.m

    def __exit__(self, *a):
        with _cache_lock:
            self.m._users -= 1
            if self.m._retired and self.m._users == 0:
                self.m.close()


def _retire(m: DeviceModel) -> None:
    # caller holds _cache_lock
    m._retired = True
    if m._users == 0:
        m.close()


def _device_model(field: RadianceField, grid: OccupancyGrid, device: int) -> _Lease:
    with _cache_lock:
        per_grid = _model_cache.setdefault(field, weakref.WeakKeyDictionary())
        per_dev = per_grid.setdefault(grid, {})
        m = per_dev.get(device)
        if m is None or m.field_version != field.version:
            if m is not None:
                _retire(m)
            m = DeviceModel(field, grid, device)
            m._users, m._retired = 0, False
            per_dev[device] = m
        elif m.grid_version != grid.version:
            if m._users == 0:
                m.set_occupancy(grid)
            else:  # in use by another render: give this one a fresh copy
                _retire(m)
                m = DeviceModel(field, grid, device)
                m._users, m._retired = 0, False
                per_dev[device] = m
        m._users += 1
        return _Lease(m)


def render_rows(field: RadianceField, grid: OccupancyGrid, cam: CameraModel, opts: RenderOptions,
                row_begin: int, row_end: int, out, depth_out=None, opacity_out=None,
                stats: Optional[List[RowStats]] = None, device: int = 0) -> None:
    """Drop-in for lumi::render_rows (renderer.h:252-278): renders rows [row_begin, row_end)
    of `cam` into the full-size planar `out` (Image or float32 [3,H,W]); optional depth /
    opacity planes; `stats` is appended one RowStats per row.  Raises Error on a bad row range
    exactly like the reference's require()."""
    def arr(a):
        return None if a is None else (a.data if isinstance(a, Image) else a)

    if not (row_begin >= 0 and row_end <= cam.height and row_begin <= row_end):
        raise Error("render_rows: row range outside image")
    with _device_model(field, grid, device) as m:
        m.render_rows(cam, opts, row_begin, row_end, arr(out), arr(depth_out), arr(opacity_out),
                      stats)


def lod_levels_of(cfg: FieldConfig) -> List[int]:
    return [cfg.grid.resolution(l) for l in range(cfg.grid.levels)]


def load_checkpoint(path: str):
    """Reads a reference LUMICKPT v1 checkpoint (proj/src/scene.cpp:353-394): returns
    (RadianceField, OccupancyGrid, info dict with samples_per_ray / background /
    contraction / n_cameras).  Raises Error with the reference's messages on bad files."""
    L = _abi.lib()
    info = _abi.CheckpointInfo()
    p = str(path).encode()
    check(L.lumi_checkpoint_read(p, C.byref(info), None, None, None, None))
    f = info.field
    cfg = FieldConfig(HashGridConfig(f.levels, f.features_per_level, f.base_resolution,
                                     f.per_level_scale, f.table_size), f.hidden_width,
                      f.bottleneck, ColorSpaceMode(f.color_space))
    field = RadianceField(cfg)
    occ = np.zeros(info.occ_res ** 3, np.uint8)
    check(L.lumi_checkpoint_read(p, C.byref(info), _p(field.grid_params),
                                 _p(field.density_params), _p(field.color_params), _p(occ)))
    field.touch()
    grid = OccupancyGrid(info.occ_res, occ)
    meta = dict(samples_per_ray=info.samples_per_ray, background=tuple(info.background),
                contraction=ContractionMode(info.contraction), n_cameras=info.n_cameras)
    return field, grid, meta


def save_checkpoint(path: str, field: RadianceField, grid: OccupancyGrid,
                    samples_per_ray: int = 256, background=(0.0, 0.0, 0.0),
                    contraction: "ContractionMode" = ContractionMode.kLInfCubic,
                    camera_alpha_v=()) -> None:
    """save_checkpoint (proj/src/scene.cpp:320-351) of a rendering model in the reference's
    LUMICKPT v1 format (the occupancy grid's training trackers are written as zeros)."""
    info = _abi.CheckpointInfo()
    info.field = field.cfg.desc()
    info.samples_per_ray = int(samples_per_ray)
    info.contraction = int(contraction)
    info.background[:] = [float(v) for v in background]
    info.occ_res = grid.res
    av = np.ascontiguousarray(camera_alpha_v, np.float64)
    info.n_cameras = int(av.size)
    check(_abi.lib().lumi_checkpoint_write(str(path).encode(), C.byref(info), _p(field.grid_params),
                                           _p(field.density_params), _p(field.color_params),
                                           _p(av) if av.size else None, _p(grid.bits)))
