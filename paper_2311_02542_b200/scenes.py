"""Synthetic VR-NeRF scenes and eyebuffer camera rigs (BASELINE.json configs C1-C5).

The reference ships no trained model, so every config renders a seeded synthetic
"bake":

* parameters: ``RadianceField<float>::init_random(seed)`` (proj/include/lumi/field.h:88-93,
  pcg32 He-normal nets, network.h:73-78) followed by a grid overwrite with
  ``Rng(seed + 1).uniform(-amp, amp)`` (the pattern of proj/src/trainer.cpp:257-259);
* occupancy: a 128^3 ``OccupancyGrid::probe`` (k = 2 points per axis, all-ones LOD,
  density head only; occupancy.cpp:97-142, trainer.cpp:651-657) + ``prune(alpha)``
  (occupancy.cpp:144-154) from one probe camera.

This module is plain data; it does not load the CUDA library.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

# -- model recipe -------------------------------------------------
SEED = 1234
GRID_AMPLITUDE = 1.0
PRUNE_ALPHA = 2.0
PROBE_POINTS_PER_AXIS = 2
OCC_RES = 128
SAMPLES_PER_RAY = 256

# probe / hero camera: camera z -> world +y, camera y -> world -z
PROBE_ROT = (1.0, 0.0, 0.0, 0.0, 0.0, -1.0, 0.0, 1.0, 0.0)
PROBE_ORIGIN = (0.1, -0.3, 0.05)
T_NEAR, T_FAR = 0.05, 10.0

# interpupillary offset along camera x
EYE_HALF_IPD = 0.032


@dataclass(frozen=True)
class ModelSpec:
    name: str
    table_log2: int
    levels: int = 16
    features_per_level: int = 2
    base_resolution: int = 128
    per_level_scale: float = 1.4
    hidden_width: int = 64
    bottleneck: int = 16
    seed: int = SEED
    amplitude: float = GRID_AMPLITUDE
    prune_alpha: float = PRUNE_ALPHA
    occ_res: int = OCC_RES
    dense_occupancy: bool = False  # C5 stress: all voxels occupied

    @property
    def table_size(self) -> int:
        return 1 << self.table_log2


SMALL = ModelSpec("small-T19", 19)  # C1, C2
FULL = ModelSpec("full-T22", 22)  # C3, C4
STRESS = ModelSpec("full-T22-dense", 22, dense_occupancy=True)  # C5


@dataclass(frozen=True)
class CameraSpec:
    rot: tuple
    origin: tuple
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    t_near: float = T_NEAR
    t_far: float = T_FAR


def pinhole(width: int, height: int, rot=PROBE_ROT, origin=PROBE_ORIGIN) -> CameraSpec:
    """fx = fy = 0.6 * size, principal point at the centre (proj/src/presets.cpp:36-48)."""
    f = 0.6 * width
    return CameraSpec(tuple(rot), tuple(origin), f, f, width / 2.0, height / 2.0, width, height)


def _matmul3(a, b):
    return tuple(sum(a[3 * i + k] * b[3 * k + j] for k in range(3)) for i in range(3) for j in range(3))


def _rot_yaw_pitch(yaw: float, pitch: float):
    """Camera-frame rotation: yaw about camera y, then pitch about camera x."""
    cy, sy, cp, sp = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch)
    ry = (cy, 0.0, sy, 0.0, 1.0, 0.0, -sy, 0.0, cy)
    rx = (1.0, 0.0, 0.0, 0.0, cp, -sp, 0.0, sp, cp)
    return _matmul3(ry, rx)


def head_pose(frame: int, frames: int = 120):
    """Deterministic head-motion path (C4): a yaw/pitch sweep with a small translation that
    stays inside the unit cube.  Returns (rot row-major world<-head, origin)."""
    ph = 2.0 * math.pi * frame / max(frames, 1)
    yaw = 0.35 * math.sin(ph)
    pitch = 0.12 * math.sin(2.0 * ph)
    rot = _matmul3(PROBE_ROT, _rot_yaw_pitch(yaw, pitch))
    origin = (PROBE_ORIGIN[0] + 0.05 * math.sin(ph), PROBE_ORIGIN[1] + 0.03 * math.cos(ph),
              PROBE_ORIGIN[2] + 0.02 * math.sin(3.0 * ph))
    return rot, origin


def eye_cameras(size: int, rot=PROBE_ROT, origin=PROBE_ORIGIN):
    """Left/right eyebuffer cameras: the head pose offset by -/+ half the IPD along the
    head's x axis (world offset = R * (+-ipd/2, 0, 0))."""
    eyes = []
    for s in (-1.0, 1.0):
        off = (rot[0] * s * EYE_HALF_IPD, rot[3] * s * EYE_HALF_IPD, rot[6] * s * EYE_HALF_IPD)
        o = (origin[0] + off[0], origin[1] + off[1], origin[2] + off[2])
        eyes.append(pinhole(size, size, rot, o))
    return eyes


# -- BASELINE.json configs ------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    key: str
    description: str
    model: ModelSpec
    eye_size: int
    eyes: int
    frames: int = 1


CONFIGS = {
    "C1": Config("C1", "small model @ 256x256, one camera (CPU-runnable)", SMALL, 256, 1),
    "C2": Config("C2", "small model @ one 2048x2048 eyebuffer", SMALL, 2048, 1),
    "C3": Config("C3", "full model (T=2^22, LOD on), dual 2Kx2K eyebuffers", FULL, 2048, 2),
    "C4": Config("C4", "dual 2Kx2K, dynamic row balancing, 120-frame head path", FULL, 2048, 2,
                 frames=120),
    "C5": Config("C5", "stress: 4Kx4K per eye, dense occupancy", STRESS, 4096, 2),
}


# -- synthetic training batches (the reverse path) ----------------
def _ray_dir(cam: CameraSpec, px: float, py: float):
    """generate_ray (proj/src/camera.cpp:10-24): dir = normalize(R * ((px-cx)/fx, (py-cy)/fy, 1))."""
    x, y = (px - cam.cx) / cam.fx, (py - cam.cy) / cam.fy
    r = cam.rot
    d = ((r[0] * x + r[1] * y) + r[2], (r[3] * x + r[4] * y) + r[5], (r[6] * x + r[7] * y) + r[8])
    n = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    return (d[0] / n, d[1] / n, d[2] / n)


def train_cameras(size: int = 256, count: int = 4):
    """Training views: `count` poses of the head path at eyebuffer size `size`."""
    return [pinhole(size, size, *head_pose(i * 120 // max(count, 1))) for i in range(count)]


def train_batch(cams, rays_per_camera: int, seed: int = 7, depth_fraction: float = 0.5):
    """A seeded synthetic TrainRay batch (trainer.h:90-97) as a numpy structured array with
    the LumiTrainRay / lo_train_ray layout: pixels uniform over each camera, the right
    neighbour at x + 1.5 (renderer.h:264-265), PQ-space targets uniform in [0, 1), a
    ground-truth depth on `depth_fraction` of the rays (else -1), vignette radius
    |p - c| / |c| (the normalised radius trainer.cpp uses)."""
    import numpy as np
    from .train import TRAIN_RAY_DTYPE

    rng = np.random.default_rng(seed)
    out = np.zeros(len(cams) * rays_per_camera, TRAIN_RAY_DTYPE)
    k = 0
    for ci, cam in enumerate(cams):
        px = rng.integers(0, cam.width, rays_per_camera)
        py = rng.integers(0, cam.height, rays_per_camera)
        for x, y in zip(px.tolist(), py.tolist()):
            r = out[k]
            r["origin"] = cam.origin
            r["norigin"] = cam.origin
            r["dir"] = _ray_dir(cam, x + 0.5, y + 0.5)
            r["ndir"] = _ray_dir(cam, x + 1.5, y + 0.5)
            r["camera"] = ci
            k += 1
        sl = slice(k - rays_per_camera, k)
        out["gt"][sl] = rng.random((rays_per_camera, 3), dtype=np.float32)
        has_d = rng.random(rays_per_camera) < depth_fraction
        out["gt_depth"][sl] = np.where(has_d, rng.uniform(0.3, 3.0, rays_per_camera), -1.0)
        rx = (px + 0.5 - cam.cx) / cam.cx
        ry = (py + 0.5 - cam.cy) / cam.cy
        out["vignette_r"][sl] = np.sqrt(rx * rx + ry * ry) / math.sqrt(2.0)
    return out
