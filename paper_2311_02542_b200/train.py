"""Training-side reverse of the rendering path on the GPU.

Mirrors the per-ray body of the reference training loop (proj/src/trainer.cpp:549-561):
``march_ray(record = true)`` (renderer.h:126-237) -> ``ray_loss`` (train_step.h:16-123) ->
``backward_ray`` (train_step.h:127-154: ``composite_backward_sigma`` renderer.h:110-120,
``RadianceField::backward_chunk`` field.h:141-179, ``Mlp::backward`` network.h:115-136,
``MultiResHashGrid::encode_backward`` grid.h:118-137), accumulated into ``FieldGradients``
(field.h:48-62).  The optimizer (``adam_step``, simd.h:106-121) and the training loop are out
of scope; tools/device_trainer.py shows a device-resident loop
built on this reverse path.
"""
from __future__ import annotations

import numpy as np

# LumiTrainRay (include/lumi_cuda.h) == TrainRay (trainer.h:90-97) flattened
TRAIN_RAY_DTYPE = np.dtype([
    ("origin", "<f8", (3,)), ("dir", "<f8", (3,)),
    ("norigin", "<f8", (3,)), ("ndir", "<f8", (3,)),
    ("gt", "<f4", (3,)), ("camera", "<i4"),
    ("gt_depth", "<f8"), ("vignette_r", "<f8"),
], align=True)
assert TRAIN_RAY_DTYPE.itemsize == 128

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _abi
from ._abi import Error, check
from .renderer import CameraModel, DeviceModel, RenderOptions


def _p(a) -> Optional[int]:
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class TrainConfig:
    """The reverse-path fields of TrainConfig (proj/include/lumi/trainer.h:18-60)."""

    lr_grid: float = 0.01
    lr_net: float = 0.005
    beta1: float = 0.9
    beta2: float = 0.99
    adam_eps: float = 1e-15
    samples_per_ray: int = 256
    termination_transmittance: float = 1e-4
    lambda_depth: float = 0.1
    lambda_dvar: float = 0.01
    lambda_dist: float = 0.001

    def loss_desc(self, inv_batch: float, depth_active: bool) -> _abi.LossConfig:
        return _abi.LossConfig(float(self.lambda_depth), float(self.lambda_dvar),
                               float(self.lambda_dist), float(inv_batch),
                               1 if depth_active else 0, 0)


@dataclass
class LossTerms:
    """LossTerms (trainer.h:99-102), the ray-dependent part."""

    total: float = 0.0
    image: float = 0.0
    depth: float = 0.0
    dvar: float = 0.0
    dist: float = 0.0


class FieldGradients:
    """FieldGradients<float> (field.h:48-62) on the host: grid, density, color."""

    def __init__(self, layout: _abi.GridLayout):
        self.grid = np.zeros(layout.total_floats, np.float32)
        self.density = np.zeros(layout.density_params, np.float32)
        self.color = np.zeros(layout.color_params, np.float32)

    def zero(self) -> None:
        self.grid[:] = 0
        self.density[:] = 0
        self.color[:] = 0


def _cam_tnf(cameras: Sequence[CameraModel]) -> np.ndarray:
    return np.ascontiguousarray([[c.t_near, c.t_far] for c in cameras], np.float64)


def _check_rays(rays: np.ndarray) -> np.ndarray:
    if not isinstance(rays, np.ndarray) or rays.dtype != TRAIN_RAY_DTYPE:
        raise Error("rays must be a numpy array of TRAIN_RAY_DTYPE (LumiTrainRay)")
    return np.ascontiguousarray(rays)


def train_backward(model: DeviceModel, rays: np.ndarray, cameras: Sequence[CameraModel],
                   alpha_v: Sequence[float], opts: RenderOptions, cfg: TrainConfig,
                   grads: FieldGradients, alpha_grad: np.ndarray, depth_active: bool = True,
                   inv_batch: Optional[float] = None):
    """The training loop's per-ray body over a batch (trainer.cpp:549-562) on the GPU, host
    buffers: march_ray(record) + ray_loss + backward_ray, gradients ACCUMULATED into `grads`
    and `alpha_grad` ([len(cameras)] float64).  Returns (LossTerms summed over the rays,
    evals[n] = rec.t.size(), contributing[n])."""
    rays = _check_rays(rays)
    n = int(rays.shape[0])
    tnf = _cam_tnf(cameras)
    av = np.ascontiguousarray(alpha_v, np.float64)
    if av.size != len(cameras) or alpha_grad.dtype != np.float64 or alpha_grad.size != len(cameras):
        raise Error("alpha_v / alpha_grad need one float64 entry per camera")
    loss = _abi.LossTermsDesc()
    g = _abi.TrainGrads(_p(grads.grid), _p(grads.density), _p(grads.color), _p(alpha_grad),
                        C.addressof(loss))
    lc = cfg.loss_desc(1.0 / max(n, 1) if inv_batch is None else inv_batch, depth_active)
    od = opts.desc()
    ev = np.zeros(max(n, 1), np.int32)
    co = np.zeros(max(n, 1), np.int32)
    check(_abi.lib().lumi_train_backward(model.h, _p(rays), n, _p(tnf), _p(av), len(cameras),
                                         C.byref(od), C.byref(lc), C.byref(g), _p(ev), _p(co)))
    return (LossTerms(loss.total, loss.image, loss.depth, loss.dvar, loss.dist), ev[:n], co[:n])
