"""Training-side reverse of the rendering path on the GPU.

Mirrors the per-ray body of the reference training loop (proj/src/trainer.cpp:549-561):
``march_ray(record = true)`` (renderer.h:126-237) -> ``ray_loss`` (train_step.h:16-123) ->
``backward_ray`` (train_step.h:127-154: ``composite_backward_sigma`` renderer.h:110-120,
``RadianceField::backward_chunk`` field.h:141-179, ``Mlp::backward`` network.h:115-136,
``MultiResHashGrid::encode_backward`` grid.h:118-137), accumulated into ``FieldGradients``
(field.h:48-62), plus the ``adam_step`` update (simd.h:106-121, trainer.cpp:228-235).
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


def adam_c(beta: float, t: int) -> float:
    """1 / (1 - beta^t) as trainer.cpp:230-231 computes it (double, then float)."""
    return float(np.float32(1.0 / (1.0 - math.pow(beta, t))))


class DeviceTrainer:
    """A device-resident optimisation step over a DeviceModel: zero the gradients, run the
    reverse path for a batch of rays, apply Adam to the grid and both networks in place
    (trainer.cpp:547-625, the field-parameter part), refresh the renderer's derived copies.
    Device memory comes from torch (plumbing); every kernel is in liblumi_cuda.so."""

    def __init__(self, model: DeviceModel, cameras: Sequence[CameraModel], cfg: TrainConfig,
                 alpha_v: Sequence[float]):
        import torch

        self.torch = torch
        self.model, self.cfg = model, cfg
        self.cameras = list(cameras)
        self.alpha_v = np.ascontiguousarray(alpha_v, np.float64)
        dev = torch.device("cuda", model.device)
        lay = _abi.GridLayout()
        d = model.cfg.desc()
        check(_abi.lib().lumi_field_layout(C.byref(d), C.byref(lay)))
        sizes = (int(lay.total_floats), int(lay.density_params), int(lay.color_params))
        z = lambda k: torch.zeros(k, dtype=torch.float32, device=dev)  # noqa: E731
        self.grads = [z(k) for k in sizes]
        self.m = [z(k) for k in sizes]
        self.v = [z(k) for k in sizes]
        self.alpha_grad = torch.zeros(len(self.cameras), dtype=torch.float64, device=dev)
        self.loss = torch.zeros(5, dtype=torch.float64, device=dev)
        t, dp, cp = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(_abi.lib().lumi_model_device_params(model.h, C.byref(t), C.byref(dp), C.byref(cp)))
        self.params = (t.value, dp.value, cp.value)
        self.sizes = sizes
        self.t = 0

    def step(self, rays, depth_active: bool = True, opts: Optional[RenderOptions] = None,
             stream: int = 0) -> LossTerms:
        """One iteration on a device tensor of LumiTrainRay records (uint8 [n, 128]) or a
        host TRAIN_RAY_DTYPE array (copied)."""
        torch = self.torch
        if isinstance(rays, np.ndarray):
            host = _check_rays(rays)
            rays = torch.from_numpy(host.view(np.uint8).reshape(-1, 128)).to(self.grads[0].device)
        n = int(rays.shape[0])
        opts = opts or RenderOptions(samples_per_ray=self.cfg.samples_per_ray,
                                     termination_transmittance=self.cfg.termination_transmittance)
        for b in (*self.grads, self.alpha_grad, self.loss):
            b.zero_()
        g = _abi.TrainGrads(self.grads[0].data_ptr(), self.grads[1].data_ptr(),
                            self.grads[2].data_ptr(), self.alpha_grad.data_ptr(),
                            self.loss.data_ptr())
        tnf = _cam_tnf(self.cameras)
        lc = self.cfg.loss_desc(1.0 / max(n, 1), depth_active)
        od = opts.desc()
        L = _abi.lib()
        check(L.lumi_train_backward_async(self.model.h, rays.data_ptr(), n, _p(tnf),
                                          _p(self.alpha_v), len(self.cameras), C.byref(od),
                                          C.byref(lc), C.byref(g), None, None, stream))
        self.t += 1
        c = self.cfg
        for k, (ptr, size) in enumerate(zip(self.params, self.sizes)):
            lr = c.lr_grid if k == 0 else c.lr_net
            check(L.lumi_adam_step_async(ptr, self.grads[k].data_ptr(), self.m[k].data_ptr(),
                                         self.v[k].data_ptr(), size, lr, c.beta1, c.beta2,
                                         c.adam_eps, adam_c(c.beta1, self.t),
                                         adam_c(c.beta2, self.t), stream))
        check(L.lumi_model_params_updated(self.model.h))
        lv = self.loss.cpu().numpy()
        return LossTerms(*map(float, lv))
