"""A device-resident training loop over the GPU reverse path (tool, not product).

The reverse path itself -- march_ray(record) + ray_loss + backward_ray (trainer.cpp:549-561)
-- is paper_2311_02542_b200.train.train_backward / lumi_train_backward_async.  The optimizer
(simd::adam_step, simd.h:106-121; trainer.cpp:228-235) and the loop are outside the rendering
path's scope, so this module keeps them in torch.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import sys
from typing import Optional, Sequence

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_02542_b200 import _abi  # noqa: E402
from paper_2311_02542_b200._abi import check  # noqa: E402
from paper_2311_02542_b200.renderer import CameraModel, DeviceModel, RenderOptions  # noqa: E402
from paper_2311_02542_b200.train import (LossTerms, TrainConfig, _cam_tnf, _check_rays,  # noqa: E402
                                         _p)


def _device_view(torch, ptr: int, n: int, dev):
    """A float32 torch view of n floats of device memory owned by the model."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3}
    return torch.as_tensor(_Arr(), device=dev)


def adam_step(torch, p, g, m, v, lr, beta1, beta2, eps, c1, c2) -> None:
    """simd::adam_step (simd.h:106-121) with trainer.cpp:230-231's bias corrections c1, c2."""
    m.mul_(beta1).add_(g, alpha=1.0 - beta1)
    v.mul_(beta2).addcmul_(g, g, value=1.0 - beta2)
    p.sub_(lr * (m * c1) / (torch.sqrt(v * c2) + eps))


def adam_c(beta: float, t: int) -> float:
    """1 / (1 - beta^t) as trainer.cpp:230-231 computes it (double, then float)."""
    return float(np.float32(1.0 / (1.0 - math.pow(beta, t))))


class DeviceTrainer:
    """A device-resident optimisation step over a DeviceModel: zero the gradients, run the
    reverse path for a batch of rays, apply Adam to the grid and both networks in place
    (trainer.cpp:547-625, the field-parameter part), refresh the renderer's derived copies.
    Device memory and the Adam update come from torch (the optimizer is outside the rendering
    path's scope); the reverse path is liblumi_cuda.so's."""

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
        self.param_views = [_device_view(torch, ptr, k, dev) for ptr, k in zip(self.params, sizes)]
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
        for k, (p, size) in enumerate(zip(self.param_views, self.sizes)):
            lr = c.lr_grid if k == 0 else c.lr_net
            adam_step(torch, p, self.grads[k], self.m[k], self.v[k], lr, c.beta1, c.beta2,
                      c.adam_eps, adam_c(c.beta1, self.t), adam_c(c.beta2, self.t))
        check(L.lumi_model_params_updated(self.model.h))
        lv = self.loss.cpu().numpy()
        return LossTerms(*map(float, lv))
