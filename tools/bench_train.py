#!/usr/bin/env python
"""Training-side reverse path benchmark: one optimisation iteration of
the reference's batch shape -- 50 images x 256 rays = 12,800 rays (trainer.h:20-21) -- on the
full T=2^22 synthetic model, through the C ABI with device-resident rays and gradients.

  python tools/bench_train.py [--steps K --warmup W] [--rays-per-camera 256 --cameras 50]

Reports (one JSON line): rays/s of lumi_train_backward_async (march(record) + ray_loss +
backward_ray, the body of trainer.cpp:549-561), the Adam update of all 65M+ grid and 9.7K
network parameters (trainer.cpp:612-625), and the whole iteration; next to the reference's
own CPU path (oracle/_ref ref_train_backward: the same templates the reference trainer
runs, single-threaded as train() is) on the same batch.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cameras", type=int, default=50)
    ap.add_argument("--rays-per-camera", type=int, default=256)
    ap.add_argument("--image", type=int, default=2048)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()

    import torch
    import paper_2311_02542_b200 as L
    from paper_2311_02542_b200 import _abi, scenes, train as T
    sys.path.insert(0, ROOT)
    from bench import load_scene

    spec = scenes.FULL
    field, grid = load_scene(spec)
    dm = L.DeviceModel(field, grid, 0)
    cams = scenes.train_cameras(a.image, a.cameras)
    rays = scenes.train_batch(cams, a.rays_per_camera, seed=3)
    n = len(rays)
    cmodels = [L.CameraModel.from_spec(c) for c in cams]
    av = np.linspace(0.0, 0.2, a.cameras)
    cfg = T.TrainConfig()
    import device_trainer as DT
    tr = DT.DeviceTrainer(dm, cmodels, cfg, av)
    d_rays = torch.from_numpy(rays.view(np.uint8).reshape(-1, 128)).cuda()
    lib = _abi.lib()
    g = _abi.TrainGrads(tr.grads[0].data_ptr(), tr.grads[1].data_ptr(), tr.grads[2].data_ptr(),
                        tr.alpha_grad.data_ptr(), tr.loss.data_ptr())
    tnf = np.ascontiguousarray([[c.t_near, c.t_far] for c in cmodels], np.float64)
    lc = cfg.loss_desc(1.0 / n, True)
    od = L.RenderOptions().desc()
    evals = torch.zeros(n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream

    def backward():
        for b in (*tr.grads, tr.alpha_grad, tr.loss):
            b.zero_()
        _abi.check(lib.lumi_train_backward_async(dm.h, d_rays.data_ptr(), n, tnf.ctypes.data,
                                                 av.ctypes.data, a.cameras, C.byref(od),
                                                 C.byref(lc), C.byref(g), evals.data_ptr(), None,
                                                 stream))

    def adam(t):
        for k, (p, size) in enumerate(zip(tr.param_views, tr.sizes)):
            lr = cfg.lr_grid if k == 0 else cfg.lr_net
            DT.adam_step(torch, p, tr.grads[k], tr.m[k], tr.v[k], lr, cfg.beta1, cfg.beta2,
                         cfg.adam_eps, DT.adam_c(cfg.beta1, t), DT.adam_c(cfg.beta2, t))

    def timed(fn, steps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for i in range(steps):
            fn(i + 1)
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / steps

    for i in range(a.warmup):
        backward()
        adam(i + 1)
    ms_bwd = timed(lambda t: backward(), a.steps)
    ev_total = int(evals.sum().item())
    ms_adam = timed(adam, a.steps)
    # the whole device iteration through the public API (DeviceTrainer.step: zero, backward,
    # Adam, refresh of the renderer's fp16 table / fused layer, loss read back)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        tr.step(d_rays)
    torch.cuda.synchronize()
    ms_iter = (time.perf_counter() - t0) * 1e3 / a.steps

    out = {
        "metric": "training iteration (reference batch: 50 images x 256 rays), full T=2^22 model",
        "rays_per_iteration": n, "evaluated_samples": ev_total,
        "backward_ms": round(ms_bwd, 3), "backward_Mrays_s": round(n / ms_bwd / 1e3, 3),
        "backward_Msamples_s": round(ev_total / ms_bwd / 1e3, 2),
        "adam_ms": round(ms_adam, 3),
        "adam_GBs": round(28 * sum(tr.sizes) / ms_adam / 1e6, 1),
        "iteration_ms": round(ms_iter, 3),
        "steps": a.steps, "warmup": a.warmup, "device": torch.cuda.get_device_name(0),
    }
    if not a.no_cpu:
        import oracle as O
        ref = O.Reference()
        ocfg = O.field_config(table_size=spec.table_size)
        params = O.Params(ocfg, field.grid_params, field.density_params, field.color_params)
        rm = ref.model(params, grid.bits, grid.res)
        sub = rays[: max(1, n // 8)]  # bounded sample: one eighth of the batch
        t0 = time.perf_counter()
        ref.train_backward(rm, tnf, av, sub, O.render_options(),
                           O.loss_config(inv_batch=1.0 / n))
        cpu_s = time.perf_counter() - t0
        out["cpu_reference"] = {"rays_per_s": round(len(sub) / cpu_s, 1), "cores": 1,
                                "kind": "reference", "simd": ref.simd_name(),
                                "sample": f"ref_train_backward over {len(sub)} rays of the batch "
                                          f"({cpu_s:.2f} s), single thread as train() runs"}
        out["speedup_backward_vs_cpu"] = round(n / ms_bwd * 1e3 / (len(sub) / cpu_s), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
