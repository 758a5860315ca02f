"""GPU parity of the training reverse path through the C ABI against
the oracle (tests/test_train_oracle.py pins the oracle bit-exactly to the reference).

Tolerances (floating point; the reference's own gradient checks use relative error):
* per-ray evaluated / contributing sample counts: identical (the march is exact double
  and the GPU forward reproduces the reference's AVX-512 accumulation order);
* loss terms: relative 1e-6;
* gradients: max |g_gpu - g_oracle| <= 1e-4 * max |g_oracle| per parameter group (the GPU
  sums in a different order: 128-sample tiles and fp32 atomics instead of 32-sample chunks);
"""
import numpy as np
import pytest

import oracle as O
from conftest import load_occ
from paper_2311_02542_b200 import scenes

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-4
LOSS_RTOL = 1e-6


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch


@pytest.fixture(scope="module")
def L():
    import paper_2311_02542_b200 as lumi
    return lumi


def _models(L, oracle, spec, color_space=0):
    cfg = L.FieldConfig(grid=L.HashGridConfig(spec.levels, spec.features_per_level,
                                              spec.base_resolution, spec.per_level_scale,
                                              spec.table_size),
                        color_space=L.ColorSpaceMode(color_space))
    field = L.RadianceField.synthetic(cfg, spec.seed, spec.amplitude)
    bits, res, _ = load_occ(spec.name)
    dm = L.DeviceModel(field, L.OccupancyGrid(res, bits), 0)
    ocfg = O.field_config(spec.levels, spec.features_per_level, spec.base_resolution,
                          spec.per_level_scale, spec.table_size, spec.hidden_width,
                          spec.bottleneck, color_space)
    params = O.Params(ocfg, field.grid_params, field.density_params, field.color_params)
    return field, dm, oracle.model(params, bits, res)


def _compare(L, oracle, dm, om, rays, cams, av, ropts, oopts, lcfg, depth_active=True):
    from paper_2311_02542_b200 import train as T
    grads = T.FieldGradients(dm_layout(L, dm))
    ag = np.zeros(len(cams), np.float64)
    loss, ev, co = T.train_backward(dm, rays, [L.CameraModel.from_spec(c) for c in cams], av,
                                    ropts, lcfg, grads, ag, depth_active=depth_active)
    tnf = np.array([[c.t_near, c.t_far] for c in cams])
    lc = O.loss_config(lcfg.lambda_depth, lcfg.lambda_dvar, lcfg.lambda_dist, 1.0 / len(rays),
                       depth_active)
    og, ol, oev, oco = oracle.train_backward(om, tnf, av, rays, oopts, lc)
    assert np.array_equal(ev, oev), f"evals differ on {(ev != oev).sum()} rays"
    assert np.array_equal(co, oco), f"contributing differ on {(co != oco).sum()} rays"
    for k in ("total", "image", "depth", "dvar", "dist"):
        assert getattr(loss, k) == pytest.approx(getattr(ol, k), rel=LOSS_RTOL, abs=1e-12), k
    for k, mine in (("grid", grads.grid), ("density", grads.density), ("color", grads.color)):
        ref = og[k]
        scale = float(np.abs(ref).max())
        err = float(np.abs(mine - ref).max())
        assert scale > 0, k
        assert err <= GRAD_RTOL * scale, f"{k}: max err {err:.3e} vs scale {scale:.3e}"
    assert np.allclose(ag, og["alpha"], rtol=LOSS_RTOL, atol=1e-12)
    return loss, ev


def dm_layout(L, dm):
    from paper_2311_02542_b200 import _abi
    import ctypes as C
    lay = _abi.GridLayout()
    d = dm.cfg.desc()
    _abi.check(_abi.lib().lumi_field_layout(C.byref(d), C.byref(lay)))
    return lay


@pytest.mark.parametrize("case", ["default", "no_cut_lod_off", "chunk7_bias", "linear_head"])
def test_train_backward_matches_oracle(L, torch_cuda, oracle, case):
    from paper_2311_02542_b200 import train as T
    cs = {"linear_head": 1}.get(case, 0)
    field, dm, om = _models(L, oracle, scenes.SMALL, cs)
    cams = scenes.train_cameras(256, 3)
    rays = scenes.train_batch(cams, 96, seed=11)
    av = np.array([0.0, 0.05, 0.1])
    o = dict(default=dict(background=(0.1, 0.2, 0.3)),
             no_cut_lod_off=dict(termination_transmittance=0.0, lod_enabled=False),
             chunk7_bias=dict(chunk_size=7, lod_bias=-1.5), linear_head=dict())[case]
    ropts = L.RenderOptions(**o)
    oopts = O.render_options(**o)
    lcfg = T.TrainConfig(lambda_dvar=0.0 if case == "linear_head" else 0.01)
    loss, ev = _compare(L, oracle, dm, om, rays, cams, av, ropts, oopts, lcfg,
                        depth_active=(case != "chunk7_bias"))
    assert ev.sum() > 0 and loss.total > 0


def test_train_backward_per_camera_sampling_intervals(L, torch_cuda, oracle):
    """Cameras with their own (t_near, t_far) (trainer.cpp:553 marches each ray with its
    camera's interval): per-camera sample distances, 128 samples per ray."""
    import dataclasses
    from paper_2311_02542_b200 import train as T
    field, dm, om = _models(L, oracle, scenes.SMALL)
    cams = scenes.train_cameras(192, 3)
    cams = [dataclasses.replace(c, t_near=tn, t_far=tf)
            for c, (tn, tf) in zip(cams, [(0.05, 10.0), (0.2, 2.5), (0.1, 6.0)])]
    rays = scenes.train_batch(cams, 64, seed=21)
    o = dict(samples_per_ray=128)
    loss, ev = _compare(L, oracle, dm, om, rays, cams, np.array([0.02, 0.0, 0.07]),
                        L.RenderOptions(**o), O.render_options(**o), T.TrainConfig())
    assert ev.sum() > 0


def test_train_backward_reference_batch_full_model(L, torch_cuda, oracle):
    """The reference's batch shape (50 images x 256 rays, trainer.h:20-21) on the full
    T=2^22 model (dense level 0)."""
    from paper_2311_02542_b200 import train as T
    field, dm, om = _models(L, oracle, scenes.FULL)
    cams = scenes.train_cameras(256, 50)
    rays = scenes.train_batch(cams, 256, seed=3)
    av = np.linspace(0.0, 0.2, 50)
    loss, ev = _compare(L, oracle, dm, om, rays, cams, av, L.RenderOptions(),
                        O.render_options(), T.TrainConfig())
    assert ev.sum() > 10000


def test_empty_batch_and_empty_grid(L, torch_cuda, oracle):
    from paper_2311_02542_b200 import train as T
    field, dm, om = _models(L, oracle, scenes.SMALL)
    cams = scenes.train_cameras(64, 2)
    g = T.FieldGradients(dm_layout(L, dm))
    ag = np.zeros(2)
    loss, ev, co = T.train_backward(dm, scenes.train_batch(cams, 0), [L.CameraModel.from_spec(c) for c in cams],
                                    [0.0, 0.0], L.RenderOptions(), T.TrainConfig(), g, ag)
    assert loss.total == 0 and not g.grid.any()
    dm.set_occupancy(L.OccupancyGrid(128, np.zeros(128 ** 3, np.uint8)))
    rays = scenes.train_batch(cams, 16)
    loss, ev, co = T.train_backward(dm, rays, [L.CameraModel.from_spec(c) for c in cams],
                                    [0.0, 0.0], L.RenderOptions(background=(0.5, 0.5, 0.5)),
                                    T.TrainConfig(), g, ag)
    assert (ev == 0).all() and not g.grid.any() and loss.image > 0


def test_bad_camera_interval_raises(L, torch_cuda, oracle):
    from paper_2311_02542_b200 import train as T
    field, dm, om = _models(L, oracle, scenes.SMALL)
    cams = scenes.train_cameras(64, 1)
    bad = L.CameraModel.from_spec(cams[0])
    bad.t_far = bad.t_near
    g = T.FieldGradients(dm_layout(L, dm))
    with pytest.raises(L.Error):
        T.train_backward(dm, scenes.train_batch(cams, 4), [bad], [0.0], L.RenderOptions(),
                         T.TrainConfig(), g, np.zeros(1))


def test_device_trainer_steps_reduce_loss_and_refresh_renderer(L, torch_cuda, oracle):
    """A few device-resident iterations (backward + Adam in place + refresh of the renderer's
    fp16 / fused copies) on a fixed batch lower the loss; the production renderer then renders
    the updated field (its pixels agree with the SIMT cross-check kernel)."""
    import os
    import sys
    from paper_2311_02542_b200 import train as T
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from device_trainer import DeviceTrainer
    field, dm, om = _models(L, oracle, scenes.SMALL)
    cams = scenes.train_cameras(128, 2)
    rays = scenes.train_batch(cams, 512, seed=9)
    tr = DeviceTrainer(dm, [L.CameraModel.from_spec(c) for c in cams], T.TrainConfig(),
                         [0.0, 0.0])
    losses = [tr.step(rays).total for _ in range(8)]
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
    cam = L.CameraModel.from_spec(cams[0])
    out = {}
    for k in ("ws", "simt"):
        dm.set_kernel(k)
        img = np.zeros((3, cam.height, cam.width), np.float32)
        dm.render_rows(cam, L.RenderOptions(), 0, cam.height, img)
        out[k] = img
    assert np.abs(out["ws"] - out["simt"]).max() < 1e-3
