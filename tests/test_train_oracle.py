"""Pins the oracle's restatement of the training reverse path (oracle/lumi_oracle.c
lo_train_backward / lo_adam_step) against the UNMODIFIED reference (oracle/_ref) before it
is trusted as the checker for the GPU reverse path:

* under LUMI_SIMD=scalar (simd_dispatch.cpp:60-70) the reference's dense kernels run the
  scalar order the oracle restates (simd.h:35-121), so every gradient, loss term and
  per-ray count must be BIT-identical;
* under the host's default ISA the forward still matches (the oracle replays the AVX-512 /
  AVX2 forward order) and the backward sums differ only in float summation order.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, load_occ
from paper_2311_02542_b200 import scenes

pytestmark = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")


def _setup(orc, table_log2=19, color_space=0):
    s = scenes.SMALL
    cfg = O.field_config(s.levels, s.features_per_level, s.base_resolution, s.per_level_scale,
                         1 << table_log2, s.hidden_width, s.bottleneck, color_space)
    params = orc.synth_params(cfg, s.seed, s.amplitude)
    bits, res, _ = load_occ(s.name)
    return cfg, params, bits, res


def _batch(ncam=3, per=48, seed=5):
    cams = scenes.train_cameras(256, ncam)
    rays = scenes.train_batch(cams, per, seed=seed)
    tnf = np.array([[c.t_near, c.t_far] for c in cams])
    av = np.linspace(0.0, 0.1, ncam)
    return rays, tnf, av


CASES = {
    "default": dict(opts=dict(background=(0.1, 0.2, 0.3)), lc=dict()),
    "no_cut_lod_off": dict(opts=dict(termination_transmittance=0.0, lod_enabled=False), lc=dict()),
    "chunk7_bias": dict(opts=dict(chunk_size=7, lod_bias=-1.5), lc=dict(depth_active=False)),
    "linear_head": dict(opts=dict(), lc=dict(lambda_dvar=0.0), color_space=1),
}


def _run(backend_name, case):
    import oracle as O_  # noqa: F811 (fresh import in a subprocess)
    c = CASES[case]
    orc = O_.Oracle()
    ref = O_.Reference()
    orc.mlp_mode = ref.mlp_mode_equivalent()
    cfg, params, bits, res = _setup(orc, color_space=c.get("color_space", 0))
    rays, tnf, av = _batch()
    opts = O_.render_options(**c["opts"])
    lc = O_.loss_config(inv_batch=1.0 / len(rays), **c["lc"])
    be = orc if backend_name == "oracle" else ref
    model = be.model(params, bits, res)
    g, loss, ev, co = be.train_backward(model, tnf, av, rays, opts, lc)
    return g, loss, ev, co


_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle'); sys.path.insert(0, {root!r} + '/tests')
import test_train_oracle as T
out = {{}}
for be in ('oracle', 'reference'):
    g, loss, ev, co = T._run(be, {case!r})
    for k, v in g.items(): out[be + '_' + k] = v
    out[be + '_loss'] = np.array([loss.total, loss.image, loss.depth, loss.dvar, loss.dist])
    out[be + '_ev'] = ev; out[be + '_co'] = co
np.savez({path!r}, **out)
"""


@pytest.mark.parametrize("case", sorted(CASES))
def test_train_backward_bit_exact_under_scalar_simd(case, tmp_path):
    path = str(tmp_path / "out.npz")
    env = dict(os.environ, LUMI_SIMD="scalar")
    subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, case=case, path=path)],
                   env=env, check=True, timeout=300)
    z = np.load(path)
    for k in ("grid", "density", "color", "alpha", "loss", "ev", "co"):
        assert np.array_equal(z["oracle_" + k], z["reference_" + k]), k
    assert z["oracle_ev"].sum() > 0 and np.abs(z["oracle_grid"]).max() > 0


def test_train_backward_matches_reference_default_isa():
    g, loss, ev, co = _run("oracle", "default")
    gr, lr_, er, cr = _run("reference", "default")
    assert np.array_equal(ev, er) and np.array_equal(co, cr)
    for k in ("total", "image", "depth", "dvar", "dist"):
        assert getattr(loss, k) == pytest.approx(getattr(lr_, k), rel=1e-12, abs=1e-15)
    for k in ("grid", "density", "color"):
        scale = np.abs(gr[k]).max()
        assert scale > 0
        assert np.abs(g[k] - gr[k]).max() <= 1e-5 * scale, k
    assert np.allclose(g["alpha"], gr["alpha"], rtol=1e-12, atol=1e-15)


def test_train_loss_terms_closed_form_empty_grid(oracle):
    """An empty occupancy grid marches no samples (test_renderer.cpp:201-217): the image loss
    is |v * background - gt| / 3 per channel and no field gradient flows."""
    cfg, params, bits, res = _setup(oracle)
    empty = np.zeros_like(bits)
    model = oracle.model(params, empty, res)
    rays, tnf, av = _batch(ncam=2, per=8)
    bg = (0.2, 0.4, 0.6)
    opts = O.render_options(background=bg)
    lc = O.loss_config(inv_batch=1.0 / len(rays))
    g, loss, ev, co = oracle.train_backward(model, tnf, av, rays, opts, lc)
    assert (ev == 0).all() and not g["grid"].any() and not g["density"].any()
    v = np.maximum(1.0 - av[rays["camera"]] * rays["vignette_r"], 1e-3)
    want = (np.abs(v[:, None] * np.array(bg) - rays["gt"].astype(np.float64)) / 3.0).sum() / len(rays)
    assert loss.image == pytest.approx(want, rel=1e-12)


def test_adam_step_matches_reference(oracle, reference):
    rng = np.random.default_rng(0)
    n = 1037
    p0 = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    m0 = rng.standard_normal(n).astype(np.float32) * 0.1
    v0 = np.abs(rng.standard_normal(n)).astype(np.float32) * 0.1
    args = (0.01, 0.9, 0.99, 1e-15, 1.0 / (1 - 0.9 ** 3), 1.0 / (1 - 0.99 ** 3))
    a = [p0.copy(), g, m0.copy(), v0.copy()]
    b = [p0.copy(), g, m0.copy(), v0.copy()]
    oracle.adam_step(*a, *args)
    reference.adam_step(*b, *args)
    for x, y in zip(a, b):
        assert np.allclose(x, y, rtol=2e-6, atol=1e-7)
