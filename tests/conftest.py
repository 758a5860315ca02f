"""Shared fixtures.  `-m "not gpu"` runs on any CPU host; `-m gpu` needs a B200."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    o = O.Oracle()
    if O.reference_available():
        o.mlp_mode = O.Reference().mlp_mode_equivalent()  # replay the host ISA's sum order
    return o


@pytest.fixture(scope="session")
def reference():
    import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref/liblumi_ref.so not built (make -C oracle ref)")
    return O.Reference()


def load_occ(name):
    z = np.load(os.path.join(GOLDEN, f"occ_{name}.npz"))
    res = int(z["res"])
    bits = np.unpackbits(z["bits"])[: res ** 3].astype(np.uint8)
    return bits, res, z


@pytest.fixture(scope="session")
def golden_meta():
    return json.load(open(os.path.join(GOLDEN, "meta.json")))


@pytest.fixture(scope="session")
def golden_c1():
    return dict(np.load(os.path.join(GOLDEN, "render_c1.npz")))


@pytest.fixture(scope="session")
def small_scene(oracle):
    """C1/C2 model: T=2^19 synthetic bake, reference-baked occupancy (tests/golden)."""
    import oracle as O
    from paper_2311_02542_b200 import scenes
    s = scenes.SMALL
    cfg = O.field_config(s.levels, s.features_per_level, s.base_resolution, s.per_level_scale,
                         s.table_size, s.hidden_width, s.bottleneck, 0)
    params = oracle.synth_params(cfg, s.seed, s.amplitude)
    bits, res, _ = load_occ(s.name)
    return dict(spec=s, cfg=cfg, params=params, occ=bits, res=res,
                model=oracle.model(params, bits, res))


def ocam(spec):
    import oracle as O
    return O.camera(spec.rot, spec.origin, spec.fx, spec.fy, spec.cx, spec.cy, spec.width,
                    spec.height, spec.t_near, spec.t_far)
