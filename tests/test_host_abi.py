"""CPU checks of the product boundary: the C-ABI library loads and exports every symbol
include/lumi_cuda.h declares; host-side model construction (layout, seeded synthetic
parameters) and argument validation match the reference -- no GPU compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2311_02542_b200 as L
from paper_2311_02542_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lumi_cuda.h")).read()
    return sorted(set(re.findall(r"\b(lumi_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_abi.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.SIGNATURES)  # the Python binding covers the whole ABI
    assert _abi.lib().lumi_abi_version() == 1


def test_layout_matches_reference_grid(oracle):
    for ts in (1 << 15, 1 << 19, 1 << 22):
        cfg = L.FieldConfig(grid=L.HashGridConfig(table_size=ts))
        f = L.RadianceField(cfg)
        lo = oracle.layout(O.field_config(table_size=ts))
        assert f.layout.total_floats == lo.total_floats
        for l in range(16):
            assert f.layout.resolution[l] == lo.resolution[l] == cfg.grid.resolution(l)
            assert f.layout.dense[l] == lo.dense[l]
            assert f.layout.offset[l] == lo.offset[l]
    # level 0 dense only at T=2^22; 65,061,249 entries -> 130M floats
    f = L.RadianceField(L.FieldConfig(grid=L.HashGridConfig(table_size=1 << 22)))
    assert f.level_is_dense(0) and not f.level_is_dense(1)
    assert f.layout.total_floats == 2 * 65061249
    assert f.layout.density_params == 3217 and f.layout.color_params == 6467


@pytest.mark.parametrize("seed,amp,ts", [(1234, 1.0, 1 << 19), (7, 0.0, 1 << 12), (99, 0.5, 1 << 15)])
def test_synthetic_params_bit_identical_to_reference_rng(oracle, seed, amp, ts):
    f = L.RadianceField.synthetic(L.FieldConfig(grid=L.HashGridConfig(table_size=ts)), seed, amp)
    p = oracle.synth_params(O.field_config(table_size=ts), seed, amp)
    assert np.array_equal(f.grid_params, p.table)
    assert np.array_equal(f.density_params, p.dparams)
    assert np.array_equal(f.color_params, p.cparams)
    g = L.RadianceField(L.FieldConfig(grid=L.HashGridConfig(table_size=ts)))
    if amp == 0.0:
        g.init_random(seed)
        assert np.array_equal(g.grid_params, p.table)


def test_unsupported_and_invalid_configs_fail_loudly():
    with pytest.raises(L.Error):
        L.RadianceField(L.FieldConfig(grid=L.HashGridConfig(table_size=1000)))
    with pytest.raises(L.Error):
        L.RadianceField(L.FieldConfig(hidden_width=32))
    with pytest.raises(L.Error):
        L.OccupancyGrid(0)


def test_occupancy_index_matches_oracle(oracle):
    g = L.OccupancyGrid(16)
    rng = np.random.default_rng(3)
    for p in rng.uniform(-2.2, 2.2, (300, 3)):
        assert g.voxel_index(p) == oracle.voxel_index(16, p)


def test_render_without_gpu_fails_loudly():
    """No CPU fallback: on a host without a B200 model creation raises a CUDA error."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    f = L.RadianceField(L.FieldConfig(grid=L.HashGridConfig(table_size=1 << 12)))
    with pytest.raises(L.Error) as ei:
        L.DeviceModel(f, L.OccupancyGrid(8))
    assert ei.value.code == _abi.LUMI_ERR_CUDA


def test_checkpoint_ingest_matches_reference_writer(reference, tmp_path):
    """§8f row 2: a LUMICKPT file written by the reference's save_checkpoint
    (scene.cpp:320-351) is read back by the product's native reader bit for bit."""
    cfg = O.field_config(table_size=1 << 12, base=16)
    p = reference.synth_params(cfg, 5, 0.8)
    rng = np.random.default_rng(2)
    occ = (rng.random(32 ** 3) < 0.3).astype(np.uint8)
    m = reference.model(p, occ, 32)
    path = tmp_path / "model.lumickpt"
    reference.save_checkpoint(m, path, spp=192, background=(0.1, 0.2, 0.3), contraction=1)
    field, grid, meta = L.load_checkpoint(path)
    assert np.array_equal(field.grid_params, p.table)
    assert np.array_equal(field.density_params, p.dparams)
    assert np.array_equal(field.color_params, p.cparams)
    assert grid.res == 32 and np.array_equal(grid.bits, occ)
    assert meta["samples_per_ray"] == 192 and meta["background"] == (0.1, 0.2, 0.3)
    assert meta["contraction"] == L.ContractionMode.kLInfCubic and meta["n_cameras"] == 2
    assert field.cfg.grid.table_size == 1 << 12 and field.cfg.grid.base_resolution == 16
    # corrupt / truncated files fail with the reference's messages
    raw = path.read_bytes()
    bad = tmp_path / "bad.lumickpt"
    bad.write_bytes(b"NOTACKPT" + raw[8:])
    with pytest.raises(L.Error, match="bad magic"):
        L.load_checkpoint(bad)
    bad.write_bytes(raw[: len(raw) - 100])
    with pytest.raises(L.Error, match="truncated"):
        L.load_checkpoint(bad)


def test_checkpoint_writer_byte_identical_to_reference(reference, tmp_path):
    """lumi_checkpoint_write (the product's save_checkpoint) produces the same bytes as the
    reference's save_checkpoint (scene.cpp:320-351) for a rendering model (zero trackers)."""
    cfg = O.field_config(table_size=1 << 12, base=16)
    p = reference.synth_params(cfg, 9, 0.7)
    rng = np.random.default_rng(4)
    occ = (rng.random(24 ** 3) < 0.4).astype(np.uint8)
    m = reference.model(p, occ, 24)
    ref_path = tmp_path / "ref.lumickpt"
    reference.save_checkpoint(m, ref_path, spp=128, background=(0.25, 0.5, 0.75), contraction=1)
    f = L.RadianceField(L.FieldConfig(grid=L.HashGridConfig(table_size=1 << 12, base_resolution=16)))
    f.grid_params[:] = p.table
    f.density_params[:] = p.dparams
    f.color_params[:] = p.cparams
    ours = tmp_path / "ours.lumickpt"
    L.save_checkpoint(ours, f, L.OccupancyGrid(24, occ), samples_per_ray=128,
                      background=(0.25, 0.5, 0.75), camera_alpha_v=(0.01, 0.02))
    assert ours.read_bytes() == ref_path.read_bytes()


def test_pfm_writer_byte_identical_to_reference(reference, tmp_path):
    """§8f row 3: the parity-artefact PFM writer (image.cpp:20-35) -- same bytes as the
    reference's write_pfm, and read_pfm (image.cpp:36-66) round-trips them."""
    from paper_2311_02542_b200.image_io import read_pfm, write_pfm
    rng = np.random.default_rng(6)
    for shape in ((3, 17, 23), (1, 8, 5)):
        img = rng.standard_normal(shape).astype(np.float32)
        ours, ref = tmp_path / "ours.pfm", tmp_path / "ref.pfm"
        write_pfm(ours, img)
        reference.write_pfm(ref, img)
        assert ours.read_bytes() == ref.read_bytes()
        assert np.array_equal(read_pfm(ours), img)
    with pytest.raises(L.Error, match="1 or 3 channels"):
        write_pfm(tmp_path / "x.pfm", np.zeros((2, 4, 4), np.float32))
