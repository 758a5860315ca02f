"""Pins the CPU oracle (oracle/lumi_oracle.c) before it is trusted as the parity checker:

1. the reference unit tests' known-answer values (proj/tests/test_*.cpp), restated;
2. the committed golden fixtures produced by the UNMODIFIED reference (tests/golden/);
3. differential runs against the reference library compiled from its own sources
   (oracle/_ref), when present.
"""
import math

import numpy as np
import pytest

import oracle as O
from conftest import ocam
from paper_2311_02542_b200 import scenes


# ---------------------------------------------------------------- known answers ----

def test_pq_known_answers(oracle):  # proj/tests/test_color.cpp:13-52
    c1, c2, c3 = 107.0 / 128.0, 2413.0 / 128.0, 2392.0 / 128.0
    assert c1 + c2 == 1.0 + c3
    assert oracle.pq_encode(100.0) == 1.0
    assert oracle.pq_encode(0.0) == pytest.approx(7.30955902578e-7, rel=1e-6)
    assert oracle.pq_encode(1.0) == pytest.approx(0.508078421517, rel=1e-9)
    assert oracle.pq_encode(2.5) == pytest.approx(0.602559154991, rel=1e-9)
    assert oracle.pq_decode(1.0) == pytest.approx(100.0, rel=1e-12)
    assert oracle.pq_decode(0.5081) == pytest.approx(1.0002150252, rel=1e-6)
    for s in range(-14, 7):
        y = math.ldexp(1.0, s)
        assert oracle.pq_decode(oracle.pq_encode(y)) == pytest.approx(y, rel=1e-6)
    prev = -1.0
    for i in range(0, 10001, 7):
        v = oracle.pq_encode(100.0 * i / 10000.0)
        assert v > prev
        prev = v


def test_lod_level_known_answers(oracle):  # proj/tests/test_grid.cpp:13-23
    cfg = O.field_config(table_size=1 << 15)
    assert oracle.lod_level(1.0 / 256.0, cfg) == pytest.approx(0.0, abs=1e-12)
    assert oracle.lod_level(1.0 / (256.0 * 1.4 * 1.4), cfg) == pytest.approx(2.0, rel=1e-9)
    assert oracle.lod_level(1.68437949364e-3, cfg) == pytest.approx(2.5, rel=1e-6)
    assert oracle.lod_level(1e-12, cfg) == 15.0


def test_lod_weights_case_structure(oracle):  # proj/tests/test_grid.cpp:25-51
    w = oracle.lod_weights(2.5, 0.0, 16)
    assert list(w[:3]) == [1.0, 1.0, 1.0] and w[3] == pytest.approx(0.5) and not w[4:].any()
    w = oracle.lod_weights(0.0, 0.0, 16)
    assert w[0] == 1.0 and not w[1:].any()
    assert (oracle.lod_weights(15.0, 0.0, 16) == 1.0).all()
    w = oracle.lod_weights(4.5, -2.0, 16)
    assert w[2] == 1.0 and w[3] == pytest.approx(0.5) and w[4] == 0.0
    w = oracle.lod_weights(1.0, -3.0, 16)
    assert w[0] == pytest.approx(1e-4) and not w[1:].any()


def test_lod_property_suite(oracle):  # proj/tests/test_grid.cpp:53-73
    cfg = O.field_config()
    rng = np.random.default_rng(21)
    for r in np.exp(rng.uniform(math.log(1e-5), math.log(0.2), 2000)):
        l = oracle.lod_level(float(r), cfg)
        w = oracle.lod_weights(l, 0.0, 16)
        assert (np.diff(w) <= 0).all() and (w >= 0).all() and (w <= 1).all()
        if 0 < l < 15 and l != math.floor(l):
            assert int((w > 0).sum()) == math.ceil(l) + 1


def test_contract_known_answers(oracle):  # proj/tests/test_camera.cpp:91-105
    assert list(oracle.contract([0.5, -0.3, 0.2])) == [0.5, -0.3, 0.2]
    assert oracle.contract([2, 0, 0]) == pytest.approx([1.5, 0, 0])
    assert oracle.contract([4, 2, 0]) == pytest.approx([1.75, 0.5, 0.0])
    with pytest.raises(ValueError):
        oracle.contract([float("nan"), 0, 0])
    rng = np.random.default_rng(12)  # bounded by [-2, 2] (test_camera.cpp:121-135)
    for p in rng.uniform(-6, 6, (500, 3)):
        assert np.abs(oracle.contract(p)).max() <= 2.0


def test_generate_ray_known_answers(oracle):  # proj/tests/test_camera.cpp:28-58
    cam = O.camera([1, 0, 0, 0, 1, 0, 0, 0, 1], [0, 0, 0], 100, 100, 32, 32, 64, 64, 0.1, 10)
    _, d = oracle.generate_ray(cam, 32, 32)
    assert d == pytest.approx([0, 0, 1])
    cam = O.camera([1, 0, 0, 0, 1, 0, 0, 0, 1], [0, 0, 0], 5.0, 7.0, 1.7, 2.3, 4, 4)
    _, d = oracle.generate_ray(cam, 3.5, 0.5)
    dx, dy = (3.5 - 1.7) / 5.0, (0.5 - 2.3) / 7.0
    inv = 1.0 / math.sqrt(dx * dx + dy * dy + 1.0)
    assert d == pytest.approx([dx * inv, dy * inv, inv], rel=1e-12)


def test_sample_distances(oracle):  # proj/tests/test_camera.cpp:224-238
    ts, _ = oracle.sample_distances(0.3, 7.0, 2)
    assert list(ts) == [0.3, 7.0]
    ts, _ = oracle.sample_distances(0.1, 10.0, 3)
    assert ts[1] == pytest.approx(1.0)
    ts, ratio = oracle.sample_distances(0.05, 20.0, 1024)
    assert np.allclose(ts[1:] / ts[:-1], ts[1] / ts[0], rtol=1e-9)
    assert (np.diff(ts) > 0).all()


def test_voxel_index_oracle(oracle):  # proj/tests/test_occupancy.cpp:224-235
    rng = np.random.default_rng(48)
    for p in rng.uniform(-2.2, 2.2, (500, 3)):
        i = oracle.voxel_index(16, p)
        u = (p + 2.0) * 0.25
        if (u < 0).any() or (u > 1).any():
            assert i == -1
        else:
            ix, iy, iz = np.minimum((u * 16).astype(int), 15)
            assert i == (iz * 16 + iy) * 16 + ix


def test_scheduler_known_answers(oracle):  # proj/tests/test_scheduler.cpp:13-61
    rows, shares = oracle.equal_assignment(400, 3)
    r, _ = oracle.assign_rows(400, [2e5, 1e5, 1e5], shares, rows, 1.0)
    assert list(r) == [200, 100, 100]
    r, _ = oracle.assign_rows(400, [2.0, 1.0, 1.0], [134 / 400, 133 / 400, 133 / 400],
                              [134, 133, 133], 0.5)
    assert list(r) == [167, 117, 116]
    for damp in (0.25, 0.5, 1.0):
        r, _ = oracle.assign_rows(200, [6.0, 2.0, 2.0], [0.6, 0.2, 0.2], [120, 40, 40], damp)
        assert list(r) == [120, 40, 40]
    with pytest.raises(ValueError):
        oracle.equal_assignment(3, 4)
    rows, shares = oracle.equal_assignment(4, 4)
    r, _ = oracle.assign_rows(4, [1e9, 1, 1, 1], shares, rows, 1.0)
    assert (r >= 1).all() and r.sum() == 4


def test_aggregate_stats_known_answers(oracle):  # proj/tests/test_scheduler.cpp:147-182
    ms = np.full(100, 10.0)
    mean, std, p99 = oracle.aggregate_stats(ms)
    assert mean == pytest.approx(100.0) and p99 == pytest.approx(100.0) and std == pytest.approx(0)
    ms[99] = 100.0
    mean, _, p99 = oracle.aggregate_stats(ms)
    assert p99 < mean and p99 < 100.0


# -------------------------------------------------------------- golden fixtures ----

def test_golden_occupancy_matches_survey_recipe(golden_meta):
    # S=1234, a=1.0, alpha=2.0 -> 155,144 / 2,097,152 occupied
    assert golden_meta["occ_small-T19"]["occupied"] == 155144


def test_oracle_reproduces_golden_c1(oracle, small_scene, golden_c1, golden_meta):
    """The restatement renders config C1 exactly like the reference did when the golden
    file was written (same host ISA sum order) -- and within 1e-5 on any other ISA."""
    cam = ocam(scenes.pinhole(256, 256))
    r = oracle.render_rows(small_scene["model"], cam, O.render_options(), 0, 256)
    exact = {"avx512": O.MLP_AVX512, "avx2": O.MLP_AVX2, "scalar": O.MLP_SCALAR}[
        golden_meta["reference_simd"]] == oracle.mlp_mode
    for k in ("out", "depth", "opacity"):
        if exact:
            assert np.array_equal(r[k], golden_c1[k]), k
        else:
            assert np.abs(r[k] - golden_c1[k]).max() < 1e-5, k
    if exact:
        for k in ("evals", "contributing", "kept"):
            assert np.array_equal(r[k], golden_c1[k].astype(np.int32)), k
        assert np.array_equal(r["row_evals"], golden_c1["row_evals"])


def test_oracle_kept_mask_matches_golden(oracle, small_scene, golden_c1):
    cam = ocam(scenes.pinhole(256, 256))
    b, e = (int(v) for v in golden_c1["kept_mask_rows"])
    mask, counts = oracle.march_kept(small_scene["model"], cam, O.render_options(), b, e)
    assert np.array_equal(mask[b:e, b:e], golden_c1["kept_mask"])
    assert np.array_equal(counts[b:e], golden_c1["kept_counts"])


# ------------------------------------------------------- differential vs reference ----

SMALL_CFG = dict(levels=6, fpl=2, base=4, scale=1.6, table_size=1 << 10)


def _rand_model(oracle, reference, seed, occ_p, res=16, levels=16, table_size=1 << 12):
    cfg = O.field_config(levels=levels, base=16, scale=1.4, table_size=table_size)
    po = oracle.synth_params(cfg, seed, 1.0)
    pr = reference.synth_params(cfg, seed, 1.0)
    assert np.array_equal(po.table, pr.table) and np.array_equal(po.dparams, pr.dparams)
    assert np.array_equal(po.cparams, pr.cparams)
    rng = np.random.default_rng(seed)
    occ = (rng.random(res ** 3) < occ_p).astype(np.uint8)
    return cfg, po, occ, oracle.model(po, occ, res), reference.model(pr, occ, res)


def test_synth_params_and_layout_match_reference(oracle, reference):
    for ts in (1 << 8, 1 << 15, 1 << 19):
        cfg = O.field_config(table_size=ts)
        lo, lr = oracle.layout(cfg), reference.layout(cfg)
        assert lo.total_floats == lr.total_floats
        assert [lo.dense[i] for i in range(16)] == [lr.dense[i] for i in range(16)]
        assert [lo.resolution[i] for i in range(16)] == [lr.resolution[i] for i in range(16)]
    cfg = O.field_config(table_size=1 << 15)
    for amp in (0.0, 0.5):
        po, pr = oracle.synth_params(cfg, 77, amp), reference.synth_params(cfg, 77, amp)
        assert np.array_equal(po.table, pr.table)
        assert np.array_equal(po.dparams, pr.dparams) and np.array_equal(po.cparams, pr.cparams)


def test_field_forward_matches_reference(oracle, reference):
    cfg, po, occ, mo, mr = _rand_model(oracle, reference, 5, 1.0)
    rng = np.random.default_rng(6)
    pos = rng.uniform(-2, 2, (333, 3))
    lodw = rng.uniform(0, 1, (333, 16)).astype(np.float32)
    lodw[rng.random((333, 16)) < 0.3] = 0
    sh = oracle.sh_encode(np.array([0.3, -0.5, 0.81]) / np.linalg.norm([0.3, -0.5, 0.81]))
    assert np.array_equal(sh, reference.sh_encode(np.array([0.3, -0.5, 0.81]) /
                                                  np.linalg.norm([0.3, -0.5, 0.81])))
    a = oracle.field_forward(mo, pos, lodw, sh)
    b = reference.field_forward(mr, pos, lodw, sh)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("variant", ["default", "lod_off", "bias", "nocut", "nocontract",
                                     "background", "chunk7", "spp64"])
def test_render_matches_reference(oracle, reference, variant):
    cfg, po, occ, mo, mr = _rand_model(oracle, reference, 11, 0.15)
    kw = {}
    if variant == "lod_off":
        kw["lod_enabled"] = False
    if variant == "bias":
        kw["lod_bias"] = -1.5
    if variant == "nocut":
        kw["termination_transmittance"] = 0.0
    if variant == "nocontract":
        kw["contraction"] = 0
    if variant == "background":
        kw["background"] = (0.1, 0.2, 0.3)
    if variant == "chunk7":
        kw["chunk_size"] = 7
    if variant == "spp64":
        kw["samples_per_ray"] = 64
    opts = O.render_options(**kw)
    cam = O.camera([0.8, 0.0, 0.6, 0.0, 1.0, 0.0, -0.6, 0.0, 0.8], [0.05, 0.1, -0.2], 30, 28,
                   20.3, 15.9, 40, 32, 0.05, 6.0)
    a = oracle.render_rows(mo, cam, opts, 3, 29)
    b = reference.render_rows(mr, cam, opts, 3, 29)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    ka, ca = oracle.march_kept(mo, cam, opts, 3, 29)
    kb, cb = reference.march_kept(mr, cam, opts, 3, 29)
    assert np.array_equal(ka, kb) and np.array_equal(ca, cb)


def test_probe_prune_matches_reference(oracle, reference):
    cfg, po, occ, mo, mr = _rand_model(oracle, reference, 21, 1.0, res=12)
    cams = [O.camera([1, 0, 0, 0, 0, -1, 0, 1, 0], [0.1, -0.3, 0.05], 10, 10, 8, 8, 16, 16),
            O.camera([1, 0, 0, 0, 1, 0, 0, 0, 1], [0.5, 0.5, 0.5], 10, 10, 8, 8, 16, 16, 0.1, 4)]
    pm_o = oracle.probe(mo, cams, 64, 2, 12)
    pm_r, occ_r = reference.probe_prune(mr, cams, 64, 2, 12, 2.0)
    assert np.array_equal(pm_o, pm_r)
    assert np.array_equal(oracle.prune(pm_o, 2.0), occ_r)


def test_scheduler_matches_reference(oracle, reference):
    rng = np.random.default_rng(81)
    for _ in range(50):
        workers = int(rng.integers(2, 8))
        height = workers + int(rng.integers(0, 500))
        ro, so = oracle.equal_assignment(height, workers)
        rr, sr = reference.equal_assignment(height, workers)
        assert np.array_equal(ro, rr) and np.array_equal(so, sr)
        for _ in range(10):
            tp = rng.uniform(0.1, 10.0, workers)
            damp = float(rng.uniform(0.1, 1.0))
            ro2, so2 = oracle.assign_rows(height, tp, so, ro, damp)
            rr2, sr2 = reference.assign_rows(height, tp, sr, rr, damp)
            assert np.array_equal(ro2, rr2) and np.array_equal(so2, sr2)
            ro, so, rr, sr = ro2, so2, rr2, sr2
    for _ in range(100):
        ms = rng.uniform(5, 50, int(rng.integers(20, 120)))
        assert np.array_equal(oracle.aggregate_stats(ms), reference.aggregate_stats(ms))
