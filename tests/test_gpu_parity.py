"""GPU parity: the sm_100a path (through the C ABI) against the oracle / golden fixtures.

Bars (BASELINE.json north_star): occupancy-kept sample indices and per-ray sample counts
bit-exact; pixels within 1e-3 max abs in PQ space and PSNR >= 60 dB against the reference.
"""
import numpy as np
import pytest

import oracle as O
from conftest import load_occ, ocam
from paper_2311_02542_b200 import scenes
from paper_2311_02542_b200.metrics import psnr

pytestmark = pytest.mark.gpu

PIX_TOL = 1e-3  # max abs, PQ space (north_star)
PSNR_MIN = 60.0


def dump_pfm(name, **images):
    """Parity artefacts: write the GPU / oracle images of a failing case as PFM
    (image.cpp:20-35) under gpurun_out/parity/ (merged back from the GPU box)."""
    import os
    from paper_2311_02542_b200.image_io import write_pfm
    root = os.environ.get("GRAFT_REPO_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = os.path.join(root, "gpurun_out", "parity")
    os.makedirs(d, exist_ok=True)
    for k, img in images.items():
        write_pfm(os.path.join(d, f"{name}_{k}.pfm"), img)
    return d


def check_pixels(name, got, want, tol=PIX_TOL, psnr_min=PSNR_MIN):
    """max |dPQ| <= tol and PSNR >= psnr_min; dumps both images as PFM when either fails."""
    err = float(np.abs(got - want).max())
    p = psnr(got, want)
    if not (err <= tol and p >= psnr_min):
        d = dump_pfm(name, gpu=got, oracle=want, absdiff=np.abs(got - want))
        pytest.fail(f"{name}: max|dPQ|={err:.3e} PSNR={p:.1f} dB (images in {d})")
    return err, p


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch


@pytest.fixture(scope="module")
def lumi():
    import paper_2311_02542_b200 as L
    return L


def product_model(lumi, spec, occ_bits, res):
    cfg = lumi.FieldConfig(grid=lumi.HashGridConfig(spec.levels, spec.features_per_level,
                                                    spec.base_resolution, spec.per_level_scale,
                                                    spec.table_size))
    field = lumi.RadianceField.synthetic(cfg, spec.seed, spec.amplitude)
    grid = lumi.OccupancyGrid(res, occ_bits)
    return field, grid, lumi.DeviceModel(field, grid, 0)


@pytest.fixture(scope="module")
def small(lumi, torch_cuda, small_scene):
    s = small_scene
    field, grid, dm = product_model(lumi, s["spec"], s["occ"], s["res"])
    return dict(field=field, grid=grid, dm=dm, **s)


def march_kept_gpu(torch, lumi, dm, cam, opts, b, e):
    words = (opts.samples_per_ray + 31) // 32
    mask = torch.zeros((cam.height, cam.width, words), dtype=torch.int32, device="cuda")
    counts = torch.zeros((cam.height, cam.width), dtype=torch.int32, device="cuda")
    dm.march_kept_async(cam, opts, b, e, mask.data_ptr(), counts.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return mask.cpu().numpy().view(np.uint32), counts.cpu().numpy()


def test_device_is_b200(lumi, torch_cuda):
    info = lumi.device_info(0)
    assert "sm_100" in info or "sm_10" in info, info


def test_march_kept_bitexact_c1(lumi, torch_cuda, small, golden_c1, oracle):
    cam_spec = scenes.pinhole(256, 256)
    cam = lumi.CameraModel.from_spec(cam_spec)
    opts = lumi.RenderOptions()
    mask, counts = march_kept_gpu(torch_cuda, lumi, small["dm"], cam, opts, 0, 256)
    om, oc = oracle.march_kept(small["model"], ocam(cam_spec), O.render_options(), 0, 256)
    assert np.array_equal(mask, om)
    assert np.array_equal(counts, oc)
    b, e = (int(v) for v in golden_c1["kept_mask_rows"])
    assert np.array_equal(mask[b:e, b:e], golden_c1["kept_mask"])  # the reference itself


@pytest.mark.parametrize("variant", ["nocontract", "spp1024", "rotated"])
def test_march_kept_bitexact_variants(lumi, torch_cuda, small, oracle, variant):
    spec = scenes.pinhole(96, 80)
    spp, contraction = 256, 1
    if variant == "nocontract":
        contraction = 0
    if variant == "spp1024":
        spp = 1024
    if variant == "rotated":
        rot, org = scenes.head_pose(17)
        spec = scenes.pinhole(96, 80, rot, org)
    cam = lumi.CameraModel.from_spec(spec)
    opts = lumi.RenderOptions(samples_per_ray=spp, contraction=contraction)
    mask, counts = march_kept_gpu(torch_cuda, lumi, small["dm"], cam, opts, 0, 80)
    om, oc = oracle.march_kept(small["model"], ocam(spec),
                               O.render_options(samples_per_ray=spp, contraction=contraction), 0, 80)
    assert np.array_equal(mask, om) and np.array_equal(counts, oc)


def test_march_kept_bitexact_c2_full_size(lumi, torch_cuda, small, oracle):
    """Config C2 (one 2048^2 eyebuffer): GPU over the full frame, oracle on every 16th row."""
    spec = scenes.pinhole(2048, 2048)
    cam = lumi.CameraModel.from_spec(spec)
    opts = lumi.RenderOptions()
    mask, counts = march_kept_gpu(torch_cuda, lumi, small["dm"], cam, opts, 0, 2048)
    oopts = O.render_options()
    for y in range(0, 2048, 16):
        om, oc = oracle.march_kept(small["model"], ocam(spec), oopts, y, y + 1)
        assert np.array_equal(mask[y], om[y]), y
        assert np.array_equal(counts[y], oc[y]), y
    assert counts.sum() > 0


@pytest.mark.parametrize("frame,contraction", [(0, 1), (37, 1), (90, 1), (11, 0)])
def test_filtered_march_equals_exact_full_eye(lumi, torch_cuda, small, frame, contraction):
    """The production march pass (fp32 with a certified error bound, exact double fallback)
    against the exact double march, bit for bit, over full 2048^2 eyebuffers of the
    head-motion path."""
    rot, org = scenes.head_pose(frame)
    cam = lumi.CameraModel.from_spec(scenes.eye_cameras(2048, rot, org)[frame % 2])
    opts = lumi.RenderOptions(contraction=contraction)
    dm = small["dm"]
    dm.set_kernel("simt")
    try:
        em, ec = march_kept_gpu(torch_cuda, lumi, dm, cam, opts, 0, 2048)
    finally:
        dm.set_kernel("ws")
    fm, fc = march_kept_gpu(torch_cuda, lumi, dm, cam, opts, 0, 2048)
    assert ec.sum() > 0
    assert np.array_equal(fc, ec)
    assert np.array_equal(fm, em)


def _look_rot(fwd, up=(0.0, 0.0, 1.0)):
    """Row-major world<-camera rotation whose camera z looks along `fwd`."""
    f = np.asarray(fwd, float)
    f /= np.linalg.norm(f)
    x = np.cross(up, f)
    if np.linalg.norm(x) < 1e-6:
        x = np.cross((0.0, 1.0, 0.0), f)
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    return tuple(np.stack([x, y, f], axis=1).reshape(-1).tolist())


@pytest.mark.parametrize("pose", ["diagonal", "corner", "outside", "outside_far", "axis_tie", "nocontract_out"])
def test_segment_march_equals_exact_off_axis(lumi, torch_cuda, small, pose):
    """The segment march pass (inside-cube and final-pyramid segments, general test elsewhere)
    against the exact double march on poses that stress its segment logic: diagonal views
    (max-axis ties between |d| components), a camera near a cube corner, cameras outside the
    cube looking in (no inside segment, late final pyramids), no contraction from outside."""
    fwd, org, contraction = {
        "diagonal": ((1.0, 1.0, 1.0), (0.1, -0.2, 0.05), 1),
        "corner": ((-1.0, -0.8, -0.6), (0.93, 0.9, 0.95), 1),
        "outside": ((-1.0, 0.3, 0.1), (1.7, -0.2, 0.3), 1),
        "outside_far": ((-1.0, -1.0, 0.2), (3.5, 2.5, -0.4), 1),
        "axis_tie": ((1.0, 1.0, 0.0), (0.0, 0.0, 0.0), 1),
        "nocontract_out": ((0.0, -1.0, 0.2), (0.3, 1.6, -0.1), 0),
    }[pose]
    spec = scenes.pinhole(512, 512, _look_rot(fwd), org)
    cam = lumi.CameraModel.from_spec(spec)
    opts = lumi.RenderOptions(contraction=contraction)
    dm = small["dm"]
    dm.set_kernel("simt")
    try:
        em, ec = march_kept_gpu(torch_cuda, lumi, dm, cam, opts, 0, 512)
    finally:
        dm.set_kernel("ws")
    fm, fc = march_kept_gpu(torch_cuda, lumi, dm, cam, opts, 0, 512)
    assert ec.sum() > 0
    assert np.array_equal(fc, ec)
    assert np.array_equal(fm, em)


def _render(lumi, dm, cam, opts, b=0, e=None):
    e = cam.height if e is None else e
    out = np.zeros((3, cam.height, cam.width), np.float32)
    depth = np.zeros((cam.height, cam.width), np.float32)
    opac = np.zeros((cam.height, cam.width), np.float32)
    stats = []
    dm.render_rows(cam, opts, b, e, out, depth, opac, stats)
    return out, depth, opac, stats


def test_render_c1_vs_reference_golden(lumi, torch_cuda, small, golden_c1):
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 256))
    out, depth, opac, stats = _render(lumi, small["dm"], cam, lumi.RenderOptions())
    err = np.abs(out - golden_c1["out"]).max()
    p = psnr(out, golden_c1["out"])
    print(f"C1 max|dPQ|={err:.3e} PSNR={p:.1f} dB")
    assert err <= PIX_TOL and p >= PSNR_MIN
    assert np.abs(opac - golden_c1["opacity"]).max() <= PIX_TOL
    # per-row evals (RowStats.evals): match except where sigma rounding moves the cut
    row_ev = np.array([s.evals for s in stats])
    rel = np.abs(row_ev - golden_c1["row_evals"]) / np.maximum(golden_c1["row_evals"], 1)
    assert rel.max() < 0.02
    assert [s.row for s in stats] == list(range(256)) and all(s.rays == 256 for s in stats)


def test_render_counts_vs_reference(lumi, torch_cuda, small, golden_c1):
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 256))
    counts = torch_cuda.zeros((256, 256, 2), dtype=torch_cuda.int32, device="cuda")
    rgb = torch_cuda.zeros((3, 256, 256), dtype=torch_cuda.float32, device="cuda")
    t = lumi.renderer._abi.FrameTarget()
    t.rgb, t.counts, t.width, t.height = rgb.data_ptr(), counts.data_ptr(), 256, 256
    small["dm"].render_rows_async(cam, lumi.RenderOptions(), 0, 256, t,
                                  torch_cuda.cuda.current_stream().cuda_stream)
    torch_cuda.cuda.synchronize()
    c = counts.cpu().numpy()
    ev_match = np.mean(c[..., 0] == golden_c1["evals"])
    co_match = np.mean(c[..., 1] == golden_c1["contributing"])
    print(f"evals match {ev_match:.5f} contributing match {co_match:.5f}")
    # termination-index mismatches could only come from sigma rounding at the 1e-4 cut; at C1
    # there are none (measured 1.00000 on every run)
    assert ev_match == 1.0 and co_match == 1.0


@pytest.mark.parametrize("kernel", ["ws", "simt"])
def test_both_kernels_vs_reference_golden(lumi, torch_cuda, small, golden_c1, kernel):
    """The production tcgen05 kernel and the fp32 CUDA-core cross-check kernel."""
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 256))
    small["dm"].set_kernel(kernel)
    try:
        out, _, opac, stats = _render(lumi, small["dm"], cam, lumi.RenderOptions())
    finally:
        small["dm"].set_kernel("ws")
    err = np.abs(out - golden_c1["out"]).max()
    print(f"{kernel}: C1 max|dPQ|={err:.3e} PSNR={psnr(out, golden_c1['out']):.1f} dB")
    assert err <= (1e-6 if kernel == "simt" else PIX_TOL)
    assert psnr(out, golden_c1["out"]) >= PSNR_MIN


def test_split_render_bit_identical(lumi, torch_cuda, small):
    """render_rows determinism contract (proj/tests/test_renderer.cpp:243-266)."""
    cam = lumi.CameraModel.from_spec(scenes.pinhole(128, 96))
    opts = lumi.RenderOptions()
    full, _, _, _ = _render(lumi, small["dm"], cam, opts)
    split = np.zeros_like(full)
    small["dm"].render_rows(cam, opts, 0, 37, split)
    small["dm"].render_rows(cam, opts, 37, 96, split)
    assert np.array_equal(full, split)
    with pytest.raises(lumi.Error):
        small["dm"].render_rows(cam, opts, 5, 97, split)


@pytest.mark.parametrize("variant", ["lod_off", "bias", "nocut", "background", "spp64",
                                     "chunk7", "rotated", "odd_sizes", "nocontract", "bias_up"])
def test_render_options_vs_oracle(lumi, torch_cuda, small, oracle, variant):
    kw, okw = {}, {}
    spec = scenes.pinhole(64, 48)
    if variant == "nocontract":
        kw["contraction"] = okw["contraction"] = 0
    if variant == "bias_up":
        kw["lod_bias"] = okw["lod_bias"] = 1.75
    if variant == "odd_sizes":  # partial packets on both axes, spp not a multiple of 32
        spec = scenes.pinhole(37, 48)
        kw["samples_per_ray"] = okw["samples_per_ray"] = 77
    if variant == "lod_off":
        kw["lod_enabled"] = okw["lod_enabled"] = False
    if variant == "bias":
        kw["lod_bias"] = okw["lod_bias"] = -2.5
    if variant == "nocut":
        kw["termination_transmittance"] = okw["termination_transmittance"] = 0.0
    if variant == "background":
        kw["background"] = okw["background"] = (0.2, 0.1, 0.05)
    if variant == "spp64":
        kw["samples_per_ray"] = okw["samples_per_ray"] = 64
    if variant == "chunk7":
        kw["chunk_size"] = okw["chunk_size"] = 7
    if variant == "rotated":
        spec = scenes.pinhole(64, 48, *scenes.head_pose(40))
    cam = lumi.CameraModel.from_spec(spec)
    out, depth, opac, stats = _render(lumi, small["dm"], cam, lumi.RenderOptions(**kw))
    ref = oracle.render_rows(small["model"], ocam(spec), O.render_options(**okw), 0, 48)
    assert np.abs(out - ref["out"]).max() <= PIX_TOL
    assert psnr(out, ref["out"]) >= PSNR_MIN
    assert np.abs(opac - ref["opacity"]).max() <= PIX_TOL
    row_ev = np.array([s.evals for s in stats])
    assert np.abs(row_ev - ref["row_evals"]).max() <= max(8, 0.02 * ref["row_evals"].max())


def test_render_c2_sampled_rows_vs_oracle(lumi, torch_cuda, small, oracle):
    """Config C2 at full size: GPU frame, oracle on a band of rows through the centre."""
    spec = scenes.pinhole(2048, 2048)
    cam = lumi.CameraModel.from_spec(spec)
    out, _, opac, _ = _render(lumi, small["dm"], cam, lumi.RenderOptions())
    ref = oracle.render_rows(small["model"], ocam(spec), O.render_options(), 1000, 1016)
    band = slice(1000, 1016)
    err = np.abs(out[:, band] - ref["out"][:, band]).max()
    print(f"C2 band max|dPQ|={err:.3e}")
    assert err <= PIX_TOL
    assert psnr(out[:, band], ref["out"][:, band]) >= PSNR_MIN
    assert np.isfinite(out).all() and (opac >= 0).all() and (opac <= 1 + 1e-6).all()


def test_gpu_bake_vs_reference_bake(lumi, torch_cuda, small):
    """OccupancyGrid::probe(k=2) + prune(2.0) on the GPU against the reference bake: bits may
    differ only where the probe value sits within 1% of alpha (MLP summation order)."""
    spec = scenes.SMALL
    probe_cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 256))
    grid, pm = small["dm"].bake_occupancy([probe_cam], scenes.SAMPLES_PER_RAY,
                                          scenes.PROBE_POINTS_PER_AXIS, spec.occ_res,
                                          spec.prune_alpha, want_probe=True)
    bits, res, z = load_occ(spec.name)
    diff = np.nonzero(grid.bits != bits)[0]
    assert np.isin(diff, z["near_threshold"]).all()
    assert diff.size < 100
    samp = z["probe_sample"]
    got = pm[z["probe_sample_idx"]]
    assert np.allclose(got, samp, rtol=1e-3, atol=1e-3)


def test_display_epilogue_srgb8(lumi, torch_cuda, small, oracle):
    """§8f row 3: the fused PQ -> scene-linear -> 2^bias -> sRGB8 eyebuffer store matches
    pq_to_srgb_float (trainer.cpp:175-182) + tonemap_srgb rounding (color.cpp:104-115)
    applied to the kernel's own PQ output, within one code value."""
    W = H = 64
    cam = lumi.CameraModel.from_spec(scenes.pinhole(W, H))
    rgb = torch_cuda.zeros((3, H, W), dtype=torch_cuda.float32, device="cuda")
    srgb = torch_cuda.zeros((H, W, 3), dtype=torch_cuda.uint8, device="cuda")
    for bias in (0.0, 1.5):
        t = lumi.renderer._abi.FrameTarget()
        t.rgb, t.srgb8, t.width, t.height = rgb.data_ptr(), srgb.data_ptr(), W, H
        t.exposure_bias_stops = bias
        small["dm"].render_rows_async(cam, lumi.RenderOptions(), 0, H, t,
                                      torch_cuda.cuda.current_stream().cuda_stream)
        torch_cuda.cuda.synchronize()
        pq = rgb.cpu().numpy()
        want = np.zeros((H, W, 3), np.int32)
        for c in range(3):
            for y in range(H):
                for x in range(W):
                    lin = oracle.pq_decode(min(max(float(pq[c, y, x]), 0.0), 1.0))
                    want[y, x, c] = int(round(oracle.srgb_oetf(min(lin * 2 ** bias, 1.0)) * 255))
        got = srgb.cpu().numpy().astype(np.int32)
        assert np.abs(got - want).max() <= 1, bias


def test_linear_color_head_vs_oracle(lumi, torch_cuda, small_scene, oracle):
    """field.h:135-136: the kLinear ablation head (trunc_exp instead of sigmoid)."""
    import oracle as O
    s = small_scene["spec"]
    cfg = lumi.FieldConfig(grid=lumi.HashGridConfig(table_size=s.table_size),
                           color_space=lumi.ColorSpaceMode.kLinear)
    field = lumi.RadianceField.synthetic(cfg, s.seed, s.amplitude)
    dm = lumi.DeviceModel(field, lumi.OccupancyGrid(small_scene["res"], small_scene["occ"]), 0)
    spec = scenes.pinhole(48, 40)
    cam = lumi.CameraModel.from_spec(spec)
    out = np.zeros((3, 40, 48), np.float32)
    dm.render_rows(cam, lumi.RenderOptions(), 0, 40, out)
    ocfg = O.field_config(table_size=s.table_size, color_space=1)
    om = oracle.model(oracle.synth_params(ocfg, s.seed, s.amplitude), small_scene["occ"],
                      small_scene["res"])
    ref = oracle.render_rows(om, ocam(spec), O.render_options(), 0, 40)
    scale = max(1.0, float(np.abs(ref["out"]).max()))
    assert np.abs(out - ref["out"]).max() <= 1e-3 * scale


def test_stress_dense_occupancy_4k_rows(lumi, torch_cuda, small, oracle):
    """C5 flavour: all-occupied grid (no skipping, little early termination) on a band of a
    4096^2 eye against the oracle."""
    grid = lumi.OccupancyGrid(128)
    dm = lumi.DeviceModel(small["field"], grid, 0)
    spec = scenes.pinhole(4096, 4096)
    cam = lumi.CameraModel.from_spec(spec)
    out = np.zeros((3, 4096, 4096), np.float32)
    stats = []
    dm.render_rows(cam, lumi.RenderOptions(), 2040, 2048, out, None, None, stats)
    ones = np.ones(128 ** 3, np.uint8)
    import oracle as O
    om = oracle.model(small["params"], ones, 128)
    ref = oracle.render_rows(om, ocam(spec), O.render_options(), 2040, 2048)
    band = slice(2040, 2048)
    assert np.abs(out[:, band] - ref["out"][:, band]).max() <= PIX_TOL
    assert sum(s.evals for s in stats) == pytest.approx(int(ref["row_evals"].sum()), rel=0.01)


def test_concurrent_workers_and_optional_planes(lumi, torch_cuda, small):
    """run_frame's contract (scheduler.cpp:124-142): concurrent render_rows calls on disjoint
    bands of one image from worker threads (pooled staging slots, one stream each) give the
    single-call image bit for bit; requesting depth/opacity planes does not change rgb."""
    import threading
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 192))
    opts = lumi.RenderOptions()
    dm = small["dm"]
    full = np.zeros((3, 192, 256), np.float32)
    depth = np.zeros((192, 256), np.float32)
    opac = np.zeros((192, 256), np.float32)
    dm.render_rows(cam, opts, 0, 192, full, depth, opac)
    assert depth.any() and opac.any()
    rgb_only = np.zeros_like(full)
    dm.render_rows(cam, opts, 0, 192, rgb_only)
    assert np.array_equal(full, rgb_only)
    for rep in range(3):
        par = np.zeros_like(full)
        bands = [(0, 61), (61, 130), (130, 192)]
        errs = []

        def work(b, e):
            try:
                dm.render_rows(cam, opts, b, e, par)
            except Exception as ex:  # noqa: BLE001
                errs.append(ex)

        ts = [threading.Thread(target=work, args=be) for be in bands]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs
        assert np.array_equal(par, full), f"rep {rep}"


def test_zero_copy_pinned_output_equals_staged(lumi, torch_cuda, small):
    """lumi_render_rows writes page-locked planes directly from the kernel (zero-copy) and
    pageable planes through a device staging copy: same pixels, depth, opacity and stats,
    rows outside [b, e) untouched."""
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 128))
    opts = lumi.RenderOptions()
    dm = small["dm"]
    pg = [np.full((3, 128, 256), -1, np.float32), np.full((128, 256), -1, np.float32),
          np.full((128, 256), -1, np.float32)]
    pn = [torch_cuda.full(a.shape, -1.0).pin_memory().numpy() for a in pg]
    st_pg, st_pn = [], []
    dm.render_rows(cam, opts, 20, 100, pg[0], pg[1], pg[2], st_pg)
    dm.render_rows(cam, opts, 20, 100, pn[0], pn[1], pn[2], st_pn)
    for a, b_ in zip(pg, pn):
        assert np.array_equal(a, b_)
    assert (pn[0][:, :20] == -1).all() and (pn[0][:, 100:] == -1).all()
    assert [s.evals for s in st_pg] == [s.evals for s in st_pn]


@pytest.mark.parametrize("band", [(5, 19), (0, 1), (47, 48), (13, 13)])
def test_odd_row_bands_every_kernel(lumi, torch_cuda, small, oracle, band):
    """Row bands that start and end inside a 4-row packet (and empty / one-row bands) on a
    37-pixel-wide image, every tcgen05 kernel against the oracle; rows outside the band are
    untouched (renderer.h:252-278)."""
    spec = scenes.pinhole(37, 48)
    cam = lumi.CameraModel.from_spec(spec)
    b, e = band
    ref = oracle.render_rows(small["model"], ocam(spec), O.render_options(), 0, 48)
    dm = small["dm"]
    for kernel in ("ws", "simt"):
        dm.set_kernel(kernel)
        try:
            out = np.full((3, 48, 37), -1, np.float32)
            dm.render_rows(cam, lumi.RenderOptions(), b, e, out)
        finally:
            dm.set_kernel("ws")
        assert (out[:, :b] == -1).all() and (out[:, e:] == -1).all(), kernel
        if e > b:
            assert np.abs(out[:, b:e] - ref["out"][:, b:e]).max() <= PIX_TOL, kernel


def test_mlp_batch_vs_oracle(lumi, torch_cuda, small, oracle):
    """The tcgen05 MLP stage alone (lumi_mlp_batch_async) on oracle-encoded features of random
    points: sigma and colour against RadianceField::forward_chunk (field.h:106-137) with fp16
    operands (colour within 2e-3, sigma within 1 % -- sigma = exp(raw) magnifies the fp16
    rounding of the 64-wide dot products)."""
    torch = torch_cuda
    rng = np.random.default_rng(8)
    n = 4096
    pos = rng.uniform(-1.8, 1.8, (n, 3))
    lodw = np.ones((n, 16), np.float32)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    sh = oracle.sh_encode(d)
    sigma, color, feat = oracle.field_forward(small["model"], pos, lodw, sh)
    f16 = torch.from_numpy(np.ascontiguousarray(feat.T)).half().cuda()
    dirs = torch.from_numpy(np.tile(d, (n, 1)).astype(np.float32)).cuda()
    out = torch.zeros((n, 4), dtype=torch.float32, device="cuda")
    small["dm"].mlp_batch_async(f16.data_ptr(), dirs.data_ptr(), n, out.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert np.abs(o[:, 1:] - color.T).max() <= 2e-3
    assert np.abs(o[:, 0] / sigma - 1).max() <= 1e-2


@pytest.mark.parametrize("kernel", ["ws", "simt"])
def test_empty_grid_renders_background(lumi, torch_cuda, small, kernel):
    """An empty occupancy grid marches no samples (proj/tests/test_renderer.cpp:201-217): every
    pixel is the background, depth and opacity 0, zero evaluations."""
    grid = lumi.OccupancyGrid(128, np.zeros(128 ** 3, np.uint8))
    dm = lumi.DeviceModel(small["field"], grid, 0)
    dm.set_kernel(kernel)
    cam = lumi.CameraModel.from_spec(scenes.pinhole(64, 40))
    bg = (0.25, 0.5, 0.125)
    out = np.full((3, 40, 64), -1, np.float32)
    depth = np.full((40, 64), -1, np.float32)
    opac = np.full((40, 64), -1, np.float32)
    stats = []
    dm.render_rows(cam, lumi.RenderOptions(background=bg), 0, 40, out, depth, opac, stats)
    for c in range(3):
        assert (out[c] == np.float32(bg[c])).all()
    assert not depth.any() and not opac.any()
    assert sum(s.evals for s in stats) == 0


def test_render_c3_full_model_vs_oracle(lumi, torch_cuda, oracle):
    """Config C3's model (T=2^22: level 0 dense, levels 1-15 hashed, reference-baked occupancy)
    on a 2048^2 eye of the head path: the production kernel renders the whole eye, the oracle
    a band of rows through the centre and every 256th row."""
    s = scenes.FULL
    cfg = O.field_config(s.levels, s.features_per_level, s.base_resolution, s.per_level_scale,
                         s.table_size, s.hidden_width, s.bottleneck, 0)
    params = oracle.synth_params(cfg, s.seed, s.amplitude)
    bits, res, _ = load_occ(s.name)
    om = oracle.model(params, bits, res)
    _, _, dm = product_model(lumi, s, bits, res)
    rot, org = scenes.head_pose(23)
    spec = scenes.eye_cameras(2048, rot, org)[1]
    cam = lumi.CameraModel.from_spec(spec)
    out, _, opac, stats = _render(lumi, dm, cam, lumi.RenderOptions())
    rows = list(range(1016, 1024)) + list(range(0, 2048, 256))
    errs = []
    for y in rows:
        ref = oracle.render_rows(om, ocam(spec), O.render_options(), y, y + 1)
        errs.append(np.abs(out[:, y] - ref["out"][:, y]).max())
        assert np.abs(opac[y] - ref["opacity"][y]).max() <= PIX_TOL, y
    print(f"C3 sampled rows max|dPQ|={max(errs):.3e}")
    assert max(errs) <= PIX_TOL
    assert sum(st.evals for st in stats) > 0


def test_exact_march_pass_feeds_the_renderer(tmp_path):
    """LUMI_MARCH_EXACT=1 swaps the production march pass for the double-precision one (A/B and
    debugging); it must feed the packet renderer the same kept masks and ray directions, so the
    C1 frame matches the reference golden to the same bar.  The switch is read once per
    process, hence the subprocess."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from conftest import GOLDEN, load_occ
import paper_2311_02542_b200 as L
from paper_2311_02542_b200 import scenes
s = scenes.SMALL
cfg = L.FieldConfig(grid=L.HashGridConfig(s.levels, s.features_per_level, s.base_resolution,
                                          s.per_level_scale, s.table_size))
bits, res, _ = load_occ(s.name)
dm = L.DeviceModel(L.RadianceField.synthetic(cfg, s.seed, s.amplitude), L.OccupancyGrid(res, bits), 0)
cam = L.CameraModel.from_spec(scenes.pinhole(256, 256))
out = np.zeros((3, 256, 256), np.float32)
dm.render_rows(cam, L.RenderOptions(), 0, 256, out)
ref = np.load(GOLDEN + "/render_c1.npz")["out"]
print(float(np.abs(out - ref).max()))
'''
    import os
    env = dict(os.environ, LUMI_MARCH_EXACT="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    err = float(r.stdout.strip().splitlines()[-1])
    print(f"exact march C1 max|dPQ|={err:.3e}")
    assert err <= PIX_TOL


# ---- round 2: whole frames at the headline config, the stress config, the gather, ingest ----

@pytest.fixture(scope="module")
def full_scene(lumi, torch_cuda, oracle):
    """C3's model: T=2^22 (level 0 dense, levels 1-15 hashed) + its reference-baked occupancy,
    as the oracle's model and the product's DeviceModel."""
    s = scenes.FULL
    cfg = O.field_config(s.levels, s.features_per_level, s.base_resolution, s.per_level_scale,
                         s.table_size, s.hidden_width, s.bottleneck, 0)
    params = oracle.synth_params(cfg, s.seed, s.amplitude)
    bits, res, _ = load_occ(s.name)
    field, grid, dm = product_model(lumi, s, bits, res)
    return dict(spec=s, params=params, bits=bits, res=res, om=oracle.model(params, bits, res),
                field=field, grid=grid, dm=dm)


def test_c3_full_stereo_frame_vs_oracle(lumi, torch_cuda, oracle, full_scene):
    """BASELINE config C3 on whole frames: both 2048^2 eyes of the head path's first frame (the
    bench's first timed frame), rendered by the production kernel into the stacked eyebuffer
    and by the threaded oracle over every row.  Bars: max |dPQ| <= 1e-3 and PSNR >= 60 dB over
    the whole frame; opacity within 1e-3; the occupancy-kept candidate masks and kept counts of
    both eyes bit-exact on occ_full-T22; per-pixel evals / contributing mismatch rates
    reported (they can differ only where fp16 sigma moves the 1e-4 cut)."""
    torch = torch_cuda
    S = 2048
    rot, org = scenes.head_pose(0)
    eyes = scenes.eye_cameras(S, rot, org)
    dm, om = full_scene["dm"], full_scene["om"]
    opts = lumi.RenderOptions()
    rgb = torch.zeros((3, 2 * S, S), dtype=torch.float32, device="cuda")
    opac = torch.zeros((2 * S, S), dtype=torch.float32, device="cuda")
    counts = torch.zeros((2 * S, S, 2), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for e, spec in enumerate(eyes):
        t = lumi.renderer._abi.FrameTarget()
        t.rgb, t.opacity, t.counts = rgb.data_ptr(), opac.data_ptr(), counts.data_ptr()
        t.width, t.height, t.row_offset = S, 2 * S, e * S
        dm.render_rows_async(lumi.CameraModel.from_spec(spec), opts, 0, S, t, st)
    torch.cuda.synchronize()
    got, gop, gc = rgb.cpu().numpy(), opac.cpu().numpy(), counts.cpu().numpy()
    want = np.zeros_like(got)
    wop = np.zeros_like(gop)
    wev = np.zeros((2 * S, S), np.int32)
    wco = np.zeros((2 * S, S), np.int32)
    for e, spec in enumerate(eyes):
        ref = oracle.render_rows(om, ocam(spec), O.render_options(), 0, S)
        want[:, e * S:(e + 1) * S] = ref["out"]
        wop[e * S:(e + 1) * S] = ref["opacity"]
        wev[e * S:(e + 1) * S] = ref["evals"]
        wco[e * S:(e + 1) * S] = ref["contributing"]
    err, p = check_pixels("c3_frame", got, want)
    oerr = float(np.abs(gop - wop).max())
    ev_mis = float(np.mean(gc[..., 0] != wev))
    co_mis = float(np.mean(gc[..., 1] != wco))
    print(f"C3 stereo frame 2x{S}^2: max|dPQ|={err:.3e} PSNR={p:.1f} dB max|dopacity|={oerr:.3e} "
          f"evals mismatch {ev_mis:.2e} contributing mismatch {co_mis:.2e}")
    assert oerr <= PIX_TOL
    assert ev_mis <= 1e-3 and co_mis <= 1e-3
    # the MLP-independent part is exact: kept masks and counts of both eyes
    for e, spec in enumerate(eyes):
        cam = lumi.CameraModel.from_spec(spec)
        mask, kc = march_kept_gpu(torch, lumi, dm, cam, opts, 0, S)
        omask, okc = oracle.march_kept(om, ocam(spec), O.render_options(), 0, S)
        assert np.array_equal(kc, okc), f"eye {e} kept counts"
        assert np.array_equal(mask, omask), f"eye {e} kept masks"
        assert kc.sum() > 0


def test_c5_full_model_dense_band_vs_oracle(lumi, torch_cuda, oracle, full_scene):
    """BASELINE config C5 (4096^2 per eye, dense occupancy) with the FULL model (T=2^22): the
    production kernel renders a 16-row band through the centre of a head-path eye -- every
    candidate kept, up to 256 evaluations per ray -- against the oracle on the same rows."""
    s = full_scene
    ones = np.ones(s["res"] ** 3, np.uint8)
    dm = lumi.DeviceModel(s["field"], lumi.OccupancyGrid(s["res"], ones), 0)
    om = oracle.model(s["params"], ones, s["res"])
    rot, org = scenes.head_pose(45)
    spec = scenes.eye_cameras(4096, rot, org)[0]
    cam = lumi.CameraModel.from_spec(spec)
    out = np.zeros((3, 4096, 4096), np.float32)
    opac = np.zeros((4096, 4096), np.float32)
    stats = []
    b, e = 2040, 2056
    dm.render_rows(cam, lumi.RenderOptions(), b, e, out, None, opac, stats)
    ref = oracle.render_rows(om, ocam(spec), O.render_options(), b, e)
    band = slice(b, e)
    err, p = check_pixels("c5_band", out[:, band], ref["out"][:, band])
    ev = sum(st.evals for st in stats)
    print(f"C5 band (full model, dense): max|dPQ|={err:.3e} PSNR={p:.1f} dB evals {ev} "
          f"(oracle {int(ref['row_evals'].sum())}), {ev / (16 * 4096):.1f} evals/ray")
    assert np.abs(opac[band] - ref["opacity"][band]).max() <= PIX_TOL
    assert ev == pytest.approx(int(ref["row_evals"].sum()), rel=0.01)


@pytest.mark.parametrize("which", ["small", "full"])
def test_production_gather_vs_oracle_encode(lumi, torch_cuda, oracle, small, full_scene, which):
    """The renderer's own gather (pk::gather_row: fp16 table copy, seven packed-fp16 lerps,
    the weight applied in fp16) level by level against MultiResHashGrid::encode (grid.h:90-114) in
    the oracle, on uniform random and packet-coherent points with random / edge LOD weights.
    Bound per feature, from the error model of the fp16 arithmetic (entries |e| <= 1): the
    table's rounding (2^-12 |e|), the cell fraction from the rounded fp32 product u r (half an
    ulp of r, <= 2.4e-4 x |e1 - e0|), and three lerp stages of HADD2 + HFMA2 plus the weight's
    HMUL2, each rounding to 2^-11 of values <= 2 -> <= 6e-3 x w_l worst case (measured: ~2.6e-3
    on random points, ~4.1e-3 on the cell-face / domain-edge points below); rms 5e-4; masked
    levels (w_l = 0) exactly zero, as in the reference."""
    torch = torch_cuda
    if which == "small":
        dm, om, levels = small["dm"], small["model"], 16
    else:
        dm, om, levels = full_scene["dm"], full_scene["om"], 16
    rng = np.random.default_rng(11)
    n_rand, n_coh = 4096, 4096
    pos = np.empty((n_rand + n_coh, 3), np.float32)
    pos[:n_rand] = rng.uniform(-2.0, 2.0, (n_rand, 3))
    centers = rng.uniform(-1.9, 1.9, (n_coh // 32, 3))
    off = np.stack(np.meshgrid(np.arange(8), np.arange(4), indexing="xy"), -1).reshape(32, 2) * 4e-4
    coh = np.repeat(centers, 32, axis=0)
    coh[:, :2] += np.tile(off, (n_coh // 32, 1))
    pos[n_rand:] = coh
    # edges: the domain's faces (u = 0 and u -> 1, where the kernel's nearest-rounded cell
    # coordinate may land on res itself) and exact cell faces of every level on one axis
    res = [int(np.floor(128 * 1.4 ** l)) for l in range(levels)]
    faces = [4.0 * k / r - 2.0 for r in res for k in (1, r // 3, r // 2, r - 1)]
    edge = np.array([[c, e, f] for c in (-2.0, 2.0, 1.99999, -1.99999) for e in (-2.0, 0.3, 2.0)
                     for f in (-2.0, 2.0)] + [[x, 0.1, -0.7] for x in faces] + [[0.2, x, 1.3] for x in faces],
                    np.float32)
    pos = np.concatenate([pos, edge])
    fl = rng.uniform(0.0, 16.0, len(pos)).astype(np.float32)
    fl[::17] = 16.0   # every level fully active
    fl[5::17] = 1e-4  # the reference's L_eff < 0 case: only w_0 = 1e-4
    fl[9::17] = np.floor(fl[9::17])  # integer L: the next level exactly 0
    n = len(pos)
    d_pos = torch.from_numpy(pos).cuda()
    d_fl = torch.from_numpy(fl).cuda()
    d_out = torch.zeros((n, 2 * levels), dtype=torch.float32, device="cuda")
    dm.encode_async(n, d_pos.data_ptr(), d_fl.data_ptr(), d_out.data_ptr(),
                    torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = d_out.cpu().numpy()
    lodw = np.clip(fl[:, None] - np.arange(levels, dtype=np.float32)[None, :], 0.0, 1.0).astype(np.float32)
    _, _, feat = oracle.field_forward(om, pos.astype(np.float64), lodw, oracle.sh_encode(np.array([0.0, 0.0, 1.0])))
    want = feat.T  # [n][32]
    w2 = np.repeat(lodw, 2, axis=1)
    err = np.abs(got - want)
    assert (got[w2 == 0] == 0).all() and (want[w2 == 0] == 0).all()
    act = w2 > 0
    bound = 6e-3 * w2
    worst = float((err / np.maximum(w2, 1e-30))[act].max())
    rms = float(np.sqrt(np.mean(err[act] ** 2)))
    per_level = [float(err[:, 2 * l:2 * l + 2][act[:, 2 * l:2 * l + 2]].max(initial=0.0)) for l in range(levels)]
    print(f"gather {which}: max|df|/w_l={worst:.2e} rms={rms:.2e} per level max {np.round(per_level, 5).tolist()}")
    assert (err <= bound + 1e-7).all()
    assert rms <= 5e-4


def test_checkpoint_written_by_reference_renders_on_gpu(lumi, torch_cuda, reference, oracle,
                                                        golden_c1, tmp_path):
    """§8f row 2 on the device: the reference's save_checkpoint (scene.cpp:320-351) writes the C1
    model; the product's reader (load_checkpoint, scene.cpp:353-394) loads it into a
    DeviceModel that renders C1 within the parity bars of the reference's own image (golden)
    and identically to the in-memory model."""
    s = scenes.SMALL
    cfg = O.field_config(s.levels, s.features_per_level, s.base_resolution, s.per_level_scale,
                         s.table_size, s.hidden_width, s.bottleneck, 0)
    p = reference.synth_params(cfg, s.seed, s.amplitude)
    bits, res, _ = load_occ(s.name)
    path = tmp_path / "c1.lumickpt"
    reference.save_checkpoint(reference.model(p, bits, res), path, spp=256)
    field, grid, meta = lumi.load_checkpoint(path)
    assert meta["samples_per_ray"] == 256 and meta["contraction"] == lumi.ContractionMode.kLInfCubic
    dm = lumi.DeviceModel(field, grid, 0)
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 256))
    out = np.zeros((3, 256, 256), np.float32)
    dm.render_rows(cam, lumi.RenderOptions(samples_per_ray=meta["samples_per_ray"]), 0, 256, out)
    err, p_ = check_pixels("ckpt_c1", out, golden_c1["out"])
    mem = np.zeros_like(out)
    _, _, dm2 = product_model(lumi, s, bits, res)
    dm2.render_rows(cam, lumi.RenderOptions(), 0, 256, mem)
    print(f"checkpoint C1: max|dPQ|={err:.3e} PSNR={p_:.1f} dB vs the reference image")
    assert np.array_equal(out, mem)


def test_row_stats_ms_follow_row_cost(lumi, torch_cuda, small):
    """RowStats.ms (renderer.h:261, 272-276): each row gets the share of the launch time its
    packets took on the SM (cycle counters in the render kernel), so the per-row cost
    diagnostic tracks the rows' work (evaluations), and the rows add up to the launch."""
    cam = lumi.CameraModel.from_spec(scenes.pinhole(256, 256))
    out = np.zeros((3, 256, 256), np.float32)
    stats = []
    small["dm"].render_rows(cam, lumi.RenderOptions(), 0, 256, out, None, None, stats)
    ms = np.array([s.ms for s in stats])
    ev = np.array([s.evals for s in stats], np.float64)
    assert (ms > 0).all()
    assert np.isfinite(ms).all()
    r = float(np.corrcoef(ms, ev)[0, 1])
    print(f"row ms: total {ms.sum():.3f} ms, min {ms.min():.4f} max {ms.max():.4f}, corr(ms, evals) {r:.3f}")
    assert r > 0.5
    assert ms.std() > 0.05 * ms.mean()  # not the flat launch-time / rows split
