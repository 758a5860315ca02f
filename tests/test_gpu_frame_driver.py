"""The native multi-GPU frame driver (lumi_frame_driver_*): run_frame
(scheduler.cpp:114-152) with one host thread per worker and the bands stored into one device
frame, next_assignment (scheduler.cpp:154-162) from per-worker CUDA-event ms.

The box has one GPU, so the workers share it (one stream each): the frame must equal a
single-call render of both eyes bit for bit whatever the partition, and the partition must
follow the reference scheduler's arithmetic on the measured times."""
import numpy as np
import pytest

from conftest import load_occ
from paper_2311_02542_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch


@pytest.fixture(scope="module")
def setup(torch_cuda):
    import paper_2311_02542_b200 as L
    s = scenes.SMALL
    cfg = L.FieldConfig(grid=L.HashGridConfig(table_size=s.table_size))
    field = L.RadianceField.synthetic(cfg, s.seed, s.amplitude)
    bits, res, _ = load_occ(s.name)
    grid = L.OccupancyGrid(res, bits)
    return L, field, grid


def _reference_frame(torch, L, dm, cams, opts, S):
    rgb = torch.zeros((3, 2 * S, S), dtype=torch.float32, device="cuda")
    for eye in range(2):
        t = L.renderer._abi.FrameTarget()
        t.rgb, t.width, t.height, t.row_offset = rgb.data_ptr(), S, 2 * S, eye * S
        dm.render_rows_async(cams[eye], opts, 0, S, t, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return rgb.cpu().numpy()


@pytest.mark.parametrize("workers,shared_model", [(1, True), (3, True), (4, False)])
def test_native_driver_frames_equal_single_render(setup, torch_cuda, workers, shared_model):
    L, field, grid = setup
    from paper_2311_02542_b200.multigpu import NativeFrameDriver
    from paper_2311_02542_b200.scheduler import equal_assignment
    torch = torch_cuda
    S = 192
    dm = L.DeviceModel(field, grid, 0)
    models = [dm] * workers if shared_model else [L.DeviceModel(field, grid, 0) for _ in range(workers)]
    drv = NativeFrameDriver(models, S, eyes=2, dampening=0.5)
    assert drv.assignment().rows().tolist() == equal_assignment(2 * S, workers).rows().tolist()
    opts = L.RenderOptions()
    rgb = torch.zeros((3, 2 * S, S), dtype=torch.float32, device="cuda")
    evals = torch.zeros(2 * S, dtype=torch.int64, device="cuda")
    seen = set()
    for f in range(5):
        rot, org = scenes.head_pose(7 * f)
        cams = [L.CameraModel.from_spec(c) for c in scenes.eye_cameras(S, rot, org)]
        if f == 3 and workers > 1:  # a band straddling the eye seam, the rest tiny
            rows = [1] * (workers - 1) + [2 * S - (workers - 1)]
            rows[0] = S + 5
            rows[-1] = 2 * S - sum(rows[:-1])
            drv.set_assignment(rows)
        before = drv.assignment()
        seen.add(tuple(before.rows().tolist()))
        rgb.fill_(-1.0)
        t = L.renderer._abi.FrameTarget()
        t.rgb, t.width, t.height = rgb.data_ptr(), S, 2 * S
        st = drv.render(cams, opts, t)
        got = rgb.cpu().numpy()
        want = _reference_frame(torch, L, dm, cams, opts, S)
        assert np.array_equal(got, want), f"frame {f}"
        assert len(st.worker_ms) == workers and all(m > 0 for m in st.worker_ms)
        assert st.worker_rays == [r * S for r in before.rows().tolist()]
        if workers > 1:
            # the next partition is the reference scheduler's on the measured times
            from paper_2311_02542_b200.scheduler import next_assignment
            assert drv.assignment().rows().tolist() == next_assignment(before, st, 0.5).rows().tolist()
    if workers > 1:
        assert len(seen) > 1  # the partition moved
    drv.close()
    del evals


def test_native_driver_worker_failure_fails_the_frame(setup, torch_cuda):
    L, field, grid = setup
    from paper_2311_02542_b200.multigpu import NativeFrameDriver
    torch = torch_cuda
    S = 64
    dm = L.DeviceModel(field, grid, 0)
    drv = NativeFrameDriver([dm, dm], S, eyes=2)
    rgb = torch.zeros((3, 2 * S, S), dtype=torch.float32, device="cuda")
    t = L.renderer._abi.FrameTarget()
    t.rgb, t.width, t.height = rgb.data_ptr(), S, 2 * S
    bad = L.CameraModel.from_spec(scenes.pinhole(S, S))
    bad.t_near = -1.0  # march_ray: bad sampling interval (renderer.h:134)
    with pytest.raises(L.Error, match="run_frame: worker 0 failed"):
        drv.render([bad, bad], L.RenderOptions(), t)
    # host memory is not a device frame target
    host = np.zeros((3, 2 * S, S), np.float32)
    t.rgb = host.ctypes.data
    cams = [L.CameraModel.from_spec(c) for c in scenes.eye_cameras(S)]
    with pytest.raises(L.Error):
        drv.render(cams, L.RenderOptions(), t)
    drv.close()
