"""The peer-memory frame gather on one B200: two processes share cuda:0 (the
box has one GPU; CUDA IPC maps rank 0's frame buffers into rank 1 exactly as it would across
NVLink peers), gloo carries the handle broadcast and the band-time exchange.  Rank 1's render
kernel stores its band straight into rank 0's buffer; the stacked stereo frames rank 0 ends up
with equal a single-process render of the same frames, over several frames of rebalanced
bands and alternating buffers."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

S = 96  # eye size: 2 x 96 x 96 stacked frame
FRAMES = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    import paper_2311_02542_b200 as L
    from conftest import load_occ
    from paper_2311_02542_b200 import scenes
    spec = scenes.SMALL
    cfg = L.FieldConfig(grid=L.HashGridConfig(spec.levels, spec.features_per_level,
                                              spec.base_resolution, spec.per_level_scale,
                                              spec.table_size))
    field = L.RadianceField.synthetic(cfg, spec.seed, spec.amplitude)
    bits, res, _ = load_occ(spec.name)
    return L, L.DeviceModel(field, L.OccupancyGrid(res, bits), 0)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2311_02542_b200.multigpu import StereoFrameDriver
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, dm = _model()
        drv = StereoFrameDriver(torch, dm, S, L.RenderOptions(), rank, world, dist=dist,
                                gather="p2p")
        bands = []
        for f in range(FRAMES):
            bands.append([(r.begin, r.end) for r in drv.assign.ranges])
            drv.frame(f)
            if rank == 0:
                np.save(os.path.join(out_dir, f"frame{f}.npy"), drv.frame_buffer(f).cpu().numpy())
        drv.close()
        dist.barrier()  # rank 0's buffers outlive every mapping
        if rank == 0:
            np.save(os.path.join(out_dir, "bands.npy"), np.array(bands))
    finally:
        dist.destroy_process_group()


def test_two_processes_render_into_rank0_frame(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    from paper_2311_02542_b200.multigpu import StereoFrameDriver
    L, dm = _model()
    ref = StereoFrameDriver(torch, dm, S, L.RenderOptions())
    bands = np.load(tmp_path / "bands.npy")
    assert (bands[:, 1, 1] - bands[:, 1, 0] > 0).all()  # rank 1 rendered a band every frame
    for f in range(FRAMES):
        ref.frame(f)
        want = ref.frame_buffer(f).cpu().numpy()
        got = np.load(tmp_path / f"frame{f}.npy")
        assert want.max() > 0
        assert np.array_equal(got, want), f"frame {f}: max diff {np.abs(got - want).max()}"


def test_ipc_rejects_unknown_pointer():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2311_02542_b200 as L
    from paper_2311_02542_b200 import _abi
    with pytest.raises(L.Error):
        _abi.check(_abi.lib().lumi_ipc_close(0, 12345))


def test_single_gpu_frames_back_to_back_equal_synchronous():
    """One GPU: frames enqueued back to back (frame(sync=False) + collect(), the bench's timed
    loop) render the same pixels as frames each followed by the band-time exchange, give one
    FrameStats per frame in order, and keep the single worker's assignment."""
    import torch
    from paper_2311_02542_b200.multigpu import StereoFrameDriver
    L, dm = _model()
    sync = StereoFrameDriver(torch, dm, S, L.RenderOptions())
    want = []
    for f in range(3):
        sync.frame(f)
        want.append(sync.frame_buffer(f).cpu().numpy().copy())
    drv = StereoFrameDriver(torch, dm, S, L.RenderOptions())
    for f in range(3):  # back to back: the one frame buffer ends with the last frame
        assert drv.frame(f, sync=False) is None
    stats = drv.collect()
    assert len(stats) == 3 and all(s.wall_ms > 0 for s in stats)
    assert np.array_equal(drv.frame_buffer(2).cpu().numpy(), want[2])
    assert [(r.begin, r.end) for r in drv.assign.ranges] == [(0, 2 * S)]
    for f in range(3):  # and each enqueued frame alone
        drv.frame(f, sync=False)
        torch.cuda.synchronize()
        assert np.array_equal(drv.frame_buffer(f).cpu().numpy(), want[f])
    assert len(drv.collect()) == 3 and drv.collect() == []
