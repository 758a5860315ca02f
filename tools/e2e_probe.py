#!/usr/bin/env python
"""Where the end-to-end (host-buffer) time goes for one 2K eye of C3: lumi_render_rows vs the
device-resident render + a pinned D2H of the same planes."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2311_02542_b200 as L  # noqa: E402
from paper_2311_02542_b200 import _abi, scenes  # noqa: E402
from bench import load_scene  # noqa: E402

field, grid = load_scene(scenes.FULL)
dm = L.DeviceModel(field, grid, 0)
cam = L.CameraModel.from_spec(scenes.eye_cameras(2048)[0])
opts = L.RenderOptions()
host = torch.empty((3, 2048, 2048), dtype=torch.float32).pin_memory()
hn = host.numpy()
dev = torch.empty((3, 2048, 2048), dtype=torch.float32, device="cuda")


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / n


tgt = _abi.FrameTarget()
tgt.rgb = dev.data_ptr()
tgt.width, tgt.height, tgt.row_offset = 2048, 2048, 0
s = torch.cuda.current_stream().cuda_stream
print("render_rows (host buffers)   %.2f ms" % t(lambda: dm.render_rows(cam, opts, 0, 2048, hn)))
print("render_rows_async (device)   %.2f ms" % t(lambda: dm.render_rows_async(cam, opts, 0, 2048, tgt, s)))
print("D2H 48 MB pinned             %.2f ms" % t(lambda: host.copy_(dev, non_blocking=True)))

# the bench's e2e loop: head-path frames, both eyes, per-call wall time
from paper_2311_02542_b200.multigpu import StereoFrameDriver  # noqa: E402
drv = StereoFrameDriver(torch, dm, 2048, opts, 0, 1, dist=None, counters=True)
hosts = torch.empty((2, 3, 2048, 2048), dtype=torch.float32).pin_memory().numpy()
for f in range(3, 9):
    cams = drv.cameras(f)
    ts = []
    for eye in range(2):
        t0 = time.perf_counter()
        dm.render_rows(cams[eye], opts, 0, 2048, hosts[eye])
        ts.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    drv.frame(f)
    torch.cuda.synchronize()
    print("frame %d: render_rows %.2f + %.2f ms; device frame %.2f ms" % (f, ts[0], ts[1], (time.perf_counter() - t0) * 1e3))
