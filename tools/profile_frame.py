"""Renders a few stereo frames of a config through the production path, for ncu / launch-list
captures (never for timing):  python tools/profile_frame.py [C3] [frames]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_02542_b200 as L  # noqa: E402
from paper_2311_02542_b200 import scenes  # noqa: E402
from paper_2311_02542_b200.multigpu import StereoFrameDriver  # noqa: E402

cfg = scenes.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
field, grid = bench.load_scene(cfg.model)
dm = L.DeviceModel(field, grid, 0)
drv = StereoFrameDriver(torch, dm, cfg.eye_size, L.RenderOptions(), counters=True)
for f in range(frames):
    drv.frame(f)
torch.cuda.synchronize()
print("frames", frames, "counters", drv.counters().tolist(), "launches", drv.launches)
