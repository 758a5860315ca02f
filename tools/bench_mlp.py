#!/usr/bin/env python
"""The renderer's tcgen05 MLP on an isolated dense batch: n samples of 32 fp16
features through lumi_mlp_batch_async, timed with CUDA events; reports samples/s and the
algorithmic TFLOP/s (18,944 FLOP per sample) against the measured bf16 BURST peak
(MEASURED_PEAKS.json bf16_tflops: the kernel is timed alone, not inside a long step).

  python tools/bench_mlp.py [--n 16777216 --steps 10]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import paper_2311_02542_b200 as L
    from paper_2311_02542_b200 import scenes
    from bench import load_scene, measured_peaks

    field, grid = load_scene(scenes.FULL)
    dm = L.DeviceModel(field, grid, 0)
    g = torch.Generator(device="cuda").manual_seed(0)
    feat = (torch.rand((a.n, 32), device="cuda", generator=g) * 2 - 1).half()
    dirs = torch.nn.functional.normalize(torch.randn((a.n, 3), device="cuda", generator=g), dim=1)
    out = torch.empty((a.n, 4), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        dm.mlp_batch_async(feat.data_ptr(), dirs.data_ptr(), a.n, out.data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        dm.mlp_batch_async(feat.data_ptr(), dirs.data_ptr(), a.n, out.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    tflops = 18944.0 * a.n / (ms * 1e-3) / 1e12
    peak = measured_peaks().get("bf16_tflops") or 1629.0  # burst: an isolated kernel
    print(json.dumps({"metric": "isolated MLP batch (density 32-64-17 + colour 32-64-64-3, fp16 tcgen05)",
                      "samples": a.n, "ms": round(ms, 3), "Msamples_s": round(a.n / ms / 1e3, 1),
                      "tflops": round(tflops, 2), "peak_tflops": peak, "frac": round(tflops / peak, 4),
                      "bytes_per_sample": 64 + 12 + 16}))


if __name__ == "__main__":
    main()
