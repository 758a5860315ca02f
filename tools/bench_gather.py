#!/usr/bin/env python
"""The renderer's hash-grid gather in isolation: every level of n points through
gather_row (the production producer gather) on the fp16 table, for the L2-resident T=2^19 table (C1/C2) and the T=2^22 table
(C3-C5, 260 MB > L2), with packet-coherent and uniform random points.  Reports level-samples/s
and the algorithmic gather GB/s (32 B per level-sample: 8 corners x 2 fp16 features), i.e. the
attainable gather rate the renderer's roofline can be read against.

  python tools/bench_gather.py [--n 4194304 --steps 10]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import paper_2311_02542_b200 as L
    from paper_2311_02542_b200 import scenes
    from bench import load_scene

    res = {}
    out = torch.empty(a.n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for spec in (scenes.SMALL, scenes.FULL):
        field, grid = load_scene(spec)
        dm = L.DeviceModel(field, grid, 0)
        levels = field.cfg.grid.levels
        for coherent in (True, False):
            for _ in range(2):
                dm.gather_bench_async(a.n, coherent, out.data_ptr(), st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.steps):
                dm.gather_bench_async(a.n, coherent, out.data_ptr(), st)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            ls = a.n * levels / (ms * 1e-3)
            res[f"T2^{spec.table_log2}_{'coherent' if coherent else 'random'}"] = {
                "table_MB_fp16": round(field.grid_params.nbytes / 2e6, 1), "ms": round(ms, 3),
                "Glevel_samples_s": round(ls / 1e9, 2), "gather_GBs": round(32 * ls / 1e9, 1)}
        del dm
    print(json.dumps({"metric": "hash-grid gather in isolation (renderer gather_row, all 16 levels "
                                "per point)", "points": a.n, "results": res}))


if __name__ == "__main__":
    main()
