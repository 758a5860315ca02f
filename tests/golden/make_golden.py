"""Generates the committed golden fixtures under tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/liblumi_ref.so, compiled from /root/reference by oracle/Makefile).

  python tests/golden/make_golden.py [--full]

Outputs
  occ_<model>.npz      reference-baked 128^3 occupancy (packed bits), near-threshold voxel
                       indices and a 1-in-97 sample of the probe maxima
  render_c1.npz        reference render of config C1 (256x256, probe camera) with per-pixel
                       evals / contributing / kept counts, plus the occupancy-kept sample
                       bitmask for a 64x64 crop
  meta.json            recipe, reference ISA variant, statistics

Run here (the reference checkout exists only in the build container); the GPU box uses the
committed files.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2311_02542_b200 import scenes  # noqa: E402


def cfg_of(spec):
    return O.field_config(spec.levels, spec.features_per_level, spec.base_resolution,
                          spec.per_level_scale, spec.table_size, spec.hidden_width,
                          spec.bottleneck, 0)


def cam_of(c):
    return O.camera(c.rot, c.origin, c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.t_near, c.t_far)


def bake(ref, spec, meta):
    cfg = cfg_of(spec)
    p = ref.synth_params(cfg, spec.seed, spec.amplitude)
    res = spec.occ_res
    ones = np.ones(res ** 3, np.uint8)
    m = ref.model(p, ones, res)
    probe_cam = cam_of(scenes.pinhole(256, 256))
    t = time.time()
    pm, occ = ref.probe_prune(m, [probe_cam], scenes.SAMPLES_PER_RAY, scenes.PROBE_POINTS_PER_AXIS,
                              res, spec.prune_alpha)
    dt = time.time() - t
    # bits + the voxels whose probe value is within 1% of alpha (where a different MLP
    # summation order may flip the bit) + every 97th probe value, to keep the fixture small
    near = np.nonzero(np.abs(pm - spec.prune_alpha) <= 0.01 * spec.prune_alpha)[0]
    samp = np.arange(0, pm.size, 97, dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, f"occ_{spec.name}.npz"), bits=np.packbits(occ),
                        res=res, near_threshold=near.astype(np.int32), probe_sample_idx=samp,
                        probe_sample=pm[samp].astype(np.float32))
    meta[f"occ_{spec.name}"] = dict(occupied=int(occ.sum()), voxels=int(occ.size),
                                     bake_seconds=round(dt, 1), alpha=spec.prune_alpha,
                                     probe_k=scenes.PROBE_POINTS_PER_AXIS)
    print(spec.name, "occupied", int(occ.sum()), "bake", dt, "s", flush=True)
    return p, occ


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true", help="also bake the T=2^22 model")
    args = ap.parse_args()
    ref = O.Reference()
    meta_path = os.path.join(HERE, "meta.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    meta["reference_simd"] = ref.simd_name()
    meta["recipe"] = dict(seed=scenes.SEED, amplitude=scenes.GRID_AMPLITUDE,
                          alpha=scenes.PRUNE_ALPHA, probe_rot=scenes.PROBE_ROT,
                          probe_origin=scenes.PROBE_ORIGIN, spp=scenes.SAMPLES_PER_RAY)
    p, occ = bake(ref, scenes.SMALL, meta)
    m = ref.model(p, occ, scenes.SMALL.occ_res)
    cam = cam_of(scenes.pinhole(256, 256))
    opts = O.render_options()
    t = time.time()
    r = ref.render_rows(m, cam, opts, 0, 256)
    meta["render_c1_seconds_1thread"] = round(time.time() - t, 2)
    mask, counts = ref.march_kept(m, cam, opts, 96, 160)
    np.savez_compressed(os.path.join(HERE, "render_c1.npz"), out=r["out"], depth=r["depth"],
                        opacity=r["opacity"], evals=r["evals"].astype(np.int16),
                        contributing=r["contributing"].astype(np.int16),
                        kept=r["kept"].astype(np.int16), row_evals=r["row_evals"],
                        kept_mask_rows=np.array([96, 160]),
                        kept_mask=mask[96:160, 96:160], kept_counts=counts[96:160])
    meta["render_c1"] = dict(mean_evals=float(r["evals"].mean()),
                             mean_opacity=float(r["opacity"].mean()),
                             mean_kept_all=float(counts[96:160].mean()))
    print("C1 render", meta["render_c1"], flush=True)
    if args.full:
        bake(ref, scenes.FULL, meta)
    json.dump(meta, open(meta_path, "w"), indent=1)


if __name__ == "__main__":
    main()
