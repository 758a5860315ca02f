#!/usr/bin/env python
"""Headline benchmark: dual 2048x2048 eyebuffers of the full-size synthetic VR-NeRF model
(BASELINE.json config C3 at N=1, C4's dynamic row balancing at N>1), Mrays/s and fps.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config C3]

A step is one stereo frame (2 x 2048^2 = 8,388,608 rays) along the 120-frame head path.
N>1 runs under torch.distributed.run, one rank per GPU (NCCL), rows of the stacked dual-eye
image split by the throughput-proportional scheduler and gathered to rank 0 each frame.
Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/sec and fps for dual 2K×2K eyebuffers at 1/2/4/8 B200 vs CPU ref"
UNIT = "Mrays/s"
GATHER_BYTES_PER_LEVEL_SAMPLE = 8 * 2 * 4  # 8 corners x 2 features x fp32
# what the timed kernels compute in: the hash table and the MLP operands are fp16 (tcgen05
# kind::f16, fp32 accumulators in TMEM), sample positions / contraction / LOD are fp32 (the
# occupancy decisions certified against the reference's double arithmetic, undecided ones
# re-tested in f64), the transmittance that decides the early cut is f64
DTYPE = "fp16 table + fp16 MLP operands (fp32 accum), fp32 geometry/LOD, f64 transmittance"
MLP_FLOP_PER_SAMPLE = 18944  # 9,472 MACs per evaluated sample


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3", choices=["C2", "C3", "C4", "C5"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU time of the reference baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="frames of the end-to-end leg (default: --steps, the timed frames)")
    ap.add_argument("--no-checkpoint", action="store_true",
                    help="build the scene in memory instead of through a LUMICKPT round trip")
    return ap.parse_args()


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1, as the driver does; rank 0's JSON line passes through.
    NCCL's INIT log stays on so the communicator's N ranks are visible in the output."""
    import socket
    shared = os.environ.get("LUMI_BENCH_SHARED_GPU") == "1"
    if not shared:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: this host has {have} CUDA device(s)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def occupancy_bits(spec):
    """The scene's occupancy bits: the reference-baked 128^3 grid of SURVEY.md §8d (committed
    fixture), or all-occupied for the dense stress config."""
    if spec.dense_occupancy:
        return spec.occ_res, np.ones(spec.occ_res ** 3, np.uint8)
    z = np.load(os.path.join(ROOT, "tests", "golden", f"occ_{spec.name.replace('-dense', '')}.npz"))
    res = int(z["res"])
    return res, np.unpackbits(z["bits"])[: res ** 3]


def load_scene(spec, via_checkpoint: bool = True):
    """Synthetic bake of SURVEY.md §8d: seeded parameters + the reference-baked occupancy,
    written to a LUMICKPT v1 checkpoint (save_checkpoint, scene.cpp:320-351) and loaded back
    through the product's checkpoint reader (load_checkpoint, scene.cpp:353-394) -- the model
    reaches the GPU the way a trained scene would."""
    import tempfile
    import paper_2311_02542_b200 as L
    g = L.HashGridConfig(spec.levels, spec.features_per_level, spec.base_resolution,
                         spec.per_level_scale, spec.table_size)
    field = L.RadianceField.synthetic(L.FieldConfig(grid=g), spec.seed, spec.amplitude)
    res, bits = occupancy_bits(spec)
    grid = L.OccupancyGrid(res, bits)
    if not via_checkpoint:
        return field, grid
    with tempfile.TemporaryDirectory(prefix="lumi_bench_") as d:
        path = os.path.join(d, f"{spec.name}.lumickpt")
        L.save_checkpoint(path, field, grid, samples_per_ray=256)
        field2, grid2, _ = L.load_checkpoint(path)
    return field2, grid2


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap",
              "utilization.gpu"]

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) == len(self.FIELDS):
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        busy = [r for r in rows if r[6].isdigit() and int(r[6]) > 0] or rows
        sm = sorted(float(r[0]) for r in busy if r[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(busy[0][1]) if busy[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(busy)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def gather_isolated(achieved, table_log2: int):
    """The in-frame gather rate next to the same gather code run alone (tools/bench_gather.py ->
    profiles/r02_bench_gather.json, all 16 levels of synthetic packet-coherent points on this
    table).  A comparison, not a ceiling: real ray packets are more coherent than the synthetic
    points, so the frame can gather faster than the isolated benchmark."""
    src = None
    for name in ("r02_bench_gather.json", "r01_bench_gather.json"):
        try:
            g = json.load(open(os.path.join(ROOT, "profiles", name)))
            iso = g["results"][f"T2^{table_log2}_coherent"]["gather_GBs"]
            src = name
            break
        except Exception:
            continue
    if src is None or achieved is None:
        return None
    return {"in_frame_GBs": round(achieved, 1), "isolated_coherent_GBs": iso,
            "ratio": round(achieved / iso, 4), "source": f"profiles/{src}",
            "note": "comparison with the isolated gather benchmark, not a hardware ceiling"}


def ncu_kernel(kernel: str, config: str = "C3"):
    """The render kernel's entry of the committed ncu --set full summary (profiles/), if any --
    only for the workload the capture was taken on (one C3 eye: per-launch figures do not carry
    over to another eye size or scene)."""
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        if prof.get("workload", "C3") != config:
            return {}
        k = dict(prof["kernels"].get(kernel) or {})
        k["_source"] = f"profiles/{prof.get('source', 'ncu_summary.json')}"
        return k
    except Exception:
        return {}


def ncu_traffic(kernel: str, config: str):
    """dram bytes per launch from the committed ncu --set full capture, if any."""
    return ncu_kernel(kernel, config).get("dram_bytes_per_launch")


def issue_roofline(kernel: str, config: str, ms_per_launch: float, sm_mhz):
    """The binding limit of the render kernel: warp-instruction issue.  ncu's executed warp
    instructions per launch of the same kernel and workload (one C3 eye) over the live
    per-launch time, against 4 issue slots per SM per clock x 148 SMs."""
    k = ncu_kernel(kernel, config)
    wi = k.get("warp_instructions")
    if not wi or not ms_per_launch or not sm_mhz:
        return None
    achieved = wi / (ms_per_launch / 1e3) / 1e9
    peak = 4 * 148 * float(sm_mhz) / 1e3
    return {"bound": "issue", "achieved": round(achieved, 1), "peak": round(peak, 1),
            "unit": "G warp-instructions/s", "frac": round(achieved / peak, 4),
            "ncu_issue_active": k.get("issue_active_pct"),
            "source": f"{k['_source']}: {wi:.4g} warp instructions per launch; peak = 4 issue "
                      f"slots/SM/clk x 148 SMs x {float(sm_mhz):.0f} MHz (sampled under load)"}


# --------------------------------------------------------------------------- reference

def reference_model(spec):
    """The same scene for the reference's own renderer (oracle/_ref): its own init_random +
    grid overwrite (ref_wrap.cpp ref_synth_params, bit-identical to the product's) and the same
    occupancy bits -- the reference arm loads nothing from the product library."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    ref = O.Reference()
    cfg = O.field_config(spec.levels, spec.features_per_level, spec.base_resolution,
                         spec.per_level_scale, spec.table_size, spec.hidden_width,
                         spec.bottleneck, 0)
    p = ref.synth_params(cfg, spec.seed, spec.amplitude)
    res, bits = occupancy_bits(spec)
    return O, ref, ref.model(p, bits, res)


SAMPLE_BANDS = 8


def reference_sample(O, ref, model, cam_spec, target_s, threads):
    """Times the reference run_frame (scheduler.cpp:114) over SAMPLE_BANDS bands of rows
    spread evenly down one eye (a representative sample of the frame), sized to take about
    target_s seconds in total; returns (rays/s, rows, seconds)."""
    cam = O.camera(cam_spec.rot, cam_spec.origin, cam_spec.fx, cam_spec.fy, cam_spec.cx,
                   cam_spec.cy, cam_spec.width, cam_spec.height, cam_spec.t_near, cam_spec.t_far)
    opts = O.render_options()
    H, W = cam_spec.height, cam_spec.width

    def run(band_rows):
        total_ms = 0.0
        for k in range(SAMPLE_BANDS):
            b = int((k + 0.5) * H / SAMPLE_BANDS) - band_rows // 2
            b = min(max(b, 0), H - band_rows)
            ms, _ = ref.run_frame(model, cam, opts, b, b + band_rows, threads)
            total_ms += ms
        return total_ms

    band = max(threads, 2)
    ms = run(band)
    rate = SAMPLE_BANDS * band * W / (ms / 1000.0)
    band = int(min(H // SAMPLE_BANDS, max(threads, target_s * rate / W / SAMPLE_BANDS)))
    ms = run(band)
    rows = SAMPLE_BANDS * band
    return rows * W / (ms / 1000.0), rows, ms / 1000.0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2311_02542_b200 import scenes
    cfg = scenes.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    try:
        O, ref, model = reference_model(cfg.model)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference build missing: {e}"}))
        return
    rays_frame = cfg.eyes * cfg.eye_size ** 2
    rot, origin = scenes.head_pose(0)
    eye = scenes.eye_cameras(cfg.eye_size, rot, origin)[0]
    per_step_s = min(6.0, max(1.0, 120.0 / max(args.steps + args.warmup, 1)))
    rate, rows, _ = reference_sample(O, ref, model, eye, per_step_s, threads)
    for _ in range(max(args.warmup - 1, 0)):
        reference_sample(O, ref, model, eye, per_step_s, threads)
    rates = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, rows, _ = reference_sample(O, ref, model, eye, per_step_s, threads)
        rates.append(r)
    wall = time.perf_counter() - t0
    mrays = float(np.mean(rates)) / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": round(mrays, 6), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall * 1000 / max(args.steps, 1), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 geometry / f32 field / f64 compositing",
        "data": "synthetic (seeded init_random + reference-baked occupancy)",
        "config": {"workload": f"{args.config}: {cfg.description}", "eye_size": cfg.eye_size,
                   "eyes": cfg.eyes, "table_size": cfg.model.table_size,
                   "rays_per_frame": rays_frame, "parallelism": f"{threads} host threads"},
        "fps": round(mrays * 1e6 / rays_frame, 6),
        "cpu_baseline": {"value": round(mrays, 6), "unit": UNIT, "cores": threads,
                         "kind": "reference",
                         "sample": f"run_frame over {rows} rows ({SAMPLE_BANDS} evenly spread "
                                   f"bands) x {cfg.eye_size} of the "
                                   f"left eye per step, simd={ref.simd_name()}"},
        "e2e": {"value": round(mrays, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------- ours

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2311_02542_b200 as L
    from paper_2311_02542_b200 import _abi, scenes
    from paper_2311_02542_b200.multigpu import StereoFrameDriver
    from paper_2311_02542_b200.scheduler import aggregate_stats

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # LUMI_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 over gloo, so the N>1 path
    # (scheduler bands, peer-memory gather through CUDA IPC, rebalancing) runs on a one-GPU box
    shared = os.environ.get("LUMI_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    red_dev = "cpu" if shared else "cuda"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = scenes.CONFIGS[args.config]
    spec = cfg.model
    field, grid = load_scene(spec, via_checkpoint=not args.no_checkpoint)
    dm = L.DeviceModel(field, grid, local)
    opts = L.RenderOptions()
    drv = StereoFrameDriver(torch, dm, cfg.eye_size, opts, rank, world, dist=dist if world > 1 else None,
                            counters=True)
    rays_frame = drv.H * drv.W

    for f in range(args.warmup):
        drv.frame(f)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    drv.stats.zero_()
    drv.launches = 0
    kernel_ms = 0.0
    dm.take_timing()
    dm.set_timing(True)  # events around each launch's march pass and render kernel
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_start.record()
        frames = []
        for k in range(args.steps):
            # one GPU: frames are enqueued back to back (the single worker's assignment never
            # changes); N GPUs: each frame's band times drive the next assignment
            st = drv.frame(args.warmup + k, sync=world > 1)
            if st is not None:
                frames.append(st)
        t_end.record()
        torch.cuda.synchronize()
        frames += drv.collect()
        kernel_ms = sum(st.worker_ms[rank] for st in frames)
        if world > 1:
            dist.barrier()
    dm.set_timing(False)
    march_ms, render_ms, render_launches = dm.take_timing()
    elapsed = float(t_start.elapsed_time(t_end))
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    counters = drv.counters()
    launches = drv.launches
    if world > 1:
        t = torch.tensor([float(x) for x in counters] + [float(launches), kernel_ms],
                         dtype=torch.float64, device=red_dev)
        dist.all_reduce(t)
        counters = t[:4].cpu().numpy()
        launches = int(t[4].item())
    sec = elapsed / 1000.0
    value = rays_frame * args.steps / sec / 1e6
    fstats = aggregate_stats(frames)
    fps = args.steps / sec

    # ---- end to end through the public API with host buffers -------------------------
    # the end-to-end leg renders the same head-path frames as the timed region (frame cost
    # varies along the path), so the two numbers differ only by what e2e adds
    e2e_steps = max(1, args.e2e_steps if args.e2e_steps is not None else args.steps)
    d2h = 3 * rays_frame * 4
    h2d = 2 * (C.sizeof(_abi.CameraDesc) + C.sizeof(_abi.RenderOptionsDesc))
    if world == 1:
        # the frame driver renders the stacked eye pair (rays_frame), so does the e2e leg
        host = torch.empty((2, 3, cfg.eye_size, cfg.eye_size), dtype=torch.float32).pin_memory()
        host_np = host.numpy()
        cams = drv.cameras(0)
        dm.render_rows(cams[0], opts, 0, cfg.eye_size, host_np[0])  # warm
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            cams = drv.cameras(args.warmup + k)  # the timed region's first frames
            for eye in range(2):
                dm.render_rows(cams[eye], opts, 0, cfg.eye_size, host_np[eye])
        e2e_s = time.perf_counter() - t0
    else:
        host = torch.empty((3, drv.H, drv.W), dtype=torch.float32).pin_memory()
        dist.barrier()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            drv.frame(args.warmup + k)
            if rank == 0:
                host.copy_(drv.frame_buffer(args.warmup + k), non_blocking=True)
            torch.cuda.synchronize()
        dist.barrier()
        e2e_s = time.perf_counter() - t0
        t = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = rays_frame * e2e_steps / e2e_s / 1e6
    if world > 1:
        drv.close()
        dist.barrier()  # rank 0's frame buffers outlive the peers' mappings

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    mlp_peak = peaks.get("bf16_tflops_sustained", 1398.6)
    clocks = clk.summary()
    evals, level_samples, candidates, rays = (float(x) for x in counters)
    # the tensor-core kernel gathers the fp16 copy of the table (32 B per level-sample), the
    # SIMT cross-check the reference fp32 layout (64 B)
    bytes_per_ls = GATHER_BYTES_PER_LEVEL_SAMPLE // (1 if dm.kernel == "simt" else 2)
    kname = {"simt": "k_render_simt", "ws": "k_render_ws"}[dm.kernel]
    gather_bytes = level_samples * bytes_per_ls
    # the render kernel's own launches on rank 0 (CUDA events on the launch stream around
    # each launch, march pass excluded); counters are summed over ranks, so scale by 1/world
    kernel_s = render_ms / 1000.0
    frac_rank = 1.0 / world
    achieved = gather_bytes * frac_rank / kernel_s / 1e9 if kernel_s > 0 else None
    mlp_tflops = evals * frac_rank * MLP_FLOP_PER_SAMPLE / kernel_s / 1e12 if kernel_s > 0 else None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            O, ref, model = reference_model(spec)
            rot, origin = scenes.head_pose(0)
            eye = scenes.eye_cameras(cfg.eye_size, rot, origin)[0]
            threads = os.cpu_count() or 1
            rate, rows, secs = reference_sample(O, ref, model, eye, args.cpu_seconds, threads)
            cpu = {"value": round(rate / 1e6, 6), "unit": UNIT, "cores": threads,
                   "kind": "reference",
                   "sample": f"reference run_frame over {rows} rows ({SAMPLE_BANDS} evenly "
                             f"spread bands) x {cfg.eye_size} of "
                             f"the left eye ({rows * cfg.eye_size} rays, {secs:.1f}s), "
                             f"simd={ref.simd_name()}"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic (seeded init_random + reference-baked occupancy, through a LUMICKPT "
                "checkpoint round trip)" if not args.no_checkpoint else
                "synthetic (seeded init_random + reference-baked occupancy)",
        "config": {"workload": f"{args.config}: {cfg.description}", "eye_size": cfg.eye_size,
                   "eyes": 2, "table_size": spec.table_size, "rays_per_frame": rays_frame,
                   "samples_per_ray": opts.samples_per_ray, "parallelism": f"rows{world}", "gather": drv.gather or "none",
                   **({"shared_gpu_test": True} if shared else {}),
                   "l2": ("inputs larger than L2 (hash table %.0f MB fp32, the kernel reads its %.0f MB "
                          "fp16 copy; L2 is 126 MB)" if field.grid_params.nbytes / 2 > 126e6
                          else "hash table %.0f MB fp32 / %.0f MB fp16 fits in L2 (no flush between frames)")
                         % (field.grid_params.nbytes / 1e6, field.grid_params.nbytes / 2e6),
                   "kernel": kname},
        "fps": round(fps, 3),
        # FrameStats of the timed frames (frame time = the slowest band's device ms, as
        # run_frame's wall time is the slowest worker's) through the native aggregate_stats
        "frame_stats": {k: round(getattr(fstats, k), 3) for k in ("mean_fps", "std_fps", "p99_fps")},
        "render_ms_per_step": round(kernel_ms / args.steps, 3),  # rank-0 march+render span
        "kernels": {"march_ms_per_launch": round(march_ms / max(render_launches, 1), 3),
                    f"{kname}_ms_per_launch": round(render_ms / max(render_launches, 1), 3),
                    "launches": render_launches,
                    "render_share_of_step": round(render_ms / max(elapsed, 1e-9), 4)},
        "work": {"evals_per_ray": round(evals / max(rays, 1), 3),
                 "active_levels_per_eval": round(level_samples / max(evals, 1), 3),
                 "candidates_tested_per_ray": round(candidates / max(rays, 1), 3)},
        "roofline": {"bound": "hbm", "achieved": None if achieved is None else round(achieved, 1),
                     "peak": hbm, "unit": "GB/s",
                     "frac": None if achieved is None else round(achieved / hbm, 4),
                     "traffic": ncu_traffic(kname, args.config),
                     "algorithmic": f"{bytes_per_ls} B per active (w_l>0) level-sample: 8 corners "
                                    f"x 2 features x {bytes_per_ls // 16} B "
                                    f"({'fp32 table' if dm.kernel == 'simt' else 'fp16 table copy'}); "
                                    f"{level_samples / max(world, 1):.3e} level-samples in "
                                    f"{render_launches} {kname} launches, {render_ms:.1f} ms "
                                    f"(CUDA events on the launch stream)"},
        "gather_isolated": gather_isolated(achieved, spec.table_log2),
        "roofline_mlp": {"bound": "tensor", "achieved": None if mlp_tflops is None else round(mlp_tflops, 2),
                         "peak": mlp_peak, "unit": "TFLOP/s",
                         "frac": None if mlp_tflops is None else round(mlp_tflops / mlp_peak, 4),
                         "algorithmic": "18,944 FLOP per evaluated sample (fp16 operands; "
                                        "peak = MEASURED_PEAKS bf16 sustained, the kernel runs "
                                        "inside a long step)"},
        "roofline_issue": issue_roofline(kname, args.config, render_ms / max(render_launches, 1),
                                         clocks.get("sm_mhz") or peaks.get("sm_max_mhz")),
        "clocks": clocks,
        "e2e": {"value": round(e2e, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "lumi_render_rows (C ABI) into pinned host buffers: the kernel stores the pixels over PCIe (zero-copy)" if world == 1 else
                        "StereoFrameDriver + D2H of the gathered frame"},
        "gpu_launches": launches,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
