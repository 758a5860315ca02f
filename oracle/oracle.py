"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU oracle.

Two interchangeable backends with one API:

* ``Oracle``    -- oracle/liblumi_oracle.so, the plain-C restatement of the reference
                   rendering path (oracle/lumi_oracle.c).
* ``Reference`` -- oracle/_ref/liblumi_ref.so, the UNMODIFIED reference library compiled
                   from its own sources (oracle/Makefile) behind oracle/ref_wrap.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  The product (paper_2311_02542_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblumi_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblumi_ref.so")

MLP_SCALAR, MLP_AVX2, MLP_AVX512 = 0, 1, 2
MAX_LEVELS = 32


class FieldConfig(C.Structure):
    """proj/include/lumi/grid.h:18-29 + field.h:22-27 (lo_field_config)."""

    _fields_ = [
        ("levels", C.c_int32),
        ("features_per_level", C.c_int32),
        ("base_resolution", C.c_int32),
        ("hidden_width", C.c_int32),
        ("per_level_scale", C.c_double),
        ("table_size", C.c_uint32),
        ("bottleneck", C.c_int32),
        ("color_space", C.c_int32),
        ("_pad", C.c_int32),
    ]


class GridLayout(C.Structure):
    _fields_ = [
        ("levels", C.c_int32),
        ("fpl", C.c_int32),
        ("resolution", C.c_int32 * MAX_LEVELS),
        ("entries", C.c_uint32 * MAX_LEVELS),
        ("dense", C.c_uint8 * MAX_LEVELS),
        ("offset", C.c_uint64 * MAX_LEVELS),
        ("total_floats", C.c_uint64),
    ]


class Camera(C.Structure):
    """proj/include/lumi/camera.h:15-23 (lo_camera)."""

    _fields_ = [
        ("rot", C.c_double * 9),
        ("origin", C.c_double * 3),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("t_near", C.c_double),
        ("t_far", C.c_double),
    ]


class RenderOptions(C.Structure):
    """proj/include/lumi/renderer.h:22-30 (lo_render_options)."""

    _fields_ = [
        ("samples_per_ray", C.c_int32),
        ("lod_enabled", C.c_int32),
        ("lod_bias", C.c_double),
        ("termination_transmittance", C.c_double),
        ("background", C.c_double * 3),
        ("contraction", C.c_int32),
        ("chunk_size", C.c_int32),
    ]


class Model(C.Structure):
    _fields_ = [
        ("cfg", FieldConfig),
        ("layout", GridLayout),
        ("table", C.c_void_p),
        ("dparams", C.c_void_p),
        ("cparams", C.c_void_p),
        ("occ", C.c_void_p),
        ("occ_res", C.c_int32),
        ("mlp_mode", C.c_int32),
    ]


class TrainRay(C.Structure):
    """proj/include/lumi/trainer.h:90-97 (lo_train_ray)."""

    _fields_ = [
        ("origin", C.c_double * 3),
        ("dir", C.c_double * 3),
        ("norigin", C.c_double * 3),
        ("ndir", C.c_double * 3),
        ("gt", C.c_float * 3),
        ("camera", C.c_int32),
        ("gt_depth", C.c_double),
        ("vignette_r", C.c_double),
    ]


class LossConfig(C.Structure):
    """The TrainConfig fields ray_loss reads (trainer.h:18-60) (lo_loss_config)."""

    _fields_ = [
        ("lambda_depth", C.c_double),
        ("lambda_dvar", C.c_double),
        ("lambda_dist", C.c_double),
        ("inv_batch", C.c_double),
        ("depth_active", C.c_int32),
        ("_pad", C.c_int32),
    ]


class LossTerms(C.Structure):
    """LossTerms (trainer.h:99-102), ray-dependent part."""

    _fields_ = [(k, C.c_double) for k in ("total", "image", "depth", "dvar", "dist")]


def loss_config(lambda_depth=0.1, lambda_dvar=0.01, lambda_dist=0.001, inv_batch=1.0,
                depth_active=True) -> LossConfig:
    return LossConfig(lambda_depth, lambda_dvar, lambda_dist, inv_batch,
                      1 if depth_active else 0, 0)


def field_config(levels=16, fpl=2, base=128, scale=1.4, table_size=1 << 19, hidden=64,
                 bottleneck=16, color_space=0) -> FieldConfig:
    return FieldConfig(levels, fpl, base, hidden, scale, table_size, bottleneck, color_space, 0)


def camera(rot, origin, fx, fy, cx, cy, width, height, t_near=0.05, t_far=10.0) -> Camera:
    c = Camera()
    c.rot[:] = [float(v) for v in rot]
    c.origin[:] = [float(v) for v in origin]
    c.fx, c.fy, c.cx, c.cy = fx, fy, cx, cy
    c.width, c.height = width, height
    c.t_near, c.t_far = t_near, t_far
    return c


def render_options(samples_per_ray=256, lod_enabled=True, lod_bias=0.0,
                   termination_transmittance=1e-4, background=(0.0, 0.0, 0.0), contraction=1,
                   chunk_size=32) -> RenderOptions:
    o = RenderOptions()
    o.samples_per_ray = samples_per_ray
    o.lod_enabled = 1 if lod_enabled else 0
    o.lod_bias = lod_bias
    o.termination_transmittance = termination_transmittance
    o.background[:] = [float(v) for v in background]
    o.contraction = contraction
    o.chunk_size = chunk_size
    return o


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Params:
    cfg: FieldConfig
    table: np.ndarray
    dparams: np.ndarray
    cparams: np.ndarray


def _bind_common(lib, pre):
    vp, i32, d, f = C.c_void_p, C.c_int, C.c_double, C.c_float
    lib.__getattr__(pre + "layout").argtypes = [vp, vp]
    lib.__getattr__(pre + "synth_params").argtypes = [vp, C.c_uint64, d, vp, vp, vp]


class Oracle:
    """The C restatement (oracle/lumi_oracle.c)."""

    name = "oracle"

    def __init__(self, path: str = ORACLE_SO, mlp_mode: int = MLP_AVX512):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.mlp_mode = mlp_mode
        L = self.lib
        vp, i32, d = C.c_void_p, C.c_int, C.c_double
        L.lo_layout.argtypes = [vp, vp]
        L.lo_density_param_count.argtypes = [vp]
        L.lo_density_param_count.restype = C.c_size_t
        L.lo_color_param_count.argtypes = [vp]
        L.lo_color_param_count.restype = C.c_size_t
        L.lo_synth_params.argtypes = [vp, C.c_uint64, d, vp, vp, vp]
        L.lo_generate_ray.argtypes = [vp, d, d, vp, vp]
        L.lo_contract.argtypes = [vp, i32, vp]
        L.lo_voxel_index.argtypes = [i32, vp]
        L.lo_voxel_index.restype = C.c_int64
        L.lo_lod_level.argtypes = [d, vp]
        L.lo_lod_level.restype = d
        L.lo_lod_weights.argtypes = [d, d, i32, vp]
        L.lo_sh_encode.argtypes = [vp, vp]
        L.lo_sample_distances.argtypes = [d, d, i32, vp, vp]
        for fn in ("lo_pq_encode", "lo_pq_decode", "lo_srgb_oetf"):
            getattr(L, fn).argtypes = [d]
            getattr(L, fn).restype = d
        L.lo_field_forward.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
        L.lo_render_rows.argtypes = [vp, vp, vp, i32, i32] + [vp] * 7 + [i32]
        L.lo_march_kept.argtypes = [vp, vp, vp, i32, i32, vp, vp, i32]
        L.lo_probe.argtypes = [vp, vp, i32, i32, i32, i32, vp, i32]
        L.lo_prune.argtypes = [vp, vp, vp, C.c_size_t, C.c_float, vp]
        L.lo_equal_assignment.argtypes = [i32, i32, vp, vp]
        L.lo_assign_rows.argtypes = [i32, i32, vp, vp, d, vp, vp]
        L.lo_next_assignment.argtypes = [i32, i32, vp, vp, vp, i32, d, vp, vp]
        L.lo_aggregate_stats.argtypes = [vp, i32, vp]
        L.lo_train_backward.argtypes = [vp, vp, vp, i32, vp, i32, vp, vp] + [vp] * 7
        L.lo_adam_step.argtypes = [C.c_size_t] + [vp] * 4 + [C.c_float] * 6

    # -- model -------------------------------------------------------------
    def layout(self, cfg: FieldConfig) -> GridLayout:
        lay = GridLayout()
        rc = self.lib.lo_layout(C.byref(cfg), C.byref(lay))
        if rc:
            raise ValueError(f"lo_layout failed ({rc})")
        return lay

    def param_counts(self, cfg):
        return (int(self.lib.lo_density_param_count(C.byref(cfg))),
                int(self.lib.lo_color_param_count(C.byref(cfg))))

    def synth_params(self, cfg: FieldConfig, seed: int, amp: float) -> Params:
        lay = self.layout(cfg)
        nd, nc = self.param_counts(cfg)
        table = np.empty(lay.total_floats, np.float32)
        dp = np.empty(nd, np.float32)
        cp = np.empty(nc, np.float32)
        rc = self.lib.lo_synth_params(C.byref(cfg), seed, amp, _p(table), _p(dp), _p(cp))
        if rc:
            raise ValueError(f"lo_synth_params failed ({rc})")
        return Params(cfg, table, dp, cp)

    def _model(self, params: Params, occ: np.ndarray, occ_res: int) -> Model:
        m = Model()
        m.cfg = params.cfg
        m.layout = self.layout(params.cfg)
        m.table, m.dparams, m.cparams = _p(params.table), _p(params.dparams), _p(params.cparams)
        m.occ = _p(occ)
        m.occ_res = occ_res
        m.mlp_mode = self.mlp_mode
        # keep numpy buffers alive with the struct
        m._keep = (params, occ)
        return m

    def model(self, params: Params, occ: np.ndarray, occ_res: int):
        occ = np.ascontiguousarray(occ, dtype=np.uint8)
        return self._model(params, occ, occ_res)

    # -- render ------------------------------------------------------------
    def render_rows(self, model, cam: Camera, opts: RenderOptions, b: int, e: int,
                    nthreads: int = os.cpu_count() or 1, stats: bool = True):
        W, H = cam.width, cam.height
        out = np.zeros((3, H, W), np.float32)
        depth = np.zeros((H, W), np.float32)
        opac = np.zeros((H, W), np.float32)
        ev = np.zeros((H, W), np.int32) if stats else None
        co = np.zeros((H, W), np.int32) if stats else None
        kp = np.zeros((H, W), np.int32) if stats else None
        rows = np.zeros(max(e - b, 1), np.int64)
        rc = self.lib.lo_render_rows(C.byref(model), C.byref(cam), C.byref(opts), b, e, _p(out),
                                     _p(depth), _p(opac), _p(ev), _p(co), _p(kp), _p(rows),
                                     nthreads)
        if rc:
            raise ValueError(f"lo_render_rows failed ({rc})")
        return dict(out=out, depth=depth, opacity=opac, evals=ev, contributing=co, kept=kp,
                    row_evals=rows[: e - b])

    def march_kept(self, model, cam, opts, b, e, nthreads: int = os.cpu_count() or 1):
        W, H = cam.width, cam.height
        words = (opts.samples_per_ray + 31) // 32
        mask = np.zeros((H, W, words), np.uint32)
        counts = np.zeros((H, W), np.int32)
        rc = self.lib.lo_march_kept(C.byref(model), C.byref(cam), C.byref(opts), b, e, _p(mask),
                                    _p(counts), nthreads)
        if rc:
            raise ValueError(f"lo_march_kept failed ({rc})")
        return mask, counts

    def field_forward(self, model, pos: np.ndarray, lodw: np.ndarray, sh=None):
        pos = np.ascontiguousarray(pos, np.float64)
        lodw = np.ascontiguousarray(lodw, np.float32)
        n = pos.shape[0]
        F = model.cfg.levels * model.cfg.features_per_level
        sigma = np.zeros(n, np.float32)
        color = np.zeros((3, n), np.float32) if sh is not None else None
        feat = np.zeros((F, n), np.float32)
        shp = None if sh is None else np.ascontiguousarray(sh, np.float32)
        self.lib.lo_field_forward(C.byref(model), n, _p(pos), _p(lodw), _p(shp), _p(sigma),
                                  _p(color), _p(feat))
        return sigma, color, feat

    def probe(self, model, cams, spp, k, res, nthreads=os.cpu_count() or 1):
        arr = (Camera * len(cams))(*cams)
        pm = np.zeros(res ** 3, np.float32)
        rc = self.lib.lo_probe(C.byref(model), arr, len(cams), spp, k, res, _p(pm), nthreads)
        if rc:
            raise ValueError("lo_probe failed")
        return pm

    def prune(self, probe_max, alpha):
        occ = np.zeros(probe_max.size, np.uint8)
        self.lib.lo_prune(_p(probe_max), None, None, probe_max.size, alpha, _p(occ))
        return occ

    # -- training reverse path -------------------------------------------------
    def _train_args(self, model, cam_tnf, alpha_v, rays, grads):
        cam_tnf = np.ascontiguousarray(cam_tnf, np.float64).reshape(-1, 2)
        alpha_v = np.ascontiguousarray(alpha_v, np.float64)
        nc = cam_tnf.shape[0]
        if isinstance(rays, np.ndarray):  # structured array with the lo_train_ray layout
            assert rays.dtype.itemsize == C.sizeof(TrainRay)
            rays = np.ascontiguousarray(rays)
            arr = rays.ctypes.data_as(C.c_void_p)
        else:
            arr = (TrainRay * len(rays))(*rays)
        if grads is None:
            lay = self.layout(model.cfg)
            nd, ncp = self.param_counts(model.cfg)
            grads = dict(grid=np.zeros(lay.total_floats, np.float32),
                         density=np.zeros(nd, np.float32), color=np.zeros(ncp, np.float32),
                         alpha=np.zeros(nc, np.float64))
        return cam_tnf, alpha_v, nc, arr, grads

    def train_backward(self, model, cam_tnf, alpha_v, rays, opts, lc, grads=None):
        """march_ray(record) + ray_loss + backward_ray per ray (trainer.cpp:549-561).
        Returns (grads dict, LossTerms, evals[n], contributing[n]); grads accumulate."""
        cam_tnf, alpha_v, nc, arr, grads = self._train_args(model, cam_tnf, alpha_v, rays, grads)
        loss = LossTerms()
        ev = np.zeros(len(rays), np.int32)
        co = np.zeros(len(rays), np.int32)
        rc = self.lib.lo_train_backward(C.byref(model), _p(cam_tnf), _p(alpha_v), nc, arr,
                                        len(rays), C.byref(opts), C.byref(lc), _p(grads["grid"]),
                                        _p(grads["density"]), _p(grads["color"]),
                                        _p(grads["alpha"]), C.byref(loss), _p(ev), _p(co))
        if rc:
            raise ValueError(f"lo_train_backward failed ({rc})")
        return grads, loss, ev, co

    def adam_step(self, p, g, m, v, lr, beta1, beta2, eps, c1, c2):
        self.lib.lo_adam_step(p.size, _p(p), _p(g), _p(m), _p(v), lr, beta1, beta2, eps, c1, c2)

    # -- scalar helpers ------------------------------------------------------
    def generate_ray(self, cam, px, py):
        o = np.zeros(3)
        d = np.zeros(3)
        self.lib.lo_generate_ray(C.byref(cam), px, py, _p(o), _p(d))
        return o, d

    def contract(self, x, mode=1):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(3)
        rc = self.lib.lo_contract(_p(x), mode, _p(out))
        if rc:
            raise ValueError("contract: non-finite input")
        return out

    def voxel_index(self, res, c):
        c = np.ascontiguousarray(c, np.float64)
        return int(self.lib.lo_voxel_index(res, _p(c)))

    def lod_level(self, r, cfg):
        return float(self.lib.lo_lod_level(r, C.byref(cfg)))

    def lod_weights(self, l_star, bias, levels):
        w = np.zeros(levels, np.float32)
        self.lib.lo_lod_weights(l_star, bias, levels, _p(w))
        return w

    def sh_encode(self, d):
        d = np.ascontiguousarray(d, np.float64)
        out = np.zeros(16, np.float32)
        self.lib.lo_sh_encode(_p(d), _p(out))
        return out

    def sample_distances(self, t_near, t_far, n):
        ts = np.zeros(n)
        ratio = C.c_double()
        self.lib.lo_sample_distances(t_near, t_far, n, _p(ts), C.byref(ratio))
        return ts, ratio.value

    def pq_encode(self, y):
        return float(self.lib.lo_pq_encode(y))

    def pq_decode(self, v):
        return float(self.lib.lo_pq_decode(v))

    def srgb_oetf(self, v):
        return float(self.lib.lo_srgb_oetf(v))

    # -- scheduler -----------------------------------------------------------
    def equal_assignment(self, height, workers):
        rows = np.zeros(workers, np.int32)
        shares = np.zeros(workers)
        rc = self.lib.lo_equal_assignment(height, workers, _p(rows), _p(shares))
        if rc:
            raise ValueError("equal_assignment: bad arguments")
        return rows, shares

    def assign_rows(self, height, throughputs, prev_shares, prev_rows, damp):
        n = len(throughputs)
        tp = np.ascontiguousarray(throughputs, np.float64)
        ps = np.ascontiguousarray(prev_shares, np.float64)
        rows = np.zeros(n, np.int32)
        shares = np.zeros(n)
        rc = self.lib.lo_assign_rows(height, n, _p(tp), _p(ps), damp, _p(rows), _p(shares))
        if rc:
            raise ValueError("assign_rows: bad arguments")
        return rows, shares

    def aggregate_stats(self, ms):
        ms = np.ascontiguousarray(ms, np.float64)
        out = np.zeros(3)
        rc = self.lib.lo_aggregate_stats(_p(ms), ms.size, _p(out))
        if rc:
            raise ValueError("aggregate_stats: no frames")
        return out


class Reference(Oracle):
    """The unmodified reference compiled from its sources (oracle/_ref/liblumi_ref.so)."""

    name = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        self.lib = C.CDLL(path)
        L = self.lib
        vp, i32, d = C.c_void_p, C.c_int, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_simd_name.restype = C.c_char_p
        L.ref_layout.argtypes = [vp, vp]
        L.ref_synth_params.argtypes = [vp, C.c_uint64, d, vp, vp, vp]
        L.ref_model_create.argtypes = [vp, vp, vp, vp, vp, i32]
        L.ref_model_create.restype = vp
        L.ref_model_destroy.argtypes = [vp]
        L.ref_render_rows.argtypes = [vp, vp, vp, i32, i32] + [vp] * 7
        L.ref_render_rows_plain.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.ref_run_frame.argtypes = [vp, vp, vp, i32, i32, i32, vp, vp]
        L.ref_march_kept.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.ref_field_forward.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
        L.ref_probe_prune.argtypes = [vp, vp, i32, i32, i32, i32, C.c_float, vp, vp]
        L.ref_generate_ray.argtypes = [vp, d, d, vp, vp]
        L.ref_contract.argtypes = [vp, i32, vp]
        L.ref_lod_level.argtypes = [d, vp]
        L.ref_lod_level.restype = d
        L.ref_lod_weights.argtypes = [d, d, i32, vp]
        L.ref_sh_encode.argtypes = [vp, vp]
        for fn in ("ref_pq_encode", "ref_pq_decode", "ref_srgb_oetf"):
            getattr(L, fn).argtypes = [d]
            getattr(L, fn).restype = d
        L.ref_save_checkpoint.argtypes = [vp, C.c_char_p, i32, vp, i32]
        L.ref_write_pfm.argtypes = [C.c_char_p, vp, i32, i32, i32]
        L.ref_equal_assignment.argtypes = [i32, i32, vp, vp]
        L.ref_assign_rows.argtypes = [i32, i32, vp, vp, vp, d, vp, vp]
        L.ref_aggregate_stats.argtypes = [vp, i32, vp]
        L.ref_train_backward.argtypes = [vp, vp, vp, i32, vp, i32, vp, vp] + [vp] * 7
        L.ref_adam_step.argtypes = [C.c_size_t] + [vp] * 4 + [C.c_float] * 6

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def simd_name(self) -> str:
        return self.lib.ref_simd_name().decode()

    def mlp_mode_equivalent(self) -> int:
        return {"scalar": MLP_SCALAR, "avx2": MLP_AVX2, "avx512": MLP_AVX512}[self.simd_name()]

    def layout(self, cfg):
        lay = GridLayout()
        self._check(self.lib.ref_layout(C.byref(cfg), C.byref(lay)))
        return lay

    def param_counts(self, cfg):
        return Oracle.param_counts(_ORACLE_FOR_COUNTS(), cfg)

    def synth_params(self, cfg, seed, amp):
        lay = self.layout(cfg)
        nd, nc = self.param_counts(cfg)
        table = np.empty(lay.total_floats, np.float32)
        dp = np.empty(nd, np.float32)
        cp = np.empty(nc, np.float32)
        self._check(self.lib.ref_synth_params(C.byref(cfg), seed, amp, _p(table), _p(dp), _p(cp)))
        return Params(cfg, table, dp, cp)

    def model(self, params, occ, occ_res):
        occ = np.ascontiguousarray(occ, dtype=np.uint8)
        h = self.lib.ref_model_create(C.byref(params.cfg), _p(params.table), _p(params.dparams),
                                      _p(params.cparams), _p(occ), occ_res)
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return _RefHandle(self.lib, h, params.cfg)

    def render_rows(self, model, cam, opts, b, e, nthreads=1, stats=True):
        W, H = cam.width, cam.height
        out = np.zeros((3, H, W), np.float32)
        depth = np.zeros((H, W), np.float32)
        opac = np.zeros((H, W), np.float32)
        ev = np.zeros((H, W), np.int32)
        co = np.zeros((H, W), np.int32)
        kp = np.zeros((H, W), np.int32)
        rows = np.zeros(max(e - b, 1), np.int64)
        self._check(self.lib.ref_render_rows(model.h, C.byref(cam), C.byref(opts), b, e, _p(out),
                                             _p(depth), _p(opac), _p(ev), _p(co), _p(kp),
                                             _p(rows)))
        return dict(out=out, depth=depth, opacity=opac, evals=ev, contributing=co, kept=kp,
                    row_evals=rows[: e - b])

    def run_frame(self, model, cam, opts, b, e, workers, want_image=False):
        W, H = cam.width, cam.height
        out = np.zeros((3, H, W), np.float32) if want_image else None
        ms = C.c_double()
        self._check(self.lib.ref_run_frame(model.h, C.byref(cam), C.byref(opts), b, e, workers,
                                           _p(out), C.byref(ms)))
        return ms.value, out

    def march_kept(self, model, cam, opts, b, e, nthreads=1):
        W, H = cam.width, cam.height
        words = (opts.samples_per_ray + 31) // 32
        mask = np.zeros((H, W, words), np.uint32)
        counts = np.zeros((H, W), np.int32)
        self._check(self.lib.ref_march_kept(model.h, C.byref(cam), C.byref(opts), b, e, _p(mask),
                                            _p(counts)))
        return mask, counts

    def field_forward(self, model, pos, lodw, sh=None):
        pos = np.ascontiguousarray(pos, np.float64)
        lodw = np.ascontiguousarray(lodw, np.float32)
        n = pos.shape[0]
        F = model.cfg.levels * model.cfg.features_per_level
        sigma = np.zeros(n, np.float32)
        color = np.zeros((3, n), np.float32) if sh is not None else None
        feat = np.zeros((F, n), np.float32)
        shp = None if sh is None else np.ascontiguousarray(sh, np.float32)
        self._check(self.lib.ref_field_forward(model.h, n, _p(pos), _p(lodw), _p(shp), _p(sigma),
                                               _p(color), _p(feat)))
        return sigma, color, feat

    def probe_prune(self, model, cams, spp, k, res, alpha):
        arr = (Camera * len(cams))(*cams)
        pm = np.zeros(res ** 3, np.float32)
        occ = np.zeros(res ** 3, np.uint8)
        self._check(self.lib.ref_probe_prune(model.h, arr, len(cams), spp, k, res, alpha, _p(pm),
                                             _p(occ)))
        return pm, occ

    def write_pfm(self, path, planar):
        """The reference write_pfm (image.cpp:20-35) of a float32 [C, H, W] image."""
        a = np.ascontiguousarray(planar, np.float32)
        c, h, w = a.shape
        self._check(self.lib.ref_write_pfm(str(path).encode(), _p(a), w, h, c))

    def save_checkpoint(self, model, path, spp=256, background=(0.0, 0.0, 0.0), contraction=1):
        """The reference save_checkpoint (scene.cpp:320-351) of a model."""
        bg = np.ascontiguousarray(background, np.float64)
        self._check(self.lib.ref_save_checkpoint(model.h, str(path).encode(), spp, _p(bg),
                                                 contraction))

    def train_backward(self, model, cam_tnf, alpha_v, rays, opts, lc, grads=None):
        cam_tnf, alpha_v, nc, arr, grads = self._train_args(model, cam_tnf, alpha_v, rays, grads)
        loss = LossTerms()
        ev = np.zeros(len(rays), np.int32)
        co = np.zeros(len(rays), np.int32)
        self._check(self.lib.ref_train_backward(model.h, _p(cam_tnf), _p(alpha_v), nc, arr,
                                                len(rays), C.byref(opts), C.byref(lc),
                                                _p(grads["grid"]), _p(grads["density"]),
                                                _p(grads["color"]), _p(grads["alpha"]),
                                                C.byref(loss), _p(ev), _p(co)))
        return grads, loss, ev, co

    def adam_step(self, p, g, m, v, lr, beta1, beta2, eps, c1, c2):
        self.lib.ref_adam_step(p.size, _p(p), _p(g), _p(m), _p(v), lr, beta1, beta2, eps, c1, c2)

    def generate_ray(self, cam, px, py):
        o = np.zeros(3)
        d = np.zeros(3)
        self.lib.ref_generate_ray(C.byref(cam), px, py, _p(o), _p(d))
        return o, d

    def contract(self, x, mode=1):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(3)
        self.lib.ref_contract(_p(x), mode, _p(out))
        return out

    def lod_level(self, r, cfg):
        return float(self.lib.ref_lod_level(r, C.byref(cfg)))

    def lod_weights(self, l_star, bias, levels):
        w = np.zeros(levels, np.float32)
        self.lib.ref_lod_weights(l_star, bias, levels, _p(w))
        return w

    def sh_encode(self, d):
        d = np.ascontiguousarray(d, np.float64)
        out = np.zeros(16, np.float32)
        self.lib.ref_sh_encode(_p(d), _p(out))
        return out

    def pq_encode(self, y):
        return float(self.lib.ref_pq_encode(y))

    def pq_decode(self, v):
        return float(self.lib.ref_pq_decode(v))

    def srgb_oetf(self, v):
        return float(self.lib.ref_srgb_oetf(v))

    def equal_assignment(self, height, workers):
        rows = np.zeros(workers, np.int32)
        shares = np.zeros(workers)
        self._check(self.lib.ref_equal_assignment(height, workers, _p(rows), _p(shares)))
        return rows, shares

    def assign_rows(self, height, throughputs, prev_shares, prev_rows, damp):
        n = len(throughputs)
        tp = np.ascontiguousarray(throughputs, np.float64)
        ps = np.ascontiguousarray(prev_shares, np.float64)
        pr = np.ascontiguousarray(prev_rows, np.int32)
        rows = np.zeros(n, np.int32)
        shares = np.zeros(n)
        self._check(self.lib.ref_assign_rows(height, n, _p(tp), _p(ps), _p(pr), damp, _p(rows),
                                             _p(shares)))
        return rows, shares

    def aggregate_stats(self, ms):
        ms = np.ascontiguousarray(ms, np.float64)
        out = np.zeros(3)
        self._check(self.lib.ref_aggregate_stats(_p(ms), ms.size, _p(out)))
        return out


class _RefHandle:
    def __init__(self, lib, h, cfg):
        self.lib, self.h, self.cfg = lib, h, cfg

    def __del__(self):
        try:
            self.lib.ref_model_destroy(self.h)
        except Exception:
            pass


_oracle_singleton = None


def _ORACLE_FOR_COUNTS():
    global _oracle_singleton
    if _oracle_singleton is None:
        _oracle_singleton = Oracle()
    return _oracle_singleton


def reference_available() -> bool:
    return os.path.exists(REF_SO)
