"""ctypes binding of include/lumi_cuda.h (liblumi_cuda.so, built in-tree for sm_100a).

The library is required: there is no CPU fallback.  Loading fails loudly when the .so is
missing, and every entry point raises ``lumi.Error`` on a non-zero status.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LUMI_CUDA_LIB") or os.path.join(HERE, "lib", "liblumi_cuda.so")

LUMI_MAX_LEVELS = 16
LUMI_OK, LUMI_ERR_INVALID, LUMI_ERR_CUDA, LUMI_ERR_UNSUPPORTED = 0, 1, 2, 3
LUMI_KERNEL_TC, LUMI_KERNEL_SIMT, LUMI_KERNEL_PACKET, LUMI_KERNEL_WS = 0, 1, 2, 3


class Error(RuntimeError):
    """Mirror of lumi::Error (proj/include/lumi/common.h:61-70)."""

    def __init__(self, msg: str, code: int = LUMI_ERR_INVALID):
        super().__init__(msg)
        self.code = code


class FieldDesc(C.Structure):
    _fields_ = [("levels", C.c_int32), ("features_per_level", C.c_int32),
                ("base_resolution", C.c_int32), ("hidden_width", C.c_int32),
                ("per_level_scale", C.c_double), ("table_size", C.c_uint32),
                ("bottleneck", C.c_int32), ("color_space", C.c_int32), ("_pad", C.c_int32)]


class GridLayout(C.Structure):
    _fields_ = [("levels", C.c_int32), ("features_per_level", C.c_int32),
                ("resolution", C.c_int32 * LUMI_MAX_LEVELS),
                ("entries", C.c_uint32 * LUMI_MAX_LEVELS),
                ("dense", C.c_uint8 * LUMI_MAX_LEVELS),
                ("offset", C.c_uint64 * LUMI_MAX_LEVELS), ("total_floats", C.c_uint64),
                ("density_params", C.c_uint64), ("color_params", C.c_uint64)]


class CameraDesc(C.Structure):
    _fields_ = [("rot", C.c_double * 9), ("origin", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("t_near", C.c_double),
                ("t_far", C.c_double)]


class RenderOptionsDesc(C.Structure):
    _fields_ = [("samples_per_ray", C.c_int32), ("lod_enabled", C.c_int32),
                ("lod_bias", C.c_double), ("termination_transmittance", C.c_double),
                ("background", C.c_double * 3), ("contraction", C.c_int32),
                ("chunk_size", C.c_int32)]


class RowStatsDesc(C.Structure):
    _fields_ = [("row", C.c_int32), ("_pad", C.c_int32), ("ms", C.c_double),
                ("rays", C.c_int64), ("evals", C.c_int64)]


class FrameTarget(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("opacity", C.c_void_p),
                ("counts", C.c_void_p), ("row_evals", C.c_void_p), ("srgb8", C.c_void_p),
                ("work_stats", C.c_void_p), ("exposure_bias_stops", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32), ("row_offset", C.c_int32), ("_pad", C.c_int32),
                ("row_cycles", C.c_void_p)]


class CheckpointInfo(C.Structure):
    _fields_ = [("field", FieldDesc), ("samples_per_ray", C.c_int32), ("contraction", C.c_int32),
                ("background", C.c_double * 3), ("occ_res", C.c_int32), ("n_cameras", C.c_int32),
                ("table_floats", C.c_uint64), ("density_params", C.c_uint64),
                ("color_params", C.c_uint64)]


class LossConfig(C.Structure):
    _fields_ = [("lambda_depth", C.c_double), ("lambda_dvar", C.c_double),
                ("lambda_dist", C.c_double), ("inv_batch", C.c_double),
                ("depth_active", C.c_int32), ("_pad", C.c_int32)]


class LossTermsDesc(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("total", "image", "depth", "dvar", "dist")]


class TrainGrads(C.Structure):
    _fields_ = [("grid", C.c_void_p), ("density", C.c_void_p), ("color", C.c_void_p),
                ("alpha_v", C.c_void_p), ("loss", C.c_void_p)]


# (name, argtypes) of every exported entry point, in include/lumi_cuda.h order.
_vp, _i, _d, _u64, _f = C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_float
SIGNATURES = {
    "lumi_last_error": ([], C.c_char_p),
    "lumi_abi_version": ([], C.c_int),
    "lumi_device_info": ([_i, C.c_char_p, C.c_size_t], C.c_int),
    "lumi_field_layout": ([_vp, _vp], C.c_int),
    "lumi_synth_params": ([_vp, _u64, _d, _vp, _vp, _vp], C.c_int),
    "lumi_model_create": ([_i, _vp, _vp, _vp, _vp, _vp, _i, _vp], C.c_int),
    "lumi_model_set_occupancy": ([_vp, _vp, _i], C.c_int),
    "lumi_model_set_kernel": ([_vp, _i], C.c_int),
    "lumi_model_destroy": ([_vp], C.c_int),
    "lumi_model_bytes": ([_vp, _vp], C.c_int),
    "lumi_model_device": ([_vp, _vp], C.c_int),
    "lumi_model_set_timing": ([_vp, _i], C.c_int),
    "lumi_model_take_timing": ([_vp, _vp, _vp, _vp], C.c_int),
    "lumi_render_rows": ([_vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_render_rows_async": ([_vp, _vp, _vp, _i, _i, _vp, _vp], C.c_int),
    "lumi_march_kept_async": ([_vp, _vp, _vp, _i, _i, _vp, _vp, _vp], C.c_int),
    "lumi_encode_async": ([_vp, _i, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_gather_bench_async": ([_vp, _i, _i, _vp, _vp], C.c_int),
    "lumi_mlp_batch_async": ([_vp, _vp, _vp, _i, _vp, _vp], C.c_int),
    "lumi_checkpoint_read": ([C.c_char_p, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_checkpoint_write": ([C.c_char_p, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_bake_occupancy": ([_vp, _vp, _i, _i, _i, _i, _f, _vp, _vp], C.c_int),
    "lumi_train_backward_async": ([_vp, _vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp],
                                  C.c_int),
    "lumi_train_backward": ([_vp, _vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_model_device_params": ([_vp, _vp, _vp, _vp], C.c_int),
    "lumi_model_params_updated": ([_vp], C.c_int),
    "lumi_frame_driver_create": ([_vp, _i, _i, _i, _i, _d, _vp], C.c_int),
    "lumi_frame_driver_render": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_frame_driver_render_host": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "lumi_frame_driver_assignment": ([_vp, _vp, _vp], C.c_int),
    "lumi_frame_driver_set_assignment": ([_vp, _vp], C.c_int),
    "lumi_frame_driver_destroy": ([_vp], C.c_int),
    "lumi_ipc_export": ([_vp, _vp, _vp], C.c_int),
    "lumi_ipc_open": ([_i, _vp, _u64, _vp], C.c_int),
    "lumi_ipc_close": ([_i, _vp], C.c_int),
    "lumi_equal_assignment": ([_i, _i, _vp, _vp], C.c_int),
    "lumi_assign_rows": ([_i, _i, _vp, _vp, _d, _vp, _vp], C.c_int),
    "lumi_next_assignment": ([_i, _i, _vp, _vp, _vp, _i, _d, _vp, _vp], C.c_int),
    "lumi_aggregate_stats": ([_vp, _i, _vp, _vp, _vp], C.c_int),
}

_lib = None


def lib() -> C.CDLL:
    """Loads liblumi_cuda.so once; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Error(f"{LIB_PATH} is missing: build the CUDA extension first "
                        "(python -c 'import __graft_entry__ as g; g.build()')", LUMI_ERR_CUDA)
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:
                if os.environ.get("LUMI_CUDA_LIB"):  # an older build under A/B comparison
                    continue
                raise
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != LUMI_OK:
        msg = lib().lumi_last_error().decode(errors="replace")
        raise Error(msg or f"lumi error {rc}", rc)
