"""ctypes mirror of include/prenom/prenom_gpu.h (the C-ABI drop-in boundary).

Only struct layouts and the loader live here; the reference-shaped Python API
is in :mod:`paper_2503_01582_b200.trainer`.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "_lib" / "libprenom_b200.so"

PRENOM_OK, PRENOM_USAGE, PRENOM_DATA, PRENOM_NUMERIC, PRENOM_CUDA = range(5)
TAG_FRAME, TAG_PIXEL, TAG_FINE, TAG_BG, TAG_RENDER, TAG_INIT, TAG_SYNTH = 1, 2, 3, 4, 5, 6, 7
ACT_EXP_CLAMPED, ACT_SOFTPLUS = 0, 1
MLP_FP32, MLP_BF16, MLP_BF16X3 = 0, 1, 2
DEBUG_TILE_FP32 = 3
COMM_ID_BYTES = 128  # prenom_debug_field_eval: the fp32 SIMT train-path tile forward
KERNEL_CLASSES = ["sample", "field_fwd", "composite", "mlp_bwd", "encode_bwd", "adam", "refresh"]


class FieldArchC(C.Structure):
    """prenom_field_arch (mirrors noma::FieldArch, field.hpp:20-31)."""

    _fields_ = [
        ("hash_levels", C.c_int32),
        ("features_per_level", C.c_int32),
        ("log2_table_size", C.c_int32),
        ("base_resolution", C.c_int32),
        ("per_level_scale", C.c_float),
        ("hidden_width", C.c_int32),
        ("hidden_layers", C.c_int32),
        ("density_activation", C.c_int32),
    ]


class BoxC(C.Structure):
    """prenom_box: an axis-aligned box of a synthetic scene with its albedo."""

    _fields_ = [("lo", C.c_float * 3), ("hi", C.c_float * 3), ("albedo", C.c_float * 3)]


class CameraC(C.Structure):
    """prenom_camera (mirrors noma::Camera, render.hpp:13-23)."""

    _fields_ = [
        ("fx", C.c_float),
        ("fy", C.c_float),
        ("cx", C.c_float),
        ("cy", C.c_float),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("R", C.c_float * 9),
        ("t", C.c_float * 3),
    ]


class PoseC(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class TrainCfgC(C.Structure):
    """prenom_train_cfg (MapperConfig / InnerOptions / LossWeights hot keys)."""

    _fields_ = [
        ("rays_per_iter", C.c_int32),
        ("bg_fraction", C.c_float),
        ("samples_per_ray", C.c_int32),
        ("lambda_d", C.c_float),
        ("lambda_sigma", C.c_float),
        ("coarse_samples", C.c_int32),
        ("escape_eps", C.c_float),
        ("grid_refresh_every", C.c_int32),
        ("eta", C.c_float),
        ("prior_sampling", C.c_int32),
        ("band_px", C.c_int32),
        ("mlp_precision", C.c_int32),
        ("adam_beta1", C.c_float),
        ("adam_beta2", C.c_float),
        ("adam_eps", C.c_float),
    ]


class StepStatsC(C.Structure):
    _fields_ = [
        ("total", C.c_double),
        ("color_term", C.c_double),
        ("depth_term", C.c_double),
        ("sigma_term", C.c_double),
        ("n_samples", C.c_int64),
        ("n_rays_escaped", C.c_int32),
        ("frame_index", C.c_int32),
    ]


def fptr(a):
    """float* view of a contiguous float32 numpy array (or None)."""
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(C.POINTER(C.c_float))


def dptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def u8ptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def u32ptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


# Every symbol include/prenom/prenom_gpu.h declares (checked by tests).
EXPORTED = [
    "prenom_last_error", "prenom_abi_version", "prenom_default_train_cfg",
    "prenom_param_count", "prenom_level_resolution",
    "prenom_ctx_create", "prenom_ctx_destroy", "prenom_ctx_stream", "prenom_ctx_synchronize",
    "prenom_ctx_launch_count", "prenom_ctx_profile", "prenom_ctx_kernel_times", "prenom_object_next_frame",
    "prenom_object_create", "prenom_object_destroy", "prenom_object_set_frames",
    "prenom_object_upload_frame", "prenom_object_synth_frames", "prenom_object_get_frame", "prenom_train_step", "prenom_object_last_stats",
    "prenom_train_step_async", "prenom_wait_stats", "prenom_object_frame_at",
    "prenom_object_step", "prenom_object_check",
    "prenom_render", "prenom_density_query", "prenom_extract_mesh", "prenom_get_mesh", "prenom_get_mesh_grid", "prenom_nearest_sq", "prenom_field_eval",
    "prenom_get_params", "prenom_set_params", "prenom_get_grid", "prenom_set_grid",
    "prenom_get_adam", "prenom_reset_adam", "prenom_set_adam", "prenom_train_step_many", "prenom_ctx_set_grouping",
    "prenom_reptile_delta", "prenom_reptile_apply", "prenom_object_copy_params", "prenom_reptile_update",
    "prenom_object_set_seed",
    "prenom_comm_unique_id", "prenom_ctx_init_comm", "prenom_ctx_comm_info", "prenom_reptile_step",
    "prenom_debug_philox", "prenom_debug_hash_encode", "prenom_debug_field_eval",
    "prenom_debug_field_backward", "prenom_debug_adam", "prenom_debug_sample_rays",
    "prenom_debug_batch_loss", "prenom_debug_generate_rays", "prenom_debug_umma_gemm",
    "prenom_debug_marching_cubes", "prenom_debug_mesh_get", "prenom_mc_case_triangles",
    "prenom_debug_bwd_trace", "prenom_debug_l2_read",
]

_lib = None


def load():
    """Load the in-tree CUDA library. Fails loudly when it is missing: there is
    no CPU fallback for the product path."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PRENOM_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise RuntimeError(
            f"libprenom_b200.so not found at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(path)
    _declare(lib)
    _lib = lib
    return lib


def _declare(lib):
    P = C.c_void_p
    i32, i64, u64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
    f32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_double)
    i32p, i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    u8p, u32p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)
    archp = C.POINTER(FieldArchC)
    sigs = {
        "prenom_last_error": (C.c_char_p, []),
        "prenom_abi_version": (i32, []),
        "prenom_default_train_cfg": (None, [C.POINTER(TrainCfgC)]),
        "prenom_param_count": (i32, [archp, C.POINTER(sz), C.POINTER(sz)]),
        "prenom_level_resolution": (i32, [archp, i32, i32p]),
        "prenom_ctx_create": (i32, [i32, C.POINTER(P)]),
        "prenom_ctx_destroy": (i32, [P]),
        "prenom_ctx_stream": (i32, [P, C.POINTER(P)]),
        "prenom_ctx_synchronize": (i32, [P]),
        "prenom_ctx_launch_count": (i32, [P, i64p]),
        "prenom_ctx_profile": (i32, [P, i32]),
        "prenom_ctx_kernel_times": (i32, [P, f64p, i64p]),
        "prenom_object_next_frame": (i32, [P, i32p]),
        "prenom_object_create": (i32, [P, archp, f32p, f32p, i32, u64, C.POINTER(TrainCfgC),
                                       f32p, f32p, C.POINTER(P)]),
        "prenom_object_destroy": (i32, [P]),
        "prenom_object_set_frames": (i32, [P, i32, C.POINTER(CameraC), f32p, f32p, u8p,
                                           C.c_uint8, C.POINTER(PoseC)]),
        "prenom_object_upload_frame": (i32, [P, i32, f32p, f32p, u8p]),
        "prenom_object_synth_frames": (i32, [P, i32, C.POINTER(CameraC), i32, C.POINTER(BoxC), C.c_float,
                                             C.c_float, u64, C.POINTER(PoseC)]),
        "prenom_object_get_frame": (i32, [P, i32, f32p, f32p, i32p, i32p, i32p, i32p]),
        "prenom_train_step": (i32, [P, i32, C.POINTER(StepStatsC)]),
        "prenom_object_last_stats": (i32, [P, i32, C.POINTER(StepStatsC)]),
        "prenom_train_step_async": (i32, [P, i32, i32, C.POINTER(C.c_uint64)]),
        "prenom_wait_stats": (i32, [P, C.c_uint64, C.POINTER(StepStatsC)]),
        "prenom_object_frame_at": (i32, [P, C.c_int64, i32p]),
        "prenom_object_step": (i32, [P, i64p]),
        "prenom_object_check": (i32, [P]),
        "prenom_render": (i32, [P, i32, f32p, f32p, f32p, f32p]),
        "prenom_density_query": (i32, [P, i32, f32p, i32]),
        "prenom_extract_mesh": (i32, [P, i32, C.c_float, C.c_float, f32p, i64p, i64p]),
        "prenom_get_mesh": (i32, [P, f32p, i32p]),
        "prenom_get_mesh_grid": (i32, [P, i32p, f32p]),
        "prenom_nearest_sq": (i32, [P, i32, f32p, i32, f32p, f32p]),
        "prenom_field_eval": (i32, [P, i32, f32p, f32p, f32p]),
        "prenom_get_params": (i32, [P, f32p]),
        "prenom_set_params": (i32, [P, f32p]),
        "prenom_get_grid": (i32, [P, i32p, f32p]),
        "prenom_set_grid": (i32, [P, i32, f32p]),
        "prenom_get_adam": (i32, [P, f32p, f32p, i64p]),
        "prenom_reset_adam": (i32, [P]),
        "prenom_set_adam": (i32, [P, f32p, f32p, C.c_int64]),
        "prenom_train_step_many": (i32, [C.POINTER(P), i32, i32]),
        "prenom_ctx_set_grouping": (i32, [P, i32]),
        "prenom_reptile_delta": (i32, [P, P, C.c_void_p]),
        "prenom_reptile_apply": (i32, [P, C.c_void_p, i32, C.c_float]),
        "prenom_object_copy_params": (i32, [P, P]),
        "prenom_reptile_update": (i32, [P, P, C.c_float]),
        "prenom_object_set_seed": (i32, [P, u64]),
        "prenom_comm_unique_id": (i32, [u8p]),
        "prenom_ctx_init_comm": (i32, [P, i32, i32, u8p]),
        "prenom_ctx_comm_info": (i32, [P, i32p, i32p, i32p]),
        "prenom_reptile_step": (i32, [P, C.POINTER(P), i32, i32, C.c_float]),
        "prenom_debug_philox": (i32, [P, i32, u32p, u32p]),
        "prenom_debug_hash_encode": (i32, [P, archp, f32p, i32, f32p, f32p]),
        "prenom_debug_field_eval": (i32, [P, archp, f32p, i32, f32p, f32p, f32p, f32p, i32]),
        "prenom_debug_field_backward": (i32, [P, archp, f32p, i32, f32p, f32p, f32p, f32p, i32]),
        "prenom_debug_adam": (i32, [P, sz, f32p, f32p, f32p, f32p, i64p, C.c_float, C.c_float,
                                    C.c_float, C.c_float]),
        "prenom_debug_sample_rays": (i32, [P, i32, f32p, f32p, f32p, f32p, i32, i32, f32p, i32,
                                           i32, C.c_float, u64, i64, f32p, f32p, f32p, i32p,
                                           f32p, f32p]),
        "prenom_debug_batch_loss": (i32, [P, i32, i32, i32p, f32p, f32p, i32p, f32p, f32p, f32p,
                                          f32p, f32p, C.c_float, C.c_float, f64p, f32p, f32p,
                                          f32p, f32p]),
        "prenom_debug_generate_rays": (i32, [P, i32, i64, f32p, f32p, i32p, f32p, f32p, i32p]),
        "prenom_debug_umma_gemm": (i32, [P, i32, i32, i32, i32, i32, f32p, f32p, f32p]),
        "prenom_debug_marching_cubes": (i32, [P, i32, f32p, C.c_float, i64p, i64p]),
        "prenom_debug_mesh_get": (i32, [P, f32p, i32p]),
        "prenom_mc_case_triangles": (i32, [i32, i32p]),
        "prenom_debug_bwd_trace": (i32, [P, i64p, i64p, i64p]),
        "prenom_debug_l2_read": (i32, [P, i32, i32, C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
