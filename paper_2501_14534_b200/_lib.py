"""ctypes binding of libtgs.so (include/tgs.h).

The product path has exactly one implementation: the CUDA library.  If the
shared object is missing or fails to load, every entry point raises
NativeLibraryError — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ContractViolationError, NativeLibraryError, raise_for_status

PKG = os.path.dirname(os.path.abspath(__file__))
# TGS_LIB: load another build of the library (A/B timing of kernel variants, profiles/)
LIB_PATH = os.environ.get("TGS_LIB") or os.path.join(PKG, "libtgs.so")

_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F = ctypes.c_float
_D = ctypes.c_double


class TgsCamera(ctypes.Structure):
    _fields_ = [("fx", _F), ("fy", _F), ("cx", _F), ("cy", _F), ("R", _F * 9), ("t", _F * 3), ("center", _F * 3),
                ("width", _I32), ("height", _I32), ("depth_row", _D * 4), ("fx64", _D), ("fy64", _D), ("cx64", _D),
                ("cy64", _D), ("R64", _D * 9), ("t64", _D * 3)]


class TgsSettings(ctypes.Structure):
    _fields_ = [("lowpass_s", _F), ("near_plane", _F), ("mask_logit_min", _F), ("sh_mask_logit_min", _F),
                ("opacity_logit_min", _F), ("background", _F * 3), ("active_sh_degree", _I32),
                ("tile_size", _I32), ("compute_sh_rest_grads", _I32), ("reserved", _I32), ("lowpass_s64", _D)]


CLOUD_FIELDS = ("positions", "log_scales", "rotations", "opacity_logits", "sh_dc", "sh_rest", "mask_logits",
                "sh_mask_logits")
GRAD_FIELDS = CLOUD_FIELDS + ("mean2d_screen",)


class TgsCloud(ctypes.Structure):
    _fields_ = [(f, _P) for f in CLOUD_FIELDS] + [("n", _I64)]


class TgsDensifyStats(ctypes.Structure):
    _fields_ = [("grad_accum", _P), ("grad_count", _P), ("area_max", _P)]


class TgsViewTarget(ctypes.Structure):
    _fields_ = [("tile_offsets", _P), ("sorted_ids", _P), ("ids_capacity", _I64), ("tile_order", _P),
                ("image", _P), ("transmit", _P), ("weight_sum", _P), ("n_contrib", _P), ("last_pos", _P),
                ("hits", _P), ("num_instances", _I64), ("row_begin", _I32), ("row_end", _I32)]


class TgsViewTrain(ctypes.Structure):
    _fields_ = [("target", _P), ("dimage", _P), ("terms", _P), ("dsplats", _P), ("loss_workspace", _P),
                ("target_ready", _P), ("exceptions", _P), ("exc_overflow", _P)]


class TgsGrads(ctypes.Structure):
    _fields_ = [(f, _P) for f in GRAD_FIELDS]


_SIGS = {
    "tgs_version": ([], _I32),
    "tgs_preprocess_forward": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "tgs_preprocess_forward_views": ([_P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "tgs_exact_records_views": ([_P, _P, _P, _I32, _P, _P, _P], _I32),
    "tgs_count_tiles": ([_P, _I64, _I32, _I32, _I32, _P, _P], _I32),
    "tgs_bin_gaussians_workspace": ([_I64, _P], _I32),
    "tgs_bin_gaussians": ([_P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P], _I32),
    "tgs_memcpy_d2h_async": ([_P, _P, _SZ, _P], _I32),
    "tgs_render_views_workspace": ([_I64, _I64, _I32, _I32, _I32, _P], _I32),
    "tgs_render_views": ([_P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P, _P, _P, _I32], _I32),
    "tgs_train_views": ([_P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _P, _SZ, _P, _P, _P, _I32], _I32),
    "tgs_bin_instances_workspace": ([_I64, _I64, _I32, _I32, _I32, _I32, _I32, _P], _I32),
    "tgs_row_histogram": ([_P, _P, _I64, _I32, _I32, _I32, _P, _P], _I32),
    "tgs_bin_instances": ([_P, _I64, _I32, _I32, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _P], _I32),
    "tgs_blend_forward": ([_P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "tgs_tile_order": ([_P, _I32, _P, _P], _I32),
    "tgs_debug_exact_pairs": ([_P, _I32], _I32),
    "tgs_blend_records": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "tgs_blend_backward_deterministic_workspace": ([_I64, _I64, _P], _I32),
    "tgs_blend_backward_deterministic": ([_P, _P, _P, _I64, _P, _P, _I64, _P, _P, _I32, _I32, _P, _P, _P, _P, _P,
                                          _P], _I32),
    "tgs_blend_backward": ([_P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "tgs_preprocess_backward": ([_P, _P, _P, _P, _P, _P, _I32, _P], _I32),
    "tgs_preprocess_backward_views": ([_P, _P, _P, _P, _P, _I32, _P, _I32, _P, _I32, _P], _I32),
    "tgs_loss_workspace": ([_I32, _I32, _P], _I32),
    "tgs_loss_l1_ssim": ([_P, _P, _I32, _I32, _F, _P, _P, _P, _P], _I32),
    "tgs_adam_step": ([_P, _P, _P, _P, _I64, _F, _F, _F, _F, _F, _F, _P], _I32),
    "tgs_adam_step_groups": ([_P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _F, _F, _F, _F, _F, _P, _I64, _P, _I32,
                              _P, _P, _P, _I32, _P], _I32),
    "tgs_gather_rows": ([_P, _P, _P, _I64, _I32, _P], _I32),
    "tgs_select_rows_workspace": ([_I64, _P], _I32),
    "tgs_select_rows": ([_P, _P, _F, _I64, _P, _P, _P, _SZ, _P], _I32),
    "tgs_significance_workspace": ([_I64, _P], _I32),
    "tgs_significance_scores": ([_P, _P, _F, _F, _I64, _P, _P, _P, _P, _SZ, _P], _I32),
    "tgs_significance_keep": ([_P, _I64, _I64, _P, _P, _SZ, _P], _I32),
    "tgs_area_resize": ([_P, _I32, _I32, _P, _I32, _I32, _P, _P], _I32),
    "tgs_gaussian_blur": ([_P, _I32, _I32, _I32, _F, _P, _P, _P], _I32),
}

_lib = None


def load():
    """Load libtgs.so once; raises NativeLibraryError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    import torch  # noqa: F401  (loads libcudart first so the library binds to the same runtime)
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover
        raise NativeLibraryError(f"failed to load {LIB_PATH}: {e}") from e
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    raise_for_status(int(getattr(load(), name)(*args)), name)


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None):
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def _logit(p: float) -> float:
    return float(np.log(p / (1.0 - p)))


def logit_floor_f32(eps: float) -> float:
    """Largest float32 <= logit(eps): sigmoid(m) > eps <=> m > this (masking.py:21-25)."""
    L = _logit(eps)
    f = np.float32(L)
    if float(f) > L:
        f = np.nextafter(f, np.float32(-np.inf))
    return float(f)


def logit_ceil_f32(p: float) -> float:
    """Smallest float32 >= logit(p): sigmoid(o) >= p <=> o >= this (rasterizer.py:178)."""
    L = _logit(p)
    f = np.float32(L)
    if float(f) < L:
        f = np.nextafter(f, np.float32(np.inf))
    return float(f)


_CAM_CACHE: dict = {}
_SET_CACHE: dict = {}


def make_camera(cam) -> TgsCamera:
    """tgs_camera for a camera; cached on the camera's VALUES (cameras are mutable, so
    the key is the pose and intrinsics themselves).  The struct is only read by C."""
    key = (float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), int(cam.width), int(cam.height),
           np.asarray(cam.R, dtype=np.float64).tobytes(), np.asarray(cam.t, dtype=np.float64).tobytes())
    c = _CAM_CACHE.get(key)
    if c is None:
        v = cam.native_fields() if hasattr(cam, "native_fields") else _native_fields(cam)
        R64 = np.asarray(cam.R, dtype=np.float64).reshape(9)
        t64 = np.asarray(cam.t, dtype=np.float64).reshape(3)
        c = TgsCamera(v["fx"], v["fy"], v["cx"], v["cy"], (_F * 9)(*v["R"]), (_F * 3)(*v["t"]),
                      (_F * 3)(*v["center"]), v["width"], v["height"], (_D * 4)(*v["depth_row"]), float(cam.fx),
                      float(cam.fy), float(cam.cx), float(cam.cy), (_D * 9)(*R64), (_D * 3)(*t64))
        if len(_CAM_CACHE) > 4096:
            _CAM_CACHE.clear()
        _CAM_CACHE[key] = c
    return c


def _native_fields(cam) -> dict:
    R = np.asarray(cam.R, dtype=np.float64).reshape(3, 3)
    t = np.asarray(cam.t, dtype=np.float64).reshape(3)
    f32 = lambda x: float(np.float32(x))  # noqa: E731
    return dict(fx=f32(cam.fx), fy=f32(cam.fy), cx=f32(cam.cx), cy=f32(cam.cy), R=[f32(x) for x in R.reshape(-1)],
                t=[f32(x) for x in t], center=[f32(x) for x in (-R.T @ t)], width=int(cam.width),
                height=int(cam.height), depth_row=[float(R[2, 0]), float(R[2, 1]), float(R[2, 2]), float(t[2])])


def make_settings(s) -> TgsSettings:
    """tgs_settings (validated like the reference); cached on the field values."""
    key = (s.lowpass_s, s.near, s.mask_threshold, s.sh_mask_threshold, tuple(s.background), s.active_sh_degree,
           s.tile_size, bool(s.compute_sh_rest_grads))
    c = _SET_CACHE.get(key)
    if c is None:
        c = _make_settings(s)
        if len(_SET_CACHE) > 1024:
            _SET_CACHE.clear()
        _SET_CACHE[key] = c
    return c


def _make_settings(s) -> TgsSettings:
    if not 0.0 < s.mask_threshold < 1.0 or not 0.0 < s.sh_mask_threshold < 1.0:
        raise ContractViolationError("mask threshold must lie in (0, 1)")  # masking.py:23-24
    if s.lowpass_s < 0:
        raise ContractViolationError("lowpass_s must be >= 0")  # geometry.py:150-151
    if not 0 <= int(s.active_sh_degree) <= 3:
        raise ContractViolationError("active_degree must be in 0..3")  # sh.py:147-148
    if int(s.tile_size) < 1:
        raise ContractViolationError("tile_size must be >= 1")  # rasterizer.py:103-104
    bg = [float(v) for v in s.background]
    return TgsSettings(float(s.lowpass_s), float(s.near), logit_floor_f32(s.mask_threshold),
                       logit_floor_f32(s.sh_mask_threshold), logit_ceil_f32(1.0 / 255.0), (_F * 3)(*bg),
                       int(s.active_sh_degree), int(s.tile_size), int(bool(s.compute_sh_rest_grads)), 0,
                       float(s.lowpass_s))
