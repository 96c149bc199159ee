"""ctypes front end of liboracle.so — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
`--impl reference` legs may import this module; the product package never does
(tests/test_boundary.py checks that).  It restates the reference pipeline
(`slimsplat.rasterizer.render_forward` / `render_backward`,
rasterizer.py:215-419) on the CPU with numpy buffers:

    dtype="f64": the reference's float64 arithmetic (pinned to golden vectors of
                 the reference itself, tests/test_oracle_golden.py)
    dtype="f32": the float32 semantics the CUDA path reproduces bit-exactly for
                 visibility, radii, tile counts and sorted tile lists.

Inputs are duck-typed: any camera with fx, fy, cx, cy, R, t, width, height and
any settings object with the RenderSettings attribute names work (the
reference's own classes included).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
FIELDS = ("positions", "log_scales", "rotations", "opacity_logits", "sh_dc", "sh_rest", "mask_logits", "sh_mask_logits")

_P = ctypes.c_void_p


class _Camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3), ("center", ctypes.c_double * 3),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class _Settings(ctypes.Structure):
    _fields_ = [("lowpass_s", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("mask_threshold", ctypes.c_double), ("sh_mask_threshold", ctypes.c_double),
                ("mask_logit_min", ctypes.c_double), ("sh_mask_logit_min", ctypes.c_double),
                ("opacity_logit_min", ctypes.c_double), ("background", ctypes.c_double * 3),
                ("active_sh_degree", ctypes.c_int32), ("tile_size", ctypes.c_int32),
                ("compute_sh_rest_grads", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _Cloud(ctypes.Structure):
    _fields_ = [(f, _P) for f in FIELDS] + [("n", ctypes.c_int64)]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.cpp")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB_PATH)
        i64 = ctypes.c_int64
        _lib.oracle_bin_f64.restype = i64
        _lib.oracle_bin_f32.restype = i64
        _lib.oracle_sem_expf.restype = ctypes.c_float
        _lib.oracle_sem_expf.argtypes = [ctypes.c_float]
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def logit_floor_f32(eps: float) -> float:
    """Largest float32 <= logit(eps): sigmoid(m) > eps  <=>  m > this (m float32)."""
    L = math.log(eps / (1.0 - eps))
    f = np.float32(L)
    if float(f) > L:
        f = np.nextafter(f, np.float32(-np.inf))
    return float(f)


def logit_ceil_f32(p: float) -> float:
    """Smallest float32 >= logit(p): sigmoid(o) >= p  <=>  o >= this (o float32)."""
    L = math.log(p / (1.0 - p))
    f = np.float32(L)
    if float(f) < L:
        f = np.nextafter(f, np.float32(np.inf))
    return float(f)


def _camera(cam) -> _Camera:
    R = np.asarray(cam.R, dtype=np.float64).reshape(9)
    t = np.asarray(cam.t, dtype=np.float64).reshape(3)
    c = -np.asarray(cam.R, dtype=np.float64).reshape(3, 3).T @ t
    return _Camera(cam.fx, cam.fy, cam.cx, cam.cy, (ctypes.c_double * 9)(*R), (ctypes.c_double * 3)(*t),
                   (ctypes.c_double * 3)(*c), int(cam.width), int(cam.height))


def default_settings(**kw):
    s = dict(lowpass_s=0.3, active_sh_degree=3, background=(0.0, 0.0, 0.0), tile_size=16, near=0.01,
             record_hits=False, mask_threshold=0.05, sh_mask_threshold=0.1, compute_sh_rest_grads=True)
    s.update(kw)
    return SimpleNamespace(**s)


def _settings(s) -> _Settings:
    bg = tuple(float(v) for v in s.background)
    return _Settings(float(s.lowpass_s), float(s.near), float(s.mask_threshold), float(s.sh_mask_threshold),
                     logit_floor_f32(s.mask_threshold), logit_floor_f32(s.sh_mask_threshold),
                     logit_ceil_f32(1.0 / 255.0), (ctypes.c_double * 3)(*bg), int(s.active_sh_degree),
                     int(s.tile_size), int(bool(s.compute_sh_rest_grads)), 0)


class _CloudHold:
    """Keeps float64 copies alive for the duration of a call."""

    def __init__(self, fields: dict):
        self.arrays = {f: np.ascontiguousarray(np.asarray(fields[f], dtype=np.float64)) for f in FIELDS}
        self.n = int(self.arrays["positions"].shape[0])
        self.c = _Cloud(*[_ptr(self.arrays[f]) for f in FIELDS], self.n)


def _fields_of(cloud) -> dict:
    if isinstance(cloud, dict):
        return cloud
    return {f: np.asarray(getattr(cloud, f) if not hasattr(getattr(cloud, f), "cpu") else getattr(cloud, f).cpu())
            for f in FIELDS}


def _rt(dtype):
    return (np.float64, "f64") if dtype == "f64" else (np.float32, "f32")


def preprocess(cloud, cam, settings, dtype="f64"):
    npt, sfx = _rt(dtype)
    hold = _CloudHold(_fields_of(cloud))
    n = hold.n
    splats = np.zeros((n, 12), dtype=npt)
    visible = np.zeros(n, dtype=np.uint8)
    tiles = np.zeros(n, dtype=np.int32)
    depth_key = np.zeros(n, dtype=np.float64)
    cc, ss = _camera(cam), _settings(settings)
    rc = getattr(lib(), f"oracle_preprocess_{sfx}")(ctypes.byref(hold.c), ctypes.byref(cc), ctypes.byref(ss),
                                                    _ptr(splats), _ptr(visible), _ptr(tiles), _ptr(depth_key))
    return dict(splats=splats, visible=visible.astype(bool), tiles_touched=tiles, depth_key=depth_key,
                status=int(rc))


def count_tiles(splats, width, height, tile_size, dtype="f64"):
    npt, sfx = _rt(dtype)
    splats = np.ascontiguousarray(splats, dtype=npt)
    tiles = np.zeros(splats.shape[0], dtype=np.int32)
    getattr(lib(), f"oracle_count_tiles_{sfx}")(_ptr(splats), ctypes.c_int64(splats.shape[0]), int(width),
                                                int(height), int(tile_size), _ptr(tiles))
    return tiles


def bin_tiles(splats, tiles_touched, width, height, tile_size, dtype="f64", depth_key=None):
    npt, sfx = _rt(dtype)
    splats = np.ascontiguousarray(splats, dtype=npt)
    tiles_touched = np.ascontiguousarray(tiles_touched, dtype=np.int32)
    tx, ty = -(-width // tile_size), -(-height // tile_size)
    offsets = np.zeros(tx * ty + 1, dtype=np.int64)
    n = ctypes.c_int64(splats.shape[0])
    fn = getattr(lib(), f"oracle_bin_{sfx}")
    total = int(tiles_touched.astype(np.int64).sum())
    ids = np.zeros(max(total, 1), dtype=np.int64)
    dk = None if depth_key is None else np.ascontiguousarray(depth_key, dtype=np.float64)
    got = fn(_ptr(splats), _ptr(tiles_touched), _ptr(dk), n, int(width), int(height), int(tile_size),
             _ptr(offsets), _ptr(ids), ctypes.c_int64(ids.size))
    assert got == total, (got, total)
    return offsets, ids[:total], tx, ty


def blend_forward(splats, offsets, ids, width, height, tile_size, background, record_hits=False, dtype="f64"):
    npt, sfx = _rt(dtype)
    splats = np.ascontiguousarray(splats, dtype=npt)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    bg = np.asarray(background, dtype=np.float64)
    image = np.zeros((height, width, 3), dtype=npt)
    T = np.ones((height, width), dtype=npt)
    ws = np.zeros((height, width), dtype=npt)
    nc = np.zeros((height, width), dtype=np.int32)
    lp = np.zeros((height, width), dtype=np.int32)
    hits = np.zeros(splats.shape[0], dtype=np.int64) if record_hits else None
    getattr(lib(), f"oracle_blend_fwd_{sfx}")(_ptr(splats), _ptr(offsets), _ptr(ids), int(width), int(height),
                                              int(tile_size), _ptr(bg), _ptr(image), _ptr(T), _ptr(ws), _ptr(nc),
                                              _ptr(lp), _ptr(hits))
    return dict(image=image, transmittance=T, weight_sum=ws, n_contrib=nc, last_pos=lp, hit_counts=hits)


def blend_backward(splats, offsets, ids, width, height, tile_size, background, transmit, last_pos, dimage,
                   dtype="f64"):
    npt, sfx = _rt(dtype)
    # every buffer handed to C is bound to a local first: a temporary passed straight into
    # _ptr() would be freed before the call (only its address survives), and under
    # concurrent callers its memory is reused at once
    splats = np.ascontiguousarray(splats, dtype=npt)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    bg = np.asarray(background, dtype=np.float64)
    transmit = np.ascontiguousarray(transmit, dtype=npt)
    last_pos = np.ascontiguousarray(last_pos, dtype=np.int32)
    dimage = np.ascontiguousarray(dimage, dtype=npt)
    dsp = np.zeros((splats.shape[0], 9), dtype=npt)
    getattr(lib(), f"oracle_blend_bwd_{sfx}")(
        _ptr(splats), _ptr(offsets), _ptr(ids), int(width), int(height), int(tile_size), _ptr(bg), _ptr(transmit),
        _ptr(last_pos), _ptr(dimage), _ptr(dsp))
    return dsp


def preprocess_backward(cloud, cam, settings, dsplats, dtype="f64"):
    npt, sfx = _rt(dtype)
    hold = _CloudHold(_fields_of(cloud))
    n = hold.n
    shapes = dict(positions=(n, 3), log_scales=(n, 3), rotations=(n, 4), opacity_logits=(n,), sh_dc=(n, 3),
                  sh_rest=(n, 15, 3), mask_logits=(n,), sh_mask_logits=(n, 3), mean2d_screen=(n, 2))
    g = {k: np.zeros(v, dtype=npt) for k, v in shapes.items()}
    cc, ss = _camera(cam), _settings(settings)
    dsp = np.ascontiguousarray(dsplats, dtype=npt)  # bound to a local: see blend_backward
    getattr(lib(), f"oracle_preprocess_bwd_{sfx}")(
        ctypes.byref(hold.c), ctypes.byref(cc), ctypes.byref(ss), _ptr(dsp),
        _ptr(g["positions"]), _ptr(g["log_scales"]), _ptr(g["rotations"]), _ptr(g["opacity_logits"]),
        _ptr(g["sh_dc"]), _ptr(g["sh_rest"]), _ptr(g["mask_logits"]), _ptr(g["sh_mask_logits"]),
        _ptr(g["mean2d_screen"]))
    return g


def render_forward(cloud, cam, settings, dtype="f64"):
    """Oracle counterpart of rasterizer.render_forward (rasterizer.py:215-284)."""
    fields = _fields_of(cloud)
    pre = preprocess(fields, cam, settings, dtype)
    if pre["status"] == 2:
        raise ValueError("degenerate rotation")
    W, H, ts = int(cam.width), int(cam.height), int(settings.tile_size)
    offsets, ids, tx, ty = bin_tiles(pre["splats"], pre["tiles_touched"], W, H, ts, dtype, pre["depth_key"])
    out = blend_forward(pre["splats"], offsets, ids, W, H, ts, settings.background,
                        getattr(settings, "record_hits", False), dtype)
    out.update(pre)
    out["offsets"], out["ids"], out["tiles_x"], out["tiles_y"] = offsets, ids, tx, ty
    out["screen_areas"] = pre["splats"][:, 11].copy()
    return out


def render_backward(cloud, cam, settings, dimage, fwd, dtype="f64"):
    """Oracle counterpart of rasterizer.render_backward (rasterizer.py:326-419)."""
    fields = _fields_of(cloud)
    W, H, ts = int(cam.width), int(cam.height), int(settings.tile_size)
    dsp = blend_backward(fwd["splats"], fwd["offsets"], fwd["ids"], W, H, ts, settings.background,
                         fwd["transmittance"], fwd["last_pos"], dimage, dtype)
    g = preprocess_backward(fields, cam, settings, dsp, dtype)
    g["dsplats"] = dsp
    return g
