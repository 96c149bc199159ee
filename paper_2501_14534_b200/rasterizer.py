"""Drop-in rasterizer API over libtgs.so.

Mirrors `slimsplat.rasterizer` (rasterizer.py:44-419): same function names,
argument lists, settings fields, output field names and exceptions, with
float32 CUDA tensors in place of float64 numpy arrays:

    render_forward(cloud, cam, settings) -> RenderOutput      (rasterizer.py:215)
    render_backward(cloud, cam, settings, dimage, output)     (rasterizer.py:326)
        -> CloudGrads
    bin_tiles(means2d, radii, depths, width, height, tile_size) -> TileBins
                                                              (rasterizer.py:95)
    sh_rest_update_step(iteration, cadence) -> bool           (rasterizer.py:88)

Deliberate differences:
  * RenderOutput.visible / screen_areas / hit_counts are full-length (N,) as in the
    reference; TileBins.indices are CLOUD ROWS (the reference indexes its
    compacted visible subset — same order, different numbering).
  * render_backward reuses the forward's projected records and tile lists instead
    of re-running _prepare (rasterizer.py:342); results are identical by
    construction because both passes see the same cloud, camera and settings.
    If `output` carries no device state (e.g. built by hand), it recomputes them.
  * extension keywords: `grads=` / `accumulate=` on render_backward let a
    multi-view step accumulate into one CloudGrads buffer; `row_band=` renders
    a band of tile rows (tile-row sharding, parallel.py); `deterministic=True`
    selects the fixed-order (bitwise reproducible) gradient reduction.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

import torch

from . import _lib
from .cameras import Camera
from .cloud import CloudGrads, GaussianCloud
from .errors import ContractViolationError, DegenerateRotationError
from .profiler import stage

NEAR_PLANE = 0.01  # geometry.py:16
ALPHA_SKIP = 1.0 / 255.0
ALPHA_MAX = 0.99
E_MIN = -4.5
T_TERMINATE = 1e-4


@dataclass
class RenderSettings:
    """rasterizer.py:44-55."""

    lowpass_s: float = 0.3
    active_sh_degree: int = 3
    background: tuple = (0.0, 0.0, 0.0)
    tile_size: int = 16
    near: float = NEAR_PLANE
    record_hits: bool = False
    record_full: bool = False
    mask_threshold: float = 0.05
    sh_mask_threshold: float = 0.1
    compute_sh_rest_grads: bool = True


@dataclass
class TileBins:
    """Per-tile depth-sorted Gaussian lists in CSR layout (rasterizer.py:78-85)."""

    offsets: torch.Tensor  # (tiles_y*tiles_x + 1,) int32
    indices: torch.Tensor  # (I,) int32 cloud rows
    tiles_x: int
    tiles_y: int
    row_begin: int = 0
    row_end: int | None = None
    order: torch.Tensor | None = None  # heaviest-first blend launch order (tgs_tile_order), 16-px tiles


@dataclass
class _DeviceState:
    """Forward products reused by the backward."""

    cloud_ptr: int
    n: int
    splats: torch.Tensor        # (N, 12)
    visible_u8: torch.Tensor    # (N,)
    tiles_touched: torch.Tensor
    depth_keys: torch.Tensor | None
    bins: TileBins
    exact: torch.Tensor | None = None  # (N, 8) exact blend-decision records (include/tgs.h TGS_EXACT_FLOATS)
    exceptions: torch.Tensor | None = None    # (H, W) int32 blend exceptions of the forward (tgs_blend_forward)
    exc_overflow: torch.Tensor | None = None  # TGS_EXC_OVERFLOW_WORDS(ntiles) int32 (uint32 words)


@dataclass
class RenderOutput:
    """rasterizer.py:58-75."""

    image: torch.Tensor          # (H, W, 3)
    transmittance: torch.Tensor  # (H, W)
    weight_sum: torch.Tensor     # (H, W)
    n_contrib: torch.Tensor      # (H, W) int32
    last_pos: torch.Tensor       # (H, W) int32
    visible: torch.Tensor        # (N,) bool
    screen_areas: torch.Tensor   # (N,)
    hit_counts: torch.Tensor | None = None
    hit_records: list | None = None
    _tiles: TileBins | None = field(default=None, repr=False)
    _state: _DeviceState | None = field(default=None, repr=False)


def sh_rest_update_step(iteration: int, cadence: int) -> bool:
    """Whether higher-band SH gradients are computed at this iteration (rasterizer.py:88-92)."""
    if cadence < 1:
        raise ContractViolationError("SH update cadence must be >= 1")
    return iteration % cadence == 0


def _tiles_y(cam, ts):
    return (cam.height + ts - 1) // ts


def _tiles_x(cam, ts):
    return (cam.width + ts - 1) // ts


@dataclass
class _BinPending:
    """First half of a binning (tgs_bin_gaussians issued, its instance count on its way to
    a pinned host buffer); _bin_end finishes it."""
    splats: torch.Tensor
    n: int
    width: int
    height: int
    ts: int
    row_begin: int
    row_end: int
    has_err: bool
    cs: object          # the stream it runs on
    ws: torch.Tensor    # tgs_bin_gaussians workspace (per-stream scratch; read by tgs_bin_instances)
    h: torch.Tensor     # pinned (count, error flag)
    ev: object          # recorded after the copy


_WS_G: dict = {}   # n -> tgs_bin_gaussians_workspace bytes
_WS_I: dict = {}   # (n, band geometry) -> (largest count queried, its workspace bytes)


def _ws_gauss(n: int) -> int:
    b = _WS_G.get(n)
    if b is None:
        b = _WS_G[n] = ctypes_size("tgs_bin_gaussians_workspace", n)
    return b


def _ws_inst(n: int, count: int, width: int, height: int, ts: int, rb: int, re: int) -> int:
    """tgs_bin_instances_workspace, queried only when the count exceeds the largest one
    seen for this geometry (the size is non-decreasing in the count, so that size is
    an upper bound for every smaller count)."""
    key = (n, width, height, ts, rb, re)
    hi = _WS_I.get(key)
    if hi is None or count > hi[0]:
        hi = _WS_I[key] = (count, ctypes_size("tgs_bin_instances_workspace", n, count, width, height, ts, rb, re))
    return hi[1]


def _bin_begin(splats: torch.Tensor, tiles_touched: torch.Tensor, n: int, width: int, height: int, ts: int,
               row_begin: int, row_end: int, err: torch.Tensor | None = None,
               depth_keys: torch.Tensor | None = None, cs=None) -> _BinPending:
    """tgs_bin_gaussians and an asynchronous read of the instance count (+ the preprocess
    error flag, forwarded by the kernel).  Callers may begin the next view's binning on
    ANOTHER stream before ending this one, so the GPU has work queued while the host
    waits for this count (not on the same stream: the workspace is that stream's
    scratch).  Only explicit-stream calls: no framework stream switch."""
    dev = splats.device
    cs = cs if cs is not None else torch.cuda.current_stream(dev)
    st = cs.cuda_stream
    ws = _scratch("bin_g", max(_ws_gauss(n), 16), dev, st)
    d_count = _scratch("count", 16, dev, st)
    with stage("bin_gaussians"):
        _lib.call("tgs_bin_gaussians", _lib.ptr(splats), _lib.ptr(tiles_touched), _lib.ptr(depth_keys), n, width,
                  height, ts, row_begin, row_end, _lib.ptr(ws), _lib.ptr(d_count), _lib.ptr(err), st)
    h = _pinned_count(st)
    _lib.call("tgs_memcpy_d2h_async", h.data_ptr(), _lib.ptr(d_count), 16, st)
    ev = torch.cuda.Event()
    ev.record(cs)
    return _BinPending(splats, n, width, height, ts, row_begin, row_end, err is not None, cs, ws, h, ev)


def _bin_end(p: _BinPending) -> TileBins:
    """Waits for the instance count (the render's only host round trip) and issues
    tgs_bin_instances on the pending binning's stream (the caller's current stream, or
    render_views' allocation stream, owns the returned buffers)."""
    dev = p.splats.device
    st = p.cs.cuda_stream
    p.ev.synchronize()
    count, flag = int(p.h[0]), int(p.h[1]) if p.has_err else 0
    if flag:
        raise DegenerateRotationError("quaternion with (near-)zero norm")
    ts, width, height, rb, re = p.ts, p.width, p.height, p.row_begin, p.row_end
    tiles_x = (width + ts - 1) // ts
    tiles_y = (height + ts - 1) // ts
    ntiles = (re - rb) * tiles_x
    offsets, ids = _alloc_many([((ntiles + 1,), torch.int32), ((_size_class(max(count, 1)),), torch.int32)], dev)
    ws2 = _scratch("bin_i", max(_ws_inst(p.n, count, width, height, ts, rb, re), 16), dev, st)
    with stage("bin_instances"):
        _lib.call("tgs_bin_instances", _lib.ptr(p.splats), p.n, width, height, ts, rb, re, _lib.ptr(p.ws),
                  count, _lib.ptr(ws2), _lib.ptr(offsets), _lib.ptr(ids), st)
        order = _blend_order(offsets, ntiles, tiles_x, re - rb, ts, dev, st)
    return TileBins(offsets, ids[:count], tiles_x, tiles_y, rb, re, order)


def _bin(splats: torch.Tensor, tiles_touched: torch.Tensor, n: int, width: int, height: int, ts: int,
         row_begin: int, row_end: int, err: torch.Tensor | None = None,
         depth_keys: torch.Tensor | None = None, cs=None) -> TileBins:
    """tgs_bin_gaussians + one host read of the instance count + tgs_bin_instances."""
    return _bin_end(_bin_begin(splats, tiles_touched, n, width, height, ts, row_begin, row_end, err, depth_keys, cs))


_PINNED = {}
_CENTER = {}

# Launch order of the 16x16-tile blend kernels (scheduling only: results are identical):
#   "center": tiles by distance from the band's centre, a cached permutation per tile grid —
#             the heavy tiles of an object-centred view start first while neighbouring tiles,
#             which share splat records in L2, are still dispatched together (measured at
#             c3: blend fwd 288 -> 275 us, bwd 612 -> 578 us per view, no extra launch);
#   "lpt":    heaviest list first (tgs_tile_order, two small kernels per view), for scenes
#             whose heavy tiles are not central;
#   "none":   row-major.
BLEND_ORDER = "center"

# Exact (float64) blend decisions at the thresholds (include/tgs.h TGS_EXACT_FLOATS): on by
# default; TGS_EXACT=0 makes the blend kernels decide every pair in float32 (A/B timing of
# the decision cost only — the north-star parity needs the records).
import os as _os
EXACT_DECISIONS = _os.environ.get("TGS_EXACT", "1") != "0"
# The blend forward's exception lists (tgs_blend_forward `exceptions`): the backward then
# decides the bracket pairs without float64.  TGS_EXC=0: the backward re-resolves them
# (A/B timing; same results).
EXCEPTION_LISTS = EXACT_DECISIONS and _os.environ.get("TGS_EXC", "1") != "0"


def _ex(exact):
    return exact if EXACT_DECISIONS else None


def _blend_order(offsets, ntiles: int, tiles_x: int, rows: int, ts: int, dev, st):
    if ts != 16 or ntiles == 0 or BLEND_ORDER == "none":
        return None
    if BLEND_ORDER == "lpt":
        order = _alloc(ntiles + 64, torch.int32, dev)
        _lib.call("tgs_tile_order", _lib.ptr(offsets), ntiles, _lib.ptr(order), st)
        return order
    key = (dev.index, tiles_x, rows)
    order = _CENTER.get(key)
    if order is None:  # (2x2 / 4x4 tile blocks ordered centre-out measured slower than plain rings)
        ty, tx = np.meshgrid(np.arange(rows), np.arange(tiles_x), indexing="ij")
        d = (tx + 0.5 - tiles_x / 2.0) ** 2 + (ty + 0.5 - rows / 2.0) ** 2
        order = _CENTER[key] = torch.from_numpy(np.argsort(d.ravel(), kind="stable").astype(np.int32)).to(dev)
    return order
_SCRATCH = {}


def _scratch(tag: str, nbytes: int, dev, stream_handle: int | None = None, owner=None) -> torch.Tensor:
    """Per-stream scratch workspace, grown geometrically and reused by every later call on
    the same stream (stream order makes the reuse safe; nothing returned references it).
    Frame-to-frame size changes (instance counts) then cost no allocator traffic.
    owner: the torch stream using it, when that is not the current stream (the block is
    then allocated from that stream's pool)."""
    sh = stream_handle if stream_handle is not None else torch.cuda.current_stream(dev).cuda_stream
    key = (dev.index, sh, tag)
    t = _SCRATCH.get(key)
    if t is None or t.numel() < nbytes:
        size = _size_class(int(nbytes * 1.25) + 4096)
        if owner is not None:
            with torch.cuda.stream(owner):
                t = torch.empty(size, dtype=torch.uint8, device=dev)
        else:
            t = torch.empty(size, dtype=torch.uint8, device=dev)
        _SCRATCH[key] = t
    return t[:nbytes]


def _size_class(k: int) -> int:
    """Round an element count up to one of 8 classes per binade (<= 12.5% slack) so
    buffers whose size follows the per-frame instance count are served from the
    allocator's cache instead of fresh cudaMalloc calls."""
    if k <= 1024:
        return 1024
    step = 1 << (k.bit_length() - 4)
    return (k + step - 1) // step * step


def _pinned_count(stream_handle: int = 0) -> torch.Tensor:
    """A pinned 2-element host buffer per (host thread, stream): a stream's read completes
    before its next binning reuses the buffer."""
    k = (threading.get_ident(), stream_handle)
    h = _PINNED.get(k)
    if h is None:
        h = _PINNED[k] = torch.empty(2, dtype=torch.int64, pin_memory=True)
    return h


def ctypes_size(fn: str, *args) -> int:
    import ctypes
    out = ctypes.c_size_t(0)
    _lib.call(fn, *args, ctypes.byref(out))
    return int(out.value)


def bin_tiles(means2d, radii, depths, width: int, height: int, tile_size: int) -> TileBins:
    """GPU bin_tiles on raw arrays (rasterizer.py:95-148); indices are input rows."""
    if tile_size < 1:
        raise ContractViolationError("tile_size must be >= 1")
    dev = torch.device("cuda")
    m = torch.as_tensor(np.asarray(means2d) if not torch.is_tensor(means2d) else means2d).to(dev, torch.float32)
    n = int(m.shape[0])
    sp = torch.zeros((max(n, 1), 12), dtype=torch.float32, device=dev)
    if n:
        sp[:n, 0:2] = m.reshape(n, 2)
        sp[:n, 9] = torch.as_tensor(np.asarray(depths) if not torch.is_tensor(depths) else depths).to(dev, torch.float32)
        sp[:n, 10] = torch.as_tensor(np.asarray(radii) if not torch.is_tensor(radii) else radii).to(dev, torch.float32)
    tiles = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    st = _lib.stream_handle(dev)
    if n:
        _lib.call("tgs_count_tiles", _lib.ptr(sp), n, width, height, tile_size, _lib.ptr(tiles), st)
    ty = (height + tile_size - 1) // tile_size
    return _bin(sp, tiles, n, width, height, tile_size, 0, ty)


def _as_cloud(cloud) -> GaussianCloud:
    if isinstance(cloud, GaussianCloud):
        return cloud
    return GaussianCloud.from_fields(cloud)


def preprocess(cloud: GaussianCloud, cam: Camera, settings: RenderSettings):
    """tgs_preprocess_forward: (splats (N,12), visible u8, tiles_touched i32, float64 depth keys, error flag,
    exact blend-decision records (N,8))."""
    n = len(cloud)
    dev = cloud.device
    splats = torch.empty((max(n, 1), 12), dtype=torch.float32, device=dev)
    vis = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    tiles = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    exact = torch.zeros((max(n, 1), 8), dtype=torch.float32, device=dev)
    if n:
        c_cloud, c_cam, c_set = cloud.native(), _lib.make_camera(cam), _lib.make_settings(settings)
        import ctypes
        with stage("preprocess_fwd"):
            _lib.call("tgs_preprocess_forward", ctypes.byref(c_cloud), ctypes.byref(c_cam), ctypes.byref(c_set),
                      _lib.ptr(splats), _lib.ptr(vis), _lib.ptr(tiles), _lib.ptr(keys), _lib.ptr(err),
                      _lib.ptr(exact), _lib.stream_handle(dev))
    return splats, vis, tiles, keys, err, exact


_ROW_BYTES = None  # bytes per cloud row of each parameter field (cloud._ROW)


def _offset_rows(c_cloud, c_grads, c_stats, r0: int, r1: int) -> None:
    """Point native cloud / gradient / statistics structs at cloud rows [r0, r1) (in place:
    every per-row field pointer advanced by r0 rows, n = r1 - r0)."""
    global _ROW_BYTES
    if _ROW_BYTES is None:
        from .cloud import PARAM_FIELDS, _ROW
        _ROW_BYTES = tuple((f, 4 * int(np.prod(_ROW[f]))) for f in PARAM_FIELDS)
    for f, w in _ROW_BYTES:
        setattr(c_cloud, f, getattr(c_cloud, f) + w * r0)
        if c_grads is not None:
            setattr(c_grads, f, getattr(c_grads, f) + w * r0)
    if c_grads is not None:
        c_grads.mean2d_screen = c_grads.mean2d_screen + 4 * 2 * r0 if c_grads.mean2d_screen else None
    c_cloud.n = r1 - r0
    if c_stats is not None:
        c_stats.grad_accum = c_stats.grad_accum + 4 * r0 if c_stats.grad_accum else None
        c_stats.grad_count = c_stats.grad_count + 4 * r0 if c_stats.grad_count else None
        c_stats.area_max = c_stats.area_max + 4 * r0 if c_stats.area_max else None


def preprocess_views(cloud: GaussianCloud, cams: list, settings: RenderSettings, stats=None,
                     exact: bool = True, cache: dict | None = None, c_cams=None, rows: tuple | None = None) -> list:
    """tgs_preprocess_forward_views: the per-view preprocess outputs of a batch of views in
    one pass over the parameters; element v is what `preprocess(cloud, cams[v], settings)`
    returns (bit-identical), the error flag shared.  stats: optional train.DensifyStats
    (its area_max takes the views' screen areas, training.py:338).  exact=False leaves the
    exact blend-decision records to a later exact_records() call (e.g. on another stream).
    cache: a dict owned by a caller that runs this every step on one stream (the
    Trainer): the output buffers, their per-view views and the pointer arrays are made
    once per (views, rows) and reused — the previous call's outputs are overwritten, so
    their consumers must be ordered before this call on the stream (~0.15 ms of host
    work per step saved, all of it GPU idle at the start of a step).
    rows=(r0, r1): only cloud rows [r0, r1) — a rank's Gaussian shard (train.Trainer
    dp_mode="gaussians"); the outputs then have r1 - r0 rows, row i being cloud row r0 + i."""
    import ctypes
    r0, r1 = rows if rows is not None else (0, len(cloud))
    n = max(r1 - r0, 0)
    dev = cloud.device
    V = len(cams)
    m = max(n, 1)
    key = (V, m, dev, r0)
    ent = cache.get(key) if cache is not None else None
    if ent is None:
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        # one allocation per output kind for the whole batch; the kernel writes every row
        # below n, the padding row of an empty cloud is zeroed
        sp = torch.empty((V, m, 12), dtype=torch.float32, device=dev)
        vis = torch.empty((V, m), dtype=torch.uint8, device=dev)
        tiles = torch.empty((V, m), dtype=torch.int32, device=dev)
        keys = torch.empty((V, m), dtype=torch.int64, device=dev)
        ex = torch.empty((V, m, 8), dtype=torch.float32, device=dev)
        outs = [(sp[v], vis[v], tiles[v], keys[v], err, ex[v]) for v in range(V)]
        ptrs = [(ctypes.c_void_p * V)(*[o[k].data_ptr() for o in outs]) for k in range(6)]
        ent = (outs, ptrs, err, (sp, vis, tiles, keys, ex))
        if cache is not None:
            cache.clear()  # one geometry at a time (a pruned cloud frees the old buffers)
            cache[key] = ent
    else:
        ent[2].zero_()
    outs, ptrs, err, bases = ent
    if n == 0:
        for t in bases:
            t.zero_()
    if n and V:
        c_cloud, c_set = cloud.native(), _lib.make_settings(settings)
        if c_cams is None:  # (a caller issuing several calls per step passes its own array)
            c_cams = (_lib.TgsCamera * V)(*[_lib.make_camera(c) for c in cams])
        with stage("preprocess_fwd"):
            c_stats = stats.native() if stats is not None else None
            if rows is not None:
                _offset_rows(c_cloud, None, c_stats, r0, r1)
            _lib.call("tgs_preprocess_forward_views", ctypes.byref(c_cloud), c_cams, ctypes.byref(c_set), V, ptrs[0],
                      ptrs[1], ptrs[2], ptrs[3], _lib.ptr(err), ctypes.byref(c_stats) if c_stats else None,
                      ptrs[5] if exact else None, _lib.stream_handle(dev))
    return outs


def exact_records(cloud: GaussianCloud, cams: list, settings: RenderSettings, pres: list,
                  cache: dict | None = None, c_cams=None, rows: tuple | None = None) -> None:
    """tgs_exact_records_views on the current stream: the exact blend-decision records
    (include/tgs.h TGS_EXACT_FLOATS) of preprocess_views(..., exact=False) outputs.
    cache: preprocess_views' cache of the same call (its pointer arrays are reused).
    rows: the preprocess_views call's row range."""
    import ctypes
    r0, r1 = rows if rows is not None else (0, len(cloud))
    n, V = max(r1 - r0, 0), len(cams)
    if n == 0 or V == 0:
        return
    c_cloud, c_set = cloud.native(), _lib.make_settings(settings)
    if rows is not None:
        _offset_rows(c_cloud, None, None, r0, r1)
    if c_cams is None:
        c_cams = (_lib.TgsCamera * V)(*[_lib.make_camera(c) for c in cams])
    ent = cache.get((V, max(n, 1), cloud.device, r0)) if cache is not None else None
    if ent is not None and ent[0] is pres:
        sps, exs = ent[1][0], ent[1][5]
    else:
        sps = (ctypes.c_void_p * V)(*[p[0].data_ptr() for p in pres])
        exs = (ctypes.c_void_p * V)(*[p[5].data_ptr() for p in pres])
    with stage("exact_records"):
        _lib.call("tgs_exact_records_views", ctypes.byref(c_cloud), c_cams, ctypes.byref(c_set), V, sps, exs,
                  _lib.stream_handle(cloud.device))


_RENDER_STREAMS = {}
_ALLOC = threading.local()  # .stream: the pool returned tensors are allocated from (None: current)


def _alloc(shape, dtype, dev) -> torch.Tensor:
    """torch.empty for tensors a render RETURNS.  Inside render_views they come from the
    caller's stream pool while the kernels writing them run on side streams: the caller's
    stream waits for the side streams before returning, so any later reuse of that memory
    is ordered after the writes (no record_stream, no allocator churn)."""
    s = getattr(_ALLOC, "stream", None)
    if s is None:
        return torch.empty(shape, dtype=dtype, device=dev)
    with torch.cuda.stream(s):
        return torch.empty(shape, dtype=dtype, device=dev)


def _alloc_many(specs, dev) -> list:
    """Several returned tensors carved from ONE allocation (256-byte aligned typed views):
    one allocator call, and one stream switch inside render_views, per frame."""
    offs, total = [], 0
    for shape, dtype in specs:
        n = 1
        for d in shape:
            n *= int(d)
        offs.append(total)
        total += (n * dtype.itemsize + 255) // 256 * 256
    blk = _alloc(max(total, 256), torch.uint8, dev)
    out = []
    for (shape, dtype), o in zip(specs, offs):
        n = 1
        for d in shape:
            n *= int(d)
        out.append(blk[o:o + n * dtype.itemsize].view(dtype).view(shape))
    return out


_RV_CAP: dict = {}  # (device, n, tile, resolutions) -> per-view instance-id capacity of the native path


def _render_views_native(cloud, cams, settings, pool, main, cap: int, bands=None):
    """tgs_render_views: the whole batch issued from C++ (see include/tgs.h).  Returns the
    outputs, or the largest instance count of the batch when a buffer was too small."""
    import ctypes
    from .errors import TGS_ERR_CAPACITY, raise_for_status
    n, dev, V, ts = len(cloud), cloud.device, len(cams), int(settings.tile_size)
    c_set = _lib.make_settings(settings)
    # preprocess outputs and every view's render outputs: allocated from the caller's
    # stream pool (the side streams wait for it first and it waits for them at the end)
    sp = torch.empty((V, n, 12), dtype=torch.float32, device=dev)
    vis = torch.empty((V, n), dtype=torch.uint8, device=dev)
    tiles = torch.empty((V, n), dtype=torch.int32, device=dev)
    keys = torch.empty((V, n), dtype=torch.int64, device=dev)
    exact = torch.empty((V, n, 8), dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    geo = []
    specs = []
    for cam in cams:
        h, w = int(cam.height), int(cam.width)
        tx, ty = (w + ts - 1) // ts, (h + ts - 1) // ts
        geo.append((h, w, tx, ty))
        specs += [((h, w, 3), torch.float32), ((h, w), torch.float32), ((h, w), torch.float32), ((h, w), torch.int32),
                  ((h, w), torch.int32), ((tx * ty + 1,), torch.int32), ((cap,), torch.int32)]
        if settings.record_hits:
            specs.append(((n,), torch.int32))
    bufs = _alloc_many(specs, dev)
    per = 8 if settings.record_hits else 7
    targets = (_lib.TgsViewTarget * V)()
    orders = []
    for v, (h, w, tx, ty) in enumerate(geo):
        b = bufs[per * v: per * (v + 1)]
        if settings.record_hits:
            b[7].zero_()
        rb, re = bands[v] if bands is not None else (0, ty)
        order = _blend_order(None, (re - rb) * tx, tx, re - rb, ts, dev, None) if BLEND_ORDER == "center" else None
        orders.append(order)
        targets[v] = _lib.TgsViewTarget(b[5].data_ptr(), b[6].data_ptr(), cap, _lib.ptr(order), b[0].data_ptr(),
                                        b[1].data_ptr(), b[2].data_ptr(), b[3].data_ptr(), b[4].data_ptr(),
                                        b[7].data_ptr() if settings.record_hits else None, -1, rb, re)
    ns = len(pool)
    wsb = max(ctypes_size("tgs_render_views_workspace", n, cap, w, h, ts) for h, w, _, _ in geo)
    wss = [_scratch("render_views", wsb, dev, s_.cuda_stream, owner=s_) for s_ in pool]
    pkey = (threading.get_ident(), "render_views", ns)  # per host thread: the driver reads it synchronously
    pinned = _PINNED.get(pkey)
    if pinned is None:
        pinned = _PINNED[pkey] = torch.empty(2 * ns, dtype=torch.int64, pin_memory=True)
    c_cams = (_lib.TgsCamera * V)(*[_lib.make_camera(c) for c in cams])
    arr = lambda t: (ctypes.c_void_p * V)(*[t[v].data_ptr() for v in range(V)])  # noqa: E731
    c_cloud = cloud.native()
    # each view's blend on a normal-priority stream after its binning (the binning pool is
    # high priority): measured +4% FPS at c3 over blending on the binning streams
    key = ("blend", dev.index, ns)
    bpool = _RENDER_STREAMS.get(key)
    if bpool is None:
        bpool = _RENDER_STREAMS[key] = [torch.cuda.Stream(device=dev, priority=0) for _ in range(ns)]
    for s_ in pool + bpool:
        s_.wait_stream(main)
    rc = int(_lib.load().tgs_render_views(
        ctypes.byref(c_cloud), c_cams, ctypes.byref(c_set), V, arr(sp), arr(vis), arr(tiles), arr(keys), arr(exact),
        err.data_ptr(), targets, (ctypes.c_void_p * ns)(*[t.data_ptr() for t in wss]), wsb, pinned.data_ptr(),
        (ctypes.c_void_p * ns)(*[s_.cuda_stream for s_ in pool]),
        (ctypes.c_void_p * ns)(*[s_.cuda_stream for s_ in bpool]), ns))
    if rc == TGS_ERR_CAPACITY:
        for s_ in pool + bpool:  # the partial batch still writes these buffers: drain first
            s_.synchronize()
        return max(int(targets[v].num_instances) for v in range(V))
    for s_ in pool + bpool:
        main.wait_stream(s_)
    raise_for_status(rc, "tgs_render_views")
    outs = []
    for v, (h, w, tx, ty) in enumerate(geo):
        b = bufs[per * v: per * (v + 1)]
        count = int(targets[v].num_instances)
        rb, re = bands[v] if bands is not None else (0, ty)
        bins = TileBins(b[5][: (re - rb) * tx + 1], b[6][:count], tx, ty, rb, re, orders[v])
        hit_counts = b[7].to(torch.int64) if settings.record_hits else None
        outs.append(RenderOutput(image=b[0], transmittance=b[1], weight_sum=b[2], n_contrib=b[3], last_pos=b[4],
                                 visible=vis[v].view(torch.bool), screen_areas=sp[v][:, 11], hit_counts=hit_counts,
                                 _tiles=bins,
                                 _state=_DeviceState(cloud.flat.data_ptr(), n, sp[v], vis[v], tiles[v], keys[v], bins,
                                                     exact[v])))
    return outs


def render_views(cloud, cams: list, settings: RenderSettings, streams: int = 3, row_bands: list | None = None) -> list:
    """Render a batch of views of one cloud (an orbit, the views of a training batch):
    every view's preprocess in ONE pass over the parameters (tgs_preprocess_forward_views),
    then per view binning + blending pipelined over `streams` CUDA streams, so the
    latency-bound binning of one view (and its instance-count read-back) overlaps the
    blending of the others.  Element v equals render_forward(cloud, cams[v], settings);
    the outputs are ordered before later work on the caller's current stream.
    row_bands: optional [(row_begin, row_end), ...] tile-row band per view (tile-row
    sharding): only those rows are binned and blended (the other pixels are unspecified)."""
    cloud = _as_cloud(cloud)
    cams = list(cams)
    if not cams:
        return []
    dev = cloud.device
    main = torch.cuda.current_stream(dev)
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), max(1, int(streams)))
    pool = _RENDER_STREAMS.get(key)
    if pool is None:
        # binning streams at high priority: their latency-bound kernels get SM slots first
        # and the (issue-bound) blends fill around them on their own streams
        pool = _RENDER_STREAMS[key] = [torch.cuda.Stream(device=dev, priority=-1) for _ in range(key[1])]
    # native path (tgs_render_views) once the batch's instance counts are known: the
    # per-view sequence is issued from C++, the Python cost is one call per batch
    _lib.make_settings(settings)
    geom = (key[0], len(cloud), int(settings.tile_size), tuple((int(c.width), int(c.height)) for c in cams))
    native = len(cloud) > 0 and not settings.record_full and len(cams) <= 64
    if native and geom in _RV_CAP:
        for _ in range(3):
            res = _render_views_native(cloud, cams, settings, pool, main, _RV_CAP[geom], row_bands)
            if isinstance(res, list):
                return res
            _RV_CAP[geom] = _size_class(int(res * 1.25) + 1024)
    outs = _render_views_py(cloud, cams, settings, pool, main, row_bands)
    if native:
        _RV_CAP[geom] = _size_class(int(max(o._tiles.indices.numel() for o in outs) * 1.25) + 1024)
    return outs


def _render_views_py(cloud, cams, settings, pool, main, row_bands=None) -> list:
    """render_views driven from Python (first batch of a geometry, record_full)."""
    dev = cloud.device
    pres = preprocess_views(cloud, cams, settings) if len(cloud) else [None] * len(cams)
    for s_ in pool:
        s_.wait_stream(main)
    outs = []
    _ALLOC.stream = main
    n = len(cloud)

    def begin(i):  # view i's depth sort and count read-back on its own stream
        if not n or len(pool) < 2:
            return None
        cam, (sp, _, tiles, keys, err, _) = cams[i], pres[i]
        ts = int(settings.tile_size)
        rb, re = row_bands[i] if row_bands is not None else (0, _tiles_y(cam, ts))
        with torch.cuda.stream(pool[i % len(pool)]):
            return _bin_begin(sp, tiles, n, int(cam.width), int(cam.height), ts, rb, re, err, keys)

    try:
        # the next len(pool) - 1 views' binnings are queued (each on its own stream) before
        # this view's count is awaited, so the GPU never idles on the host round trip
        ahead = max(len(pool) - 1, 1)
        pend = [begin(i) for i in range(min(ahead, len(cams)))]
        for i, cam in enumerate(cams):
            if i + ahead < len(cams):
                pend.append(begin(i + ahead))
            p_i = pend.pop(0)
            with torch.cuda.stream(pool[i % len(pool)]):
                bins = _bin_end(p_i) if p_i is not None else None
                outs.append(render_forward(cloud, cam, settings, pre=pres[i], bins=bins,
                                           row_band=row_bands[i] if row_bands is not None else None))
    finally:
        _ALLOC.stream = None
        for s_ in pool:
            main.wait_stream(s_)
    return outs


def render_forward(cloud, cam: Camera, settings: RenderSettings, row_band: tuple | None = None,
                   pre: tuple | None = None, bins: TileBins | None = None) -> RenderOutput:
    """Render a cloud into an (H, W, 3) image plus blending auxiliaries (rasterizer.py:215-284).

    pre: this view's outputs of `preprocess_views` (skips the per-view preprocess);
    bins: its tile lists from _bin_begin/_bin_end (pipelined callers, with `pre`)."""
    import ctypes
    cloud = _as_cloud(cloud)
    c_set = _lib.make_settings(settings)  # validates settings even for empty clouds
    if settings.tile_size > 32:
        raise ContractViolationError("tile_size > 32 is not supported by the CUDA kernels")
    h, w, ts = int(cam.height), int(cam.width), int(settings.tile_size)
    n = len(cloud)
    dev = cloud.device
    rb, re = row_band if row_band is not None else (0, _tiles_y(cam, ts))
    cs = torch.cuda.current_stream(dev)
    splats, vis, tiles, keys, err, exact = pre if pre is not None else preprocess(cloud, cam, settings)
    if bins is None:
        bins = _bin(splats, tiles, n, w, h, ts, rb, re, err, keys, cs)
    specs = [((h, w, 3), torch.float32), ((h, w), torch.float32), ((h, w), torch.float32), ((h, w), torch.int32),
             ((h, w), torch.int32)]
    if settings.record_hits:
        specs.append(((n,), torch.int64))
    bufs = _alloc_many(specs, dev)
    image, transmit, wsum, n_contrib, last_pos = bufs[:5]
    visible = vis[:n].view(torch.bool)  # the preprocess's 0/1 bytes, reinterpreted (no copy)
    if row_band is not None:  # pixels outside the band are not rendered here
        for t_, v in ((image, 0.0), (transmit, 1.0), (wsum, 0.0), (n_contrib, 0), (last_pos, 0)):
            t_.fill_(v)
    hits = torch.zeros(max(n, 1), dtype=torch.int32, device=dev) if settings.record_hits else None
    exc = ovf = None
    if EXCEPTION_LISTS and exact is not None and ts == 16:  # the backward's exception lists (include/tgs.h)
        exc, ovf = _alloc_many([((h, w), torch.int32), ((1 + (re - rb) * _tiles_x(cam, ts),), torch.int32)], dev)
    c_cam = _lib.make_camera(cam)
    with stage("blend_fwd"):
        _lib.call("tgs_blend_forward", _lib.ptr(splats), _lib.ptr(_ex(exact)), _lib.ptr(bins.offsets),
                  _lib.ptr(bins.indices),
                  ctypes.byref(c_cam), ctypes.byref(c_set), rb, re, _lib.ptr(image), _lib.ptr(transmit),
                  _lib.ptr(wsum), _lib.ptr(n_contrib), _lib.ptr(last_pos), _lib.ptr(hits), _lib.ptr(exc),
                  _lib.ptr(ovf), _lib.ptr(bins.order), cs.cuda_stream)
    hit_counts = None
    if hits is not None:
        hit_counts = bufs[5]
        hit_counts.copy_(hits[:n])
    out = RenderOutput(image=image, transmittance=transmit, weight_sum=wsum, n_contrib=n_contrib,
                       last_pos=last_pos, visible=visible, screen_areas=splats[:n, 11], hit_counts=hit_counts,
                       _tiles=bins, _state=_DeviceState(cloud.flat.data_ptr(), n, splats, vis, tiles, keys, bins, exact,
                                                        exc, ovf))
    if settings.record_full:
        out.hit_records = _records(out, splats, exact, bins, cam, c_cam, c_set, dev)
    return out


def _records(out, splats, exact, bins, cam, c_cam, c_set, dev):
    """Per-pixel [(cloud row, weight), ...] lists (rasterizer.py:287-323); debug payload."""
    import ctypes
    flat = out.n_contrib.reshape(-1).to(torch.int64)
    total = int(flat.sum().item())
    offsets = torch.zeros_like(flat)
    if flat.numel() > 1:
        offsets[1:] = torch.cumsum(flat[:-1], 0)
    g = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    wt = torch.empty(max(total, 1), dtype=torch.float32, device=dev)
    if total:
        _lib.call("tgs_blend_records", _lib.ptr(splats), _lib.ptr(_ex(exact)), _lib.ptr(bins.offsets),
                  _lib.ptr(bins.indices),
                  ctypes.byref(c_cam), ctypes.byref(c_set), _lib.ptr(offsets), _lib.ptr(g), _lib.ptr(wt),
                  _lib.stream_handle(dev))
    g, wt, cnt, off = g.cpu().numpy(), wt.cpu().numpy(), flat.cpu().numpy(), offsets.cpu().numpy()
    return [[(int(g[o + k]), float(wt[o + k])) for k in range(c)] for o, c in zip(off, cnt)]


def blend_backward(cloud: GaussianCloud, cam: Camera, settings: RenderSettings, dimage, output: RenderOutput,
                   dsplats: torch.Tensor | None = None, deterministic: bool = False):
    """First half of render_backward: the screen-space partials (N, 9) of one view
    (tgs_blend_backward, _kernels.py:92-181) plus the forward state they refer to.

    deterministic=True sums every Gaussian's per-tile partials in a fixed order
    (tgs_blend_backward_deterministic): bitwise reproducible, ~40 B/instance of scratch."""
    import ctypes
    if output is None or output.transmittance is None or output.last_pos is None:
        raise ContractViolationError("render_backward needs the forward pass auxiliaries")
    h, w = int(cam.height), int(cam.width)
    if tuple(dimage.shape) != (h, w, 3):
        raise ContractViolationError("upstream gradient shape does not match the camera")
    n = len(cloud)
    dev = cloud.device
    c_set = _lib.make_settings(settings)
    st = output._state
    if st is None or st.n != n or st.cloud_ptr != cloud.flat.data_ptr():
        # no reusable device state: recompute the forward products (rasterizer.py:342)
        splats, vis, tiles, keys, err, exact = preprocess(cloud, cam, settings)
        rb, re = (0, _tiles_y(cam, settings.tile_size))
        bins = _bin(splats, tiles, n, w, h, int(settings.tile_size), rb, re, err, keys)
        st = _DeviceState(cloud.flat.data_ptr(), n, splats, vis, tiles, keys, bins, exact)
    bins = st.bins
    rb = bins.row_begin
    re = bins.row_end if bins.row_end is not None else _tiles_y(cam, settings.tile_size)
    d = dimage if torch.is_tensor(dimage) else torch.from_numpy(np.ascontiguousarray(dimage, dtype=np.float32))
    d = d.to(dev, torch.float32).contiguous()
    transmit = output.transmittance.to(dev, torch.float32).contiguous()
    last_pos = output.last_pos.to(dev, torch.int32).contiguous()
    if dsplats is None:
        dsplats = torch.zeros((n, 9), dtype=torch.float32, device=dev)
    c_cam = _lib.make_camera(cam)
    with stage("blend_bwd"):
        if deterministic:
            ni = int(bins.indices.numel())
            nb = ctypes_size("tgs_blend_backward_deterministic_workspace", n, ni)
            ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)
            _lib.call("tgs_blend_backward_deterministic", _lib.ptr(st.splats), _lib.ptr(_ex(st.exact)),
                      _lib.ptr(st.tiles_touched), n,
                      _lib.ptr(bins.offsets), _lib.ptr(bins.indices), ni, ctypes.byref(c_cam), ctypes.byref(c_set),
                      rb, re, _lib.ptr(transmit), _lib.ptr(last_pos), _lib.ptr(d), _lib.ptr(dsplats), _lib.ptr(ws),
                      _lib.stream_handle(dev))
        else:
            _lib.call("tgs_blend_backward", _lib.ptr(st.splats), _lib.ptr(_ex(st.exact)), _lib.ptr(bins.offsets),
                      _lib.ptr(bins.indices),
                      ctypes.byref(c_cam), ctypes.byref(c_set), rb, re, _lib.ptr(transmit), _lib.ptr(last_pos),
                      _lib.ptr(st.exceptions), _lib.ptr(st.exc_overflow), _lib.ptr(d), _lib.ptr(dsplats),
                      _lib.ptr(bins.order), _lib.stream_handle(dev))
    return dsplats, st


def preprocess_backward_views(cloud: GaussianCloud, cams: list, settings: RenderSettings, visibles: list,
                              dsplats: list, grads: CloudGrads, accumulate: bool = False, stats=None,
                              clear: bool = False, rows: tuple | None = None, local: bool = False,
                              c_cams=None) -> CloudGrads:
    """Second half of render_backward for a batch of views in ONE pass over the
    parameters (tgs_preprocess_backward_views): grads (+)= sum over views.  stats:
    optional train.DensifyStats, accumulating each view's screen-space gradient norm
    (training.py:333-337).  clear=True zeroes every dsplats[v] after reading it (the
    training loop's buffers are then ready for the next step's blend backward).
    rows=(r0, r1): only cloud rows [r0, r1) (r0 a multiple of 64) — a chunk of a pipelined
    step whose Adam updates the finished rows while the next chunk runs.  local=True: the
    visibles / dsplats hold only those rows (a Gaussian shard's, train.Trainer
    dp_mode="gaussians"), row i being cloud row r0 + i.  c_cams: a caller's prebuilt
    camera array of `cams`."""
    import ctypes
    n = len(cloud)
    if n == 0 or not cams:
        return grads
    V = len(cams)
    r0, r1 = rows if rows is not None else (0, n)
    if r1 <= r0:
        return grads
    if c_cams is None:
        c_cams = (_lib.TgsCamera * V)(*[_lib.make_camera(c) for c in cams])
    o = 0 if local else r0
    vis_ptrs = (ctypes.c_void_p * V)(*[v.data_ptr() + o for v in visibles])
    ds_ptrs = (ctypes.c_void_p * V)(*[d.data_ptr() + 36 * o for d in dsplats])
    c_set = _lib.make_settings(settings)
    c_cloud, c_grads = cloud.native(), grads.native()
    c_stats = stats.native() if stats is not None else None
    if rows is not None:  # the same structs over the row sub-range (pointer offsets)
        _offset_rows(c_cloud, c_grads, c_stats, r0, r1)
    with stage("preprocess_bwd"):
        _lib.call("tgs_preprocess_backward_views", ctypes.byref(c_cloud), c_cams, ctypes.byref(c_set), vis_ptrs,
                  ds_ptrs, V, ctypes.byref(c_grads), int(bool(accumulate)),
                  ctypes.byref(c_stats) if c_stats else None, int(bool(clear)), _lib.stream_handle(cloud.device))
    return grads


def render_backward(cloud, cam: Camera, settings: RenderSettings, dimage, output: RenderOutput,
                    grads: CloudGrads | None = None, accumulate: bool = False,
                    deterministic: bool = False) -> CloudGrads:
    """Analytic gradients of sum(dimage * image) w.r.t. every cloud field (rasterizer.py:326-419)."""
    if output is None or output.transmittance is None or output.last_pos is None:
        raise ContractViolationError("render_backward needs the forward pass auxiliaries")
    if tuple(dimage.shape) != (int(cam.height), int(cam.width), 3):
        raise ContractViolationError("upstream gradient shape does not match the camera")
    cloud = _as_cloud(cloud)
    n = len(cloud)
    _lib.make_settings(settings)
    if grads is None:
        grads = CloudGrads(n, cloud.device)
        accumulate = False
    if n == 0:
        return grads
    dsplats, st = blend_backward(cloud, cam, settings, dimage, output, deterministic=deterministic)
    return preprocess_backward_views(cloud, [cam], settings, [st.visible_u8], [dsplats], grads, accumulate)
