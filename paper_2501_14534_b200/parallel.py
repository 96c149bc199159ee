"""Multi-GPU partitioning of the rasterizer path.

The reference is single-process; this module adds the two
partitions the north star asks for, one process per GPU over NCCL:

* render: IMAGE TILE-ROW SHARDING.  Every rank runs the (cheap, 47 us at 1M)
  preprocess over all Gaussians, computes the same per-tile-row instance
  histogram, and therefore the same balanced split points without any
  communication; it bins, sorts and blends only its band of tile rows, and one
  all-gather assembles the image rows.  The blend order of every pixel is the
  same as the single-GPU render, so the assembled image is bitwise identical.
* training: CAMERA-VIEW DATA PARALLELISM.  Rank r renders views r, r+W, ...;
  gradients accumulate locally into one flat buffer and ONE all-reduce(sum)
  combines them (train.Trainer), followed by a replicated Adam step.

The split / gather / shard logic below is pure host code over torch tensors
and runs under gloo on the CPU (tests/test_parallel.py); the GPU entry points
compose it with the CUDA kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .profiler import stage


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin view assignment (view v -> rank v % world)."""
    return list(range(rank, n_views, world))


def row_split(row_counts, world: int) -> list[tuple[int, int]]:
    """Split tile rows [0, R) into `world` contiguous bands of ~equal instance count.

    Deterministic in its input, so every rank derives the same bands from the
    same replicated histogram.  Every band is non-empty when R >= world."""
    c = np.asarray(row_counts, dtype=np.float64)
    R = c.size
    if world <= 1 or R == 0:
        return [(0, R)]
    world = min(world, R)
    cum = np.concatenate([[0.0], np.cumsum(c + 1e-9)])  # +eps: empty rows still split evenly
    total = cum[-1]
    cuts = [0]
    for k in range(1, world):
        target = total * k / world
        r = int(np.searchsorted(cum, target, side="left"))
        r = min(max(r, cuts[-1] + 1), R - (world - k))  # keep every band non-empty
        cuts.append(r)
    cuts.append(R)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def gather_rows(band: torch.Tensor, bands: list[tuple[int, int]], rank: int, tile: int, height: int,
                group=None) -> torch.Tensor:
    """All-gather image row bands into the full (H, ...) image on every rank.

    `band` is this rank's full-height buffer; only its own rows are read."""
    world = len(bands)
    rows = [(b * tile, min(e * tile, height)) for b, e in bands]
    maxr = max(e - b for b, e in rows)
    trailing = tuple(band.shape[1:])
    mine = torch.zeros((maxr,) + trailing, dtype=band.dtype, device=band.device)
    b0, e0 = rows[rank]
    mine[: e0 - b0] = band[b0:e0]
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    out = torch.empty((height,) + trailing, dtype=band.dtype, device=band.device)
    for (b, e), p in zip(rows, parts):
        out[b:e] = p[: e - b]
    return out


def row_histogram(splats: torch.Tensor, tiles_touched: torch.Tensor, n: int, cam, tile_size: int) -> torch.Tensor:
    """Instances per tile row (int64, tiles_y) via tgs_row_histogram."""
    ty = (cam.height + tile_size - 1) // tile_size
    out = torch.zeros(ty, dtype=torch.int64, device=splats.device)
    if n:
        _lib.call("tgs_row_histogram", _lib.ptr(splats), _lib.ptr(tiles_touched), n, int(cam.width),
                  int(cam.height), tile_size, _lib.ptr(out), _lib.stream_handle(splats.device))
    return out


def render_sharded(cloud, cam, settings, group=None):
    """Tile-row-sharded render_forward: returns the full image on every rank."""
    from .rasterizer import _bin, preprocess
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ts = int(settings.tile_size)
    n = len(cloud)
    dev = cloud.device
    splats, vis, tiles, keys, err, exact = preprocess(cloud, cam, settings)  # replicated
    with stage("row_split"):
        counts = row_histogram(splats, tiles, n, cam, ts).cpu().numpy()
    bands = row_split(counts, world)
    if rank >= len(bands):  # more ranks than tile rows: idle rank
        bands_r = (0, 0)
    else:
        bands_r = bands[rank]
    h, w = int(cam.height), int(cam.width)
    image = torch.zeros((h, w, 3), dtype=torch.float32, device=dev)
    if bands_r[1] > bands_r[0]:
        from .rasterizer import _lib as lib
        bins = _bin(splats, tiles, n, w, h, ts, bands_r[0], bands_r[1], err, keys)
        transmit = torch.empty((h, w), dtype=torch.float32, device=dev)
        wsum = torch.empty_like(transmit)
        nc = torch.empty((h, w), dtype=torch.int32, device=dev)
        lp = torch.empty_like(nc)
        c_cam, c_set = lib.make_camera(cam), lib.make_settings(settings)
        with stage("blend_fwd"):
            lib.call("tgs_blend_forward", lib.ptr(splats), lib.ptr(exact), lib.ptr(bins.offsets), lib.ptr(bins.indices),
                     ctypes.byref(c_cam), ctypes.byref(c_set), bands_r[0], bands_r[1], lib.ptr(image),
                     lib.ptr(transmit), lib.ptr(wsum), lib.ptr(nc), lib.ptr(lp), None, lib.ptr(bins.order),
                     lib.stream_handle(dev))
    while len(bands) < world:
        bands.append((bands[-1][1], bands[-1][1]))
    with stage("gather"):
        return gather_rows(image, bands, rank, ts, h, group)


def allreduce_grads(flat: torch.Tensor, group=None) -> None:
    """Sum the flat CloudGrads buffer over ranks (one NCCL all-reduce)."""
    dist.all_reduce(flat, group=group)


def grad_buckets(layout: dict, rest_grads: bool = True) -> list[tuple[tuple[str, ...], int, int]]:
    """Contiguous ranges [start, end) of the flat gradient buffer to all-reduce, with the
    parameter groups each one completes, in the order they should be reduced.

    The SH-rest bucket (45 of 63 floats per Gaussian) goes first so that its Adam
    update overlaps the reduction of the small buckets; on steps without higher-band
    gradients (compute_sh_rest_grads=False, 15 of 16 steps with the SH cadence) the
    sh_rest and sh_mask_logits gradients are exactly zero on every rank and are not
    reduced at all (15 instead of 63 floats per Gaussian).
    mean2d_screen (densification statistics) is never reduced per step."""
    end = lambda f: layout[f][0] + layout[f][1]  # noqa: E731
    geo = ("positions", "log_scales", "rotations", "opacity_logits", "sh_dc")
    out = []
    if rest_grads:
        out.append((("sh_rest",), layout["sh_rest"][0], end("sh_rest")))
    out.append((geo, layout["positions"][0], end("sh_dc")))
    # sh_mask_logits is optimised every step (its penalty gradient), but its rendering
    # gradient is zero without higher-band gradients: only mask_logits needs reducing then
    out.append((("mask_logits", "sh_mask_logits"), layout["mask_logits"][0],
                end("sh_mask_logits" if rest_grads else "mask_logits")))
    return out
