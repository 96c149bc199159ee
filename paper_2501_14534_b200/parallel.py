"""Multi-GPU partitioning of the rasterizer path.

The reference is single-process; this module adds the two
partitions the north star asks for, one process per GPU over NCCL:

* render: IMAGE TILE-ROW SHARDING.  Every rank runs the (cheap, 47 us at 1M)
  preprocess over all Gaussians, computes the same per-tile-row instance
  histogram, and therefore the same balanced split points without any
  communication; it bins, sorts and blends only its band of tile rows, and one
  all-gather assembles the image rows.  The blend order of every pixel is the
  same as the single-GPU render, so the assembled image is bitwise identical.
* training: CAMERA-VIEW DATA PARALLELISM.  Rank r renders views r, r+W, ...
  (train.Trainer).  dp_mode="gaussians" (bench.py's default) shards the Gaussians too
  (the exchanges at the end of this module): each rank preprocesses its rows of the cloud
  for every view, all-to-alls carry the outputs to the view owners and the splat
  partials back, and each rank runs the preprocess backward and Adam on its rows.
  ZeRO-1 (reduce-scatter, Adam on 1/W, all-gather; zero_plan; the Trainer's default,
  which also serves its deterministic and one-stream paths) and one bucketed
  all-reduce + replicated Adam (grad_buckets) are the other modes.

The split / gather / shard logic below is pure host code over torch tensors
and runs under gloo on the CPU (tests/test_parallel.py); the GPU entry points
compose it with the CUDA kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

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


def assemble_bands(parts: list, bands: list[tuple[int, int]], tile: int, height: int) -> list:
    """Rank 0's side of the gather: parts[r] is rank r's (frames, max band rows, W, C)
    buffer holding its band's pixel rows first; returns the full (H, W, C) frames."""
    nf, _, w = parts[0].shape[:3]
    frames = []
    for f in range(nf):
        img = torch.empty((height, w) + tuple(parts[0].shape[3:]), dtype=parts[0].dtype, device=parts[0].device)
        for (b, e), p in zip(bands, parts):
            r0, r1 = b * tile, min(e * tile, height)
            if r1 > r0:
                img[r0:r1] = p[f, : r1 - r0]
        frames.append(img)
    return frames


class ShardedRenderer:
    """Tile-row-sharded rendering of a sequence of frames (the c4 orbit) over a process group.

    Every rank runs the (replicated, cheap) multi-view preprocess and bins + blends only its
    band of tile rows of each frame, through the native batch driver (rasterizer.
    render_views with row_bands).  The bands of a batch come from the per-tile-row instance
    histogram of the PREVIOUS batch's last frame — replicated on every rank, so every rank
    derives the same split with no communication, and read back asynchronously, so no host
    round trip sits on the render path (the first batch splits the rows evenly).  The band
    rows of every frame of the batch go to rank 0 in ONE NCCL gather.  The blend order of
    each pixel is the single-GPU one: the assembled frames are bitwise identical."""

    def __init__(self, cloud, settings, group=None, streams: int = 3):
        self.cloud, self.settings, self.group, self.streams = cloud, settings, group, streams
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.hist = None      # pinned host histogram of the last frame rendered
        self.hist_ready = None
        self.last_bands = None

    def bands(self, rows: int) -> list[tuple[int, int]]:
        if self.hist is not None and self.hist.numel() == rows:
            self.hist_ready.synchronize()  # recorded a whole batch ago: long complete
            out = row_split(self.hist.numpy(), self.world)
        else:
            out = row_split(np.ones(rows), self.world)
        while len(out) < self.world:  # more ranks than tile rows: idle ranks
            out.append((out[-1][1], out[-1][1]))
        return out

    def render(self, cams) -> list | None:
        """Frames `cams` (same resolution); returns their (H, W, 3) images on rank 0, None
        on the other ranks."""
        from .rasterizer import render_views
        cams = list(cams)
        ts = int(self.settings.tile_size)
        h, w = int(cams[0].height), int(cams[0].width)
        rows = (h + ts - 1) // ts
        bands = self.bands(rows)
        self.last_bands = bands
        rb, re = bands[self.rank]
        dev = self.cloud.device
        maxr = max(min(e * ts, h) - b * ts for b, e in bands)
        buf = torch.zeros((len(cams), max(maxr, 1), w, 3), dtype=torch.float32, device=dev)
        if re > rb:
            outs = render_views(self.cloud, cams, self.settings, streams=self.streams, row_bands=[(rb, re)] * len(cams))
            r0, r1 = rb * ts, min(re * ts, h)
            for f, o in enumerate(outs):
                buf[f, : r1 - r0] = o.image[r0:r1]
            st = outs[-1]._state
            splats, tiles = st.splats, st.tiles_touched
        else:  # no rows for this rank (more ranks than tile rows): the histogram still needs
            # the last frame's preprocess, so that every rank derives the same next bands
            from .rasterizer import preprocess
            splats, _, tiles, _, _, _ = preprocess(self.cloud, cams[-1], self.settings)
        # next batch's bands: the last frame's full-view row histogram (replicated preprocess)
        with stage("row_histogram"):
            hist = row_histogram(splats, tiles, len(self.cloud), cams[-1], ts)
        if self.hist is None or self.hist.numel() != rows:
            self.hist = torch.empty(rows, dtype=torch.int64, pin_memory=True)
        self.hist.copy_(hist, non_blocking=True)
        self.hist_ready = torch.cuda.Event()
        self.hist_ready.record()
        with stage("gather"):
            parts = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(buf, parts, dst=0, group=self.group)
        if self.rank != 0:
            return None
        return assemble_bands(parts, bands, ts, h)


def render_sharded(cloud, cam, settings, group=None, renderer: ShardedRenderer | None = None):
    """Tile-row-sharded render_forward of one frame: the full image on rank 0 (None on the
    other ranks).  Pass the same `renderer` across frames to balance the bands by the
    previous frame's histogram."""
    r = renderer if renderer is not None else ShardedRenderer(cloud, settings, group)
    out = r.render([cam])
    return out[0] if out is not None else None


# ---------------------------------------------------------------- ZeRO-1 data parallelism
# The flat gradient buffer is REDUCE-SCATTERED (each rank receives the sum of one shard),
# each rank runs the fused Adam on its shard only, and the updated parameters are
# ALL-GATHERED back: the same bytes on the wire as one all-reduce, but Adam's 28 B per
# parameter float are split over the ranks (the replicated
# Adam did not shrink with the rank count).  The parameter range is cut into chunks that
# pipeline: chunk k's all-gather overlaps chunk k+1's Adam, whose reduce-scatter overlapped
# chunk k's.

@dataclass
class ZeroChunk:
    begin: int   # first float of the chunk in the flat parameter / gradient buffers
    shard: int   # floats per rank (a multiple of 64)
    end: int     # real end of the chunk's data; begin + world * shard may run past it

    def padded_end(self, world: int) -> int:
        return self.begin + world * self.shard

    def rank_range(self, rank: int) -> tuple[int, int]:
        """The floats this rank updates (possibly empty)."""
        a = self.begin + rank * self.shard
        return a, max(a, min(a + self.shard, self.end))


def zero_plan(layout: dict, world: int, rest_grads: bool = True, chunks: int = 4) -> list[ZeroChunk]:
    """Chunks of the parameter range for ZeRO-1 (layout: CloudGrads' field map).

    Segments: all parameters, or — on steps without higher-band gradients (the SH cadence),
    whose sh_rest gradient is zero and which do not update sh_rest — the fields before and
    after sh_rest.  Each segment is cut into `chunks` pieces whose lengths are multiples of
    world x 64 floats, so the padded extent of a piece never reaches into the next one
    (the reduce-scatter is in place); only a segment's LAST piece is padded past the
    segment's end, into sh_rest (zero gradient, replicated parameters not updated on such
    steps) or into the ZERO_PAD headroom after the parameters (cloud._layout)."""
    from .cloud import params_end
    world = max(1, int(world))
    unit = world * 64
    end = params_end(layout)
    if rest_grads or layout["mask_logits"][0] - layout["sh_rest"][0] < unit:
        # (a tiny cloud's sh_rest cannot hold a padded tail: one segment; the zero sh_rest
        # gradient is then reduced too, and Adam still leaves sh_rest alone on such steps)
        segments = [(0, end)]
    else:
        segments = [(0, layout["sh_rest"][0]), (layout["mask_logits"][0], end)]
    out = []
    for a, b in segments:
        n_units = -(-(b - a) // unit)
        per = max(1, -(-n_units // max(1, chunks)))
        u = 0
        while u < n_units:
            k = min(per, n_units - u)
            c0 = a + u * unit
            out.append(ZeroChunk(c0, k * 64, min(b, c0 + k * unit)))
            u += k
    return out


def _backend(group=None) -> str:
    return dist.get_backend(group)


def reduce_scatter_inplace(flat: torch.Tensor, ch: ZeroChunk, rank: int, world: int, group=None) -> None:
    """Sum chunk `ch` of `flat` over ranks into this rank's shard slice (in place).
    (gloo has no reduce-scatter: an all-reduce of the padded chunk, same result.)"""
    full = flat[ch.begin: ch.padded_end(world)]
    if world == 1:
        return
    if _backend(group) == "gloo":
        dist.all_reduce(full, group=group)
        return
    a = ch.begin + rank * ch.shard
    dist.reduce_scatter_tensor(flat[a: a + ch.shard], full, group=group)


def all_gather_inplace(flat: torch.Tensor, ch: ZeroChunk, rank: int, world: int, group=None) -> None:
    """Every rank's shard of chunk `ch` to every rank (in place)."""
    if world == 1:
        return
    full = flat[ch.begin: ch.padded_end(world)]
    a = ch.begin + rank * ch.shard
    if _backend(group) == "gloo":
        parts = [torch.empty_like(flat[a: a + ch.shard]) for _ in range(world)]
        dist.all_gather(parts, flat[a: a + ch.shard].clone(), group=group)
        full.copy_(torch.cat(parts))
        return
    dist.all_gather_into_tensor(full, flat[a: a + ch.shard], group=group)


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


# ---------------------------------------------------------------------------
# Gaussian-sharded data parallelism (train.Trainer dp_mode="gaussians").  Rank r owns
# cloud rows shard_rows(n, world)[r]: it runs the multi-view preprocess of EVERY view of
# the step over its rows only, and one all-to-all per view slot delivers to each view's
# owner the full per-Gaussian preprocess outputs of its view (rows arrive in rank order,
# which is the cloud's row order, so the depth sort and the blends are the single-GPU
# ones bit for bit).  After the view's blend backward, a second all-to-all returns each
# shard's rows of the view's splat partials to the shard owner, which runs the multi-view
# preprocess backward and Adam over its rows only.  Per step and rank this exchanges the
# preprocess outputs (GSHARD_FWD_BYTES per Gaussian and view) and the splat partials
# (36 B) instead of ZeRO-1's reduce-scatter + all-gather of the 252 B/Gaussian parameter
# range, and the preprocess forward / backward and Adam are 1/world of the cloud.

# splats (12 f32), visible (u8), tiles_touched (i32), depth keys (i64), exact records (8 f32)
GSHARD_FWD_KINDS = ((0, 48), (1, 1), (2, 4), (3, 8), (5, 32))
GSHARD_FWD_BYTES = sum(b for _, b in GSHARD_FWD_KINDS)
GSHARD_BWD_BYTES = 36


def shard_rows(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row shards of a cloud of n rows, one per rank, in rank order; shard
    starts are multiples of 64 (Adam's per-field row ranges, train._row_ranges)."""
    world = max(1, int(world))
    per = -(-max(n, 1) // world)
    per = -(-per // 64) * 64
    return [(min(n, r * per), min(n, (r + 1) * per)) for r in range(world)]


def slot_order(views_of: list[list[int]]) -> list[int]:
    """The step's global view order for the shard-local preprocess: slot-major (slot j:
    view j of rank 0, of rank 1, ...), so that slot j's outputs for all ranks are one
    contiguous block — the all-to-all's input.  Every rank must own the same number of
    views."""
    k = len(views_of[0]) if views_of else 0
    if any(len(v) != k for v in views_of):
        raise ValueError("dp_mode='gaussians' needs the same number of views on every rank")
    return [views_of[d][j] for j in range(k) for d in range(len(views_of))]


def _a2a(out: torch.Tensor, inp: torch.Tensor, out_splits: list[int], in_splits: list[int], group) -> None:
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)


def gshard_forward_exchange(sub: list, full: list, rows: list[tuple[int, int]], rank: int, group=None) -> None:
    """Slot j of every rank's shard outputs to slot j's view owners.

    sub:  per output kind, the shard-local preprocess buffer [V][n_rank][...] of this rank
          (V = k x world views in slot_order);
    full: per output kind, this rank's own views' full buffers [k][n][...];
    group None: no communication, only this rank's own rows are written into `full`
    (single-GPU simulation of one rank's share, bench.py --rank-share --dp gaussians)."""
    world = len(rows)
    a, b = rows[rank]
    for s, f in zip(sub, full):
        k = f.shape[0]
        w = s[0, 0].numel() if s.dim() > 2 else 1
        for j in range(k):
            blk = s[j * world:(j + 1) * world]
            if group is None:
                f[j, a:b].copy_(blk[rank, :b - a])
                continue
            _a2a(f[j].reshape(-1), blk[:, :b - a].reshape(-1), [(e - d) * w for d, e in rows], [(b - a) * w] * world,
                 group)


def gshard_backward_exchange(own: list, sub: torch.Tensor, rows: list[tuple[int, int]], rank: int,
                             group=None) -> None:
    """Each own view's splat partials (own[j]: [n][9]) back to the shard owners: rank r
    receives rows rows[r] of every view, as sub[j * world + d] = partials of slot j's view
    of rank d ([V][n_rank][9], slot_order).  group None: only this rank's own rows."""
    world = len(rows)
    a, b = rows[rank]
    for j, p in enumerate(own):
        blk = sub[j * world:(j + 1) * world]
        if group is None:
            blk[rank, :b - a].copy_(p[a:b])
            continue
        out = blk[:, :b - a]
        if out.is_contiguous():
            _a2a(out.reshape(-1), p.reshape(-1), [(b - a) * 9] * world, [(e - d) * 9 for d, e in rows], group)
        else:  # (an empty shard's one-row padding)
            tmp = torch.empty_like(out)
            _a2a(tmp.reshape(-1), p.reshape(-1), [(b - a) * 9] * world, [(e - d) * 9 for d, e in rows], group)
            out.copy_(tmp)
