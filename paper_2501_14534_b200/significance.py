"""Ray-hit significance scoring and scheduled percentile pruning over the CUDA path.

Mirrors the reference's significance.py (same names, arguments, exceptions):

    count_hits(cloud, cameras, settings)            significance.py:31-42
    significance_scores(hits, cloud, ...)           significance.py:45-78  (tgs_significance_scores)
    prune_by_significance(cloud, scores, rate)      significance.py:81-99  (tgs_significance_keep)
    prune_schedule(event_index, first_rate, decay)  significance.py:100-104
    report_to_csv(report, path)                     significance.py:107-121

Hits come from the forward blend kernel's per-Gaussian counters (the renderer's
own contribution rule), every view's preprocess in one multi-view pass.  The
90th-percentile volume and the pruning threshold are order statistics selected
on the device (radix select), so a pruning event needs no host sort.  Arrays are
device tensors: hit counts int64, volumes / v_norm / scores float32.
"""

from __future__ import annotations

import csv
import ctypes
import math
from dataclasses import dataclass, replace

import torch

from . import _lib
from .cloud import GaussianCloud
from .errors import ContractViolationError, EmptySceneError
from .rasterizer import RenderSettings, preprocess_views, render_forward


@dataclass
class SignificanceReport:
    hit_counts: torch.Tensor  # (N,) int64
    volumes: torch.Tensor     # (N,) float32
    v_norm: torch.Tensor      # (N,) float32
    scores: torch.Tensor      # (N,) float32
    iteration: int = 0


def count_hits(cloud: GaussianCloud, cameras: list, settings: RenderSettings) -> torch.Tensor:
    """Per-Gaussian pixel-ray hit counts accumulated over all views."""
    if not cameras:
        raise ContractViolationError("count_hits needs at least one camera")
    hit_settings = replace(settings, record_hits=True, record_full=False)
    totals = torch.zeros(len(cloud), dtype=torch.int64, device=cloud.device)
    if len(cloud) == 0:
        return totals
    pres = preprocess_views(cloud, list(cameras), hit_settings)
    for cam, pre in zip(cameras, pres):
        totals += render_forward(cloud, cam, hit_settings, pre=pre).hit_counts
    return totals


def _workspace(n: int, device) -> torch.Tensor:
    nbytes = ctypes.c_size_t(0)
    _lib.call("tgs_significance_workspace", int(n), ctypes.byref(nbytes))
    return torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=device)


def significance_scores(hit_counts, cloud: GaussianCloud, mask_threshold: float = 0.05, volume_power: float = 0.5,
                        iteration: int = 0) -> SignificanceReport:
    """Hit-weighted opacity x normalized-volume scores (nearest-rank 90th-percentile
    volume normaliser; volumes above it saturate at 1 before the power)."""
    n = len(cloud)
    if n == 0:
        raise EmptySceneError("cannot score an empty cloud")
    if not 0.0 < mask_threshold < 1.0:
        raise ContractViolationError("mask threshold must lie in (0, 1)")  # masking.py:23-24
    dev = cloud.device
    hits = torch.as_tensor(hit_counts, device=dev).to(torch.int64).contiguous()
    if hits.shape != (n,):
        raise ContractViolationError("hit_counts must have one entry per Gaussian")
    rank = max(int(math.ceil(0.9 * n)) - 1, 0)  # significance.py:65 (float64 ceil, as numpy)
    volumes = torch.empty(n, dtype=torch.float32, device=dev)
    v_norm = torch.empty_like(volumes)
    scores = torch.empty_like(volumes)
    ws = _workspace(n, dev)
    c_cloud = cloud.native()
    _lib.call("tgs_significance_scores", ctypes.byref(c_cloud), _lib.ptr(hits),
              _lib.logit_floor_f32(mask_threshold), float(volume_power), rank, _lib.ptr(volumes), _lib.ptr(v_norm),
              _lib.ptr(scores), _lib.ptr(ws), ws.numel(), _lib.stream_handle(dev))
    return SignificanceReport(hit_counts=hits, volumes=volumes, v_norm=v_norm, scores=scores, iteration=iteration)


def prune_keep_indices(scores: torch.Tensor, rate: float) -> torch.Tensor:
    """Kept row indices (ascending) after dropping the floor(rate N) lowest
    (score, row) pairs — the row selection of prune_by_significance."""
    if not 0.0 < rate < 1.0:
        raise ContractViolationError("prune rate must lie in (0, 1)")
    scores = scores.to(torch.float32).contiguous()
    n = int(scores.numel())
    k = int(math.floor(rate * n))
    if k >= n:
        raise EmptySceneError("significance pruning would remove every Gaussian")
    if k == 0:
        return torch.arange(n, dtype=torch.int64, device=scores.device)
    keep = torch.empty(n, dtype=torch.uint8, device=scores.device)
    ws = _workspace(n, scores.device)
    _lib.call("tgs_significance_keep", _lib.ptr(scores), n, k, _lib.ptr(keep), _lib.ptr(ws), ws.numel(),
              _lib.stream_handle(scores.device))
    from .pruning import select_rows
    return select_rows(n, scores.device, flags=keep)


def prune_by_significance(cloud: GaussianCloud, scores: torch.Tensor, rate: float):
    """Drop the floor(rate * N) lowest-scoring Gaussians (ties: lower index pruned
    first).  Returns (pruned cloud, kept indices sorted ascending)."""
    if not 0.0 < rate < 1.0:
        raise ContractViolationError("prune rate must lie in (0, 1)")
    keep = prune_keep_indices(scores, rate)
    if keep.numel() == len(cloud):
        return cloud, keep
    return cloud.take(keep), keep


def prune_schedule(event_index: int, first_rate: float, decay: float) -> float:
    """Pruning rate for the k-th event: first_rate * decay^k."""
    if event_index < 0:
        raise ContractViolationError("event index must be >= 0")
    return first_rate * decay ** event_index


def report_to_csv(report: SignificanceReport, path) -> None:
    hits = report.hit_counts.cpu().tolist()
    vols, vn, sc = (t.double().cpu().tolist() for t in (report.volumes, report.v_norm, report.scores))
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["index", "hit_count", "volume", "v_norm", "score"])
        for i in range(len(sc)):
            w.writerow([i, int(hits[i]), repr(vols[i]), repr(vn[i]), repr(sc[i])])
