"""Mask-based pruning with row compaction (config 5's compaction step).

`prune_by_mask` restates masking.prune_by_mask (masking.py:70-81): keep rows
whose hard mask sigmoid(m) > eps (evaluated in logit space like the kernels),
raise EmptySceneError when nothing survives, and compact the cloud with the
tgs_gather_rows kernel; `compact_adam` applies the same rows to the Adam
moments (optim.py:51-55) so optimizer state follows the cloud.
"""

from __future__ import annotations

import torch

from . import _lib
from .cloud import PARAM_FIELDS, GaussianCloud, _ROW
from .errors import ContractViolationError, EmptySceneError


def keep_indices(cloud: GaussianCloud, eps: float) -> torch.Tensor:
    if not 0.0 < eps < 1.0:
        raise ContractViolationError("mask threshold must lie in (0, 1)")
    thr = _lib.logit_floor_f32(eps)
    return torch.nonzero(cloud.mask_logits > thr, as_tuple=False).flatten()


def prune_by_mask(cloud: GaussianCloud, eps: float):
    keep = keep_indices(cloud, eps)
    if keep.numel() == 0:
        raise EmptySceneError("mask pruning would remove every Gaussian")
    if keep.numel() == len(cloud):
        return cloud, keep
    return cloud.take(keep), keep


def compact_adam(opt, old_cloud: GaussianCloud, new_cloud: GaussianCloud, keep: torch.Tensor) -> None:
    """Gather the kept rows of every moment buffer into the new cloud's layout."""
    m = torch.zeros_like(new_cloud.flat)
    v = torch.zeros_like(new_cloud.flat)
    st = _lib.stream_handle(new_cloud.device)
    k = keep.to(torch.int64).contiguous()
    for f in PARAM_FIELDS:
        row = 1
        for d in _ROW[f]:
            row *= d
        so, _ = old_cloud.field_range(f)
        do, _ = new_cloud.field_range(f)
        for src, dst in ((opt.m, m), (opt.v, v)):
            _lib.call("tgs_gather_rows", _lib.ptr(src[so:]), _lib.ptr(dst[do:]), _lib.ptr(k), int(k.numel()), row, st)
    opt.m, opt.v = m, v
