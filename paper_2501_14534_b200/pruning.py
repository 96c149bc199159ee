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


def select_rows(n: int, device, flags: torch.Tensor | None = None, x: torch.Tensor | None = None,
                threshold: float = 0.0) -> torch.Tensor:
    """Ascending int64 row numbers with flags != 0 (or x > threshold): the np.nonzero of
    the prunings, by the tgs_select_rows compaction kernel.  One host read of the count
    (the returned tensor's length)."""
    import ctypes
    nb = ctypes.c_size_t(0)
    _lib.call("tgs_select_rows_workspace", int(n), ctypes.byref(nb))
    ws = torch.empty(max(int(nb.value), 16), dtype=torch.uint8, device=device)
    idx = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    cnt = torch.zeros(1, dtype=torch.int64, device=device)
    _lib.call("tgs_select_rows", _lib.ptr(flags), _lib.ptr(x), float(threshold), int(n), _lib.ptr(idx), _lib.ptr(cnt),
              _lib.ptr(ws), ws.numel(), _lib.stream_handle(device))
    return idx[: int(cnt.item())]


def keep_indices(cloud: GaussianCloud, eps: float) -> torch.Tensor:
    """Rows whose hard mask survives: sigmoid(m) > eps <=> m > logit_floor(eps) (masking.py:21-25,
    evaluated in logit space like the kernels)."""
    if not 0.0 < eps < 1.0:
        raise ContractViolationError("mask threshold must lie in (0, 1)")
    thr = _lib.logit_floor_f32(eps)
    return select_rows(len(cloud), cloud.device, x=cloud.mask_logits, threshold=thr)


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
