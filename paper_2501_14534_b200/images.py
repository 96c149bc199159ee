"""Target-side progressive ops on the GPU (images.py:58-102 of the reference).

`area_resize` (exact fractional box filter) and `gaussian_blur` (separable,
reflect edges) over (H, W, 3) float32 CUDA tensors, via tgs_area_resize /
tgs_gaussian_blur.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import ContractViolationError


def area_resize(img: torch.Tensor, height: int, width: int) -> torch.Tensor:
    img = img.contiguous().float()
    h, w = int(img.shape[0]), int(img.shape[1])
    if height > h or width > w:
        raise ContractViolationError("area_resize only downsamples")  # images.py:72-73
    out = torch.empty((height, width, 3), dtype=torch.float32, device=img.device)
    ws = torch.empty((height, w, 3), dtype=torch.float32, device=img.device)
    _lib.call("tgs_area_resize", _lib.ptr(img), h, w, _lib.ptr(out), height, width, _lib.ptr(ws),
              _lib.stream_handle(img.device))
    return out


def gaussian_blur(img: torch.Tensor, size: int, sigma: float) -> torch.Tensor:
    img = img.contiguous().float()
    if size > 1 and size % 2 == 0:
        raise ContractViolationError("blur kernel size must be odd")  # images.py:94-95
    out = torch.empty_like(img)
    ws = torch.empty_like(img)
    _lib.call("tgs_gaussian_blur", _lib.ptr(img), int(img.shape[0]), int(img.shape[1]), int(size), float(sigma),
              _lib.ptr(out), _lib.ptr(ws), _lib.stream_handle(img.device))
    return out
