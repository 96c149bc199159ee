"""Training loss image terms on the GPU (training.py:61-106, metrics.py:138-188).

`l1_ssim(image, target, lambda_ssim)` returns the reference's LossTerms values
for the image part — l1, d_ssim = (1 - SSIM) / 2 — and dL/dimage, computed by
tgs_loss_l1_ssim (one fused pipeline of four streaming kernels).  The mask
penalties (masking.py:46-67) are per-Gaussian elementwise terms handled by
`mask_terms`.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ContractViolationError

SH_BAND_WEIGHTS = (9.0 / 45.0, 15.0 / 45.0, 21.0 / 45.0)  # masking.py:18

_WS_BYTES: dict = {}  # (W, H) -> tgs_loss_workspace bytes


def _loss_bytes(w: int, h: int) -> int:
    nb = _WS_BYTES.get((w, h))
    if nb is None:
        out = ctypes.c_size_t(0)
        _lib.call("tgs_loss_workspace", w, h, ctypes.byref(out))
        nb = _WS_BYTES[(w, h)] = int(out.value)
    return nb


def _workspace(dev, w, h):
    """The loss workspace of the CURRENT stream (the SSIM partial planes written by
    k_ssim_fwd and read by k_ssim_adj, and the per-CTA sums of k_loss_finalize).
    Per stream, never shared: views whose loss pipelines run concurrently on different
    streams (train.Trainer) each get their own, and a workspace is only reused — or
    grown, its old block returning to that stream's pool — in that stream's order."""
    from .rasterizer import _scratch
    return _scratch("loss", _loss_bytes(w, h), dev)


def l1_ssim_async(image: torch.Tensor, target: torch.Tensor, lambda_ssim: float, dimage: torch.Tensor,
                  terms: torch.Tensor) -> None:
    """Stream-ordered form: writes dimage (H,W,3) and terms = [mean L1, mean SSIM] (float64, device)."""
    if image.shape != target.shape or image.dim() != 3 or image.shape[2] != 3:
        raise ContractViolationError(f"render {tuple(image.shape)} and target {tuple(target.shape)} resolutions differ")
    h, w = int(image.shape[0]), int(image.shape[1])
    if h < 11 or w < 11:
        raise ContractViolationError("image smaller than the SSIM window")  # metrics.py:83-84
    _lib.call("tgs_loss_l1_ssim", _lib.ptr(image), _lib.ptr(target), w, h, float(lambda_ssim), _lib.ptr(dimage),
              _lib.ptr(terms), _lib.ptr(_workspace(image.device, w, h)), _lib.stream_handle(image.device))


def l1_ssim(image: torch.Tensor, target: torch.Tensor, lambda_ssim: float = 0.2):
    image = image.contiguous().float()
    target = target.to(image.device).contiguous().float()
    dimage = torch.empty_like(image)
    terms = torch.empty(2, dtype=torch.float64, device=image.device)
    l1_ssim_async(image, target, lambda_ssim, dimage, terms)
    l1, ssim = (float(v) for v in terms.cpu().tolist())
    return {"l1": l1, "ssim": ssim, "d_ssim": (1.0 - ssim) / 2.0,
            "total": (1.0 - lambda_ssim) * l1 + lambda_ssim * (1.0 - ssim) / 2.0}, dimage


def mask_terms(mask_logits: torch.Tensor, sh_mask_logits: torch.Tensor):
    """(L_m, L_sh) and their logit gradients (masking.py:46-67)."""
    n = max(int(mask_logits.shape[0]), 1)
    m = torch.sigmoid(mask_logits)
    msh = torch.sigmoid(sh_mask_logits)
    w = torch.tensor(SH_BAND_WEIGHTS, device=m.device, dtype=m.dtype)
    l_m = m.mean() if m.numel() else m.sum()
    l_sh = (msh * w).sum(dim=1).mean() if msh.numel() else msh.sum()
    return l_m, l_sh, m * (1 - m) / n, msh * (1 - msh) * w / n
