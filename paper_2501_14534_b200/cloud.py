"""Device-resident Gaussian scene container and gradient buffer.

Same field names, shapes and semantics as the reference's `GaussianCloud` /
`CloudGrads` (cloud.py:18-143), held as float32 CUDA tensors.  All fields are
views into ONE flat buffer (field-major, each field 256 B aligned) so the
multi-view gradient allreduce and the fused Adam step each touch a single
contiguous allocation.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import ContractViolationError

SH_REST_COEFFS = 15
DEFAULT_MASK_LOGIT = 2.0  # cloud.py:16
PARAM_FIELDS = ("positions", "log_scales", "rotations", "opacity_logits", "sh_dc", "sh_rest", "mask_logits",
                "sh_mask_logits")
_ROW = {"positions": (3,), "log_scales": (3,), "rotations": (4,), "opacity_logits": (), "sh_dc": (3,),
        "sh_rest": (SH_REST_COEFFS, 3), "mask_logits": (), "sh_mask_logits": (3,), "mean2d_screen": (2,)}
PARAM_FLOATS = sum(int(np.prod(_ROW[f])) for f in PARAM_FIELDS)  # 63


# Floats of headroom after the parameter fields (in both the parameter and the gradient
# layouts): a ZeRO-1 chunk is padded to a multiple of world x 64 floats, and its padded
# tail may run past the last parameter field (parallel.zero_plan, world <= 64).
ZERO_PAD = 4096


def _layout(fields, n):
    """Offsets (in floats) of each field inside the flat buffer, 64-float aligned, with
    ZERO_PAD floats between the parameter fields and anything after them."""
    off, out, padded = 0, {}, False
    for f in fields:
        if f not in PARAM_FIELDS and not padded:
            off += ZERO_PAD
            padded = True
        size = n * int(np.prod(_ROW[f]))
        out[f] = (off, size)
        off += (size + 63) // 64 * 64
    if not padded:
        off += ZERO_PAD
    return out, max(off, 64)


def params_end(layout: dict) -> int:
    """First float after the parameter fields (64-aligned)."""
    o, n = layout["sh_mask_logits"]
    return o + (n + 63) // 64 * 64


class _FlatFields:
    FIELDS: tuple = ()

    def _init_flat(self, n: int, device, flat: torch.Tensor | None = None):
        lay, total = _layout(self.FIELDS, n)
        if flat is None:
            flat = torch.zeros(total, dtype=torch.float32, device=device)
        object.__setattr__(self, "flat", flat)
        object.__setattr__(self, "_n", n)
        object.__setattr__(self, "_layout_map", lay)
        for f in self.FIELDS:
            o, s = lay[f]
            object.__setattr__(self, f, flat[o:o + s].view((n,) + _ROW[f]))

    def __len__(self) -> int:
        return self._n

    @property
    def device(self):
        return self.flat.device

    def __setattr__(self, name, value):
        if name in self.FIELDS:  # assignment copies into the flat buffer (keeps the layout)
            dst = getattr(self, name)
            src = torch.as_tensor(np.asarray(value) if not torch.is_tensor(value) else value)
            if tuple(src.shape) != tuple(dst.shape):
                raise ContractViolationError(f"field {name} has shape {tuple(src.shape)}, expected {tuple(dst.shape)}")
            dst.copy_(src.to(dtype=torch.float32))
            return
        object.__setattr__(self, name, value)

    def field_range(self, name):
        return self._layout_map[name]


class GaussianCloud(_FlatFields):
    """All per-Gaussian learnable state (cloud.py:30-107), float32 on one device."""

    FIELDS = PARAM_FIELDS

    def __init__(self, n: int = 0, device="cuda", flat: torch.Tensor | None = None, **fields):
        if fields and n == 0:
            n = int(np.asarray(fields["positions"]).shape[0]) if not torch.is_tensor(fields["positions"]) \
                else int(fields["positions"].shape[0])
        self._init_flat(n, device, flat)
        for f, v in fields.items():
            if f not in PARAM_FIELDS:
                raise ContractViolationError(f"unknown cloud field {f}")
            setattr(self, f, v)

    @classmethod
    def from_fields(cls, src, device="cuda") -> "GaussianCloud":
        """From a dict or any object with the PARAM_FIELDS attributes (e.g. the
        reference's numpy GaussianCloud); values are rounded to float32."""
        get = (lambda f: src[f]) if isinstance(src, dict) else (lambda f: getattr(src, f))
        first = get("positions")
        n = int(first.shape[0])
        host = torch.zeros(_layout(PARAM_FIELDS, n)[1], dtype=torch.float32, pin_memory=torch.cuda.is_available())
        tmp = cls.__new__(cls)
        tmp._init_flat(n, "cpu", host)
        for f in PARAM_FIELDS:
            v = get(f)
            t = v if torch.is_tensor(v) else torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float32)))
            if tuple(t.shape) != (n,) + _ROW[f]:
                raise ContractViolationError(f"cloud field {f} has shape {tuple(t.shape)}, expected {(n,) + _ROW[f]}")
            getattr(tmp, f).copy_(t)
        out = cls.__new__(cls)
        out._init_flat(n, device, host.to(device, non_blocking=True))
        return out

    @classmethod
    def zeros(cls, n: int, device="cuda") -> "GaussianCloud":
        c = cls(n, device)
        c.flat.zero_()
        c.rotations[:, 0] = 1.0
        c.mask_logits.fill_(DEFAULT_MASK_LOGIT)
        c.sh_mask_logits.fill_(DEFAULT_MASK_LOGIT)
        return c

    @property
    def opacities(self) -> torch.Tensor:
        return torch.sigmoid(self.opacity_logits)

    @property
    def scales(self) -> torch.Tensor:
        return torch.exp(self.log_scales)

    def copy(self) -> "GaussianCloud":
        out = GaussianCloud.__new__(GaussianCloud)
        out._init_flat(len(self), self.device, self.flat.clone())
        return out

    def take(self, indices) -> "GaussianCloud":
        """Row-compacted copy keeping `indices` in order (cloud.py:86-89), via the
        tgs_gather_rows kernel field by field."""
        from . import _lib
        idx = torch.as_tensor(np.asarray(indices) if not torch.is_tensor(indices) else indices,
                              dtype=torch.int64).to(self.device)
        out = GaussianCloud(int(idx.numel()), self.device)
        st = _lib.stream_handle(self.device)
        for f in PARAM_FIELDS:
            row = int(np.prod(_ROW[f]))
            _lib.call("tgs_gather_rows", _lib.ptr(getattr(self, f)), _lib.ptr(getattr(out, f)), _lib.ptr(idx),
                      int(idx.numel()), row, st)
        return out

    def to_numpy(self) -> dict:
        return {f: getattr(self, f).detach().cpu().numpy() for f in PARAM_FIELDS}

    def native(self):
        from ._lib import TgsCloud
        return TgsCloud(*[getattr(self, f).data_ptr() for f in PARAM_FIELDS], len(self))


class CloudGrads(_FlatFields):
    """Per-Gaussian partials (cloud.py:110-143) + `mean2d_screen`, one flat buffer."""

    FIELDS = PARAM_FIELDS + ("mean2d_screen",)

    def __init__(self, n: int, device="cuda", zero: bool = True):
        self._init_flat(n, device)
        if zero:
            self.flat.zero_()

    @classmethod
    def zeros(cls, n: int, device="cuda") -> "CloudGrads":
        return cls(n, device, zero=True)

    def finite(self) -> bool:
        return bool(torch.isfinite(self.flat).all())

    def native(self):
        from ._lib import TgsGrads
        return TgsGrads(*[getattr(self, f).data_ptr() for f in self.FIELDS])

    def to_numpy(self) -> dict:
        return {f: getattr(self, f).detach().cpu().numpy() for f in self.FIELDS}
