"""Adam over the flat parameter buffer (optim.py:37-73 of the reference).

The groups are contiguous ranges of GaussianCloud.flat; a full step updates all
of them in ONE `tgs_adam_step_groups` launch (per-group lr and bias
corrections, optional mask-penalty gradients added in registers), a partial
step uses `tgs_adam_step` per group.  Moments are kept in two flat buffers with
the same layout, so pruning compacts params and moments with the same gather
(optim.py:51-55).
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .cloud import PARAM_FIELDS, GaussianCloud


class Adam:
    def __init__(self, cloud: GaussianCloud, lrs: dict, beta1=0.9, beta2=0.999, eps=1e-15):
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.lrs = dict(lrs)
        self.m = torch.zeros_like(cloud.flat)
        self.v = torch.zeros_like(cloud.flat)
        self.steps = {f: 0 for f in PARAM_FIELDS}

    def set_lr(self, name: str, lr: float) -> None:
        self.lrs[name] = lr

    def update(self, cloud: GaussianCloud, grads, name: str) -> None:
        """optim.py:37-49 for one group, in place on cloud.<name>."""
        off, size = cloud.field_range(name)
        goff, _ = grads.field_range(name)
        self.steps[name] += 1
        t = self.steps[name]
        _lib.call("tgs_adam_step", _lib.ptr(cloud.flat[off:]), _lib.ptr(grads.flat[goff:]), _lib.ptr(self.m[off:]),
                  _lib.ptr(self.v[off:]), size, float(self.lrs[name]), self.beta1, self.beta2, self.eps,
                  1.0 - self.beta1 ** t, 1.0 - self.beta2 ** t, _lib.stream_handle(cloud.device))

    def step(self, cloud: GaussianCloud, grads, names=PARAM_FIELDS, lambda_m: float = 0.0,
             lambda_sh: float = 0.0, guard=None, ranges=None, count: bool = True) -> None:
        """Update the groups `names` in ONE fused launch (tgs_adam_step_groups).  lambda_m /
        lambda_sh add the mask penalties of total_loss (masking.py:60-67) to the
        mask-logit gradients first (when those groups are among `names`).

        guard: optional (terms, flag) device tensors — float64 loss terms and an int32
        flag: if any term is not finite the launch updates nothing and sets the flag
        (the reference raises DivergenceError before its update, training.py:298-308).
        The host-side step counters are still advanced; the caller rolls them back.

        ranges: optional [(begin, end), ...] flat-buffer float ranges to update (a rank's
        ZeRO-1 shard; one launch per range); count=False leaves the step counters as they
        are (the further launches of one logical step)."""
        import ctypes
        from .loss import SH_BAND_WEIGHTS
        names = sorted(set(names), key=lambda f: cloud.field_range(f)[0])  # layout order
        k = len(names)
        if k == 0:
            return
        offs, sizes, lrs, b1s, b2s, kinds = [], [], [], [], [], []
        for f in names:
            off, size = cloud.field_range(f)
            goff, _ = grads.field_range(f)
            if goff != off:
                raise ValueError("gradient and parameter layouts differ")
            if count:
                self.steps[f] += 1
            t = self.steps[f]
            offs.append(off)
            sizes.append(size)
            lrs.append(float(self.lrs[f]))
            b1s.append(1.0 - self.beta1 ** t)
            b2s.append(1.0 - self.beta2 ** t)
            kinds.append(1 if (f == "mask_logits" and lambda_m) else (2 if (f == "sh_mask_logits" and lambda_sh) else 0))
        arr = lambda ct, xs: (ct * k)(*xs)  # noqa: E731
        args = (k, arr(ctypes.c_int64, offs), arr(ctypes.c_int64, sizes), arr(ctypes.c_float, lrs),
                arr(ctypes.c_float, b1s), arr(ctypes.c_float, b2s), arr(ctypes.c_int32, kinds), self.beta1,
                self.beta2, self.eps, float(lambda_m), float(lambda_sh), (ctypes.c_float * 3)(*SH_BAND_WEIGHTS),
                len(cloud), _lib.ptr(guard[0]) if guard is not None else None,
                int(guard[0].numel()) if guard is not None else 0, _lib.ptr(guard[1]) if guard is not None else None)
        rs = [(int(a), int(b)) for a, b in ranges if b > a] if ranges is not None else []
        if ranges is not None and not rs:
            if guard is None:
                return
            rs = [(0, 0)]  # nothing to update, but the guard still writes its flag
        for i in range(0, max(len(rs), 1), 8):  # one launch per 8 ranges (nranges = 0: all)
            part = rs[i:i + 8]
            _lib.call("tgs_adam_step_groups", _lib.ptr(cloud.flat), _lib.ptr(grads.flat), _lib.ptr(self.m),
                      _lib.ptr(self.v), *args, (ctypes.c_int64 * max(len(part), 1))(*[a for a, _ in part] or [0]),
                      (ctypes.c_int64 * max(len(part), 1))(*[b for _, b in part] or [0]),
                      len(part) if ranges is not None else 0, _lib.stream_handle(cloud.device))


def exponential_lr(step: int, lr_init: float, lr_final: float, max_steps: int) -> float:
    """optim.py:68-73."""
    if step >= max_steps:
        return lr_final
    t = max(step, 0) / max_steps
    return float(math.exp((1.0 - t) * math.log(lr_init) + t * math.log(lr_final)))
