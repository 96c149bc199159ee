"""Adam over the flat parameter buffer (optim.py:37-73 of the reference).

One `tgs_adam_step` launch per named group (the groups are contiguous ranges of
GaussianCloud.flat), moments kept in two flat buffers with the same layout, so
pruning compacts params and moments with the same gather (optim.py:51-55).
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

    def step(self, cloud: GaussianCloud, grads, names=PARAM_FIELDS) -> None:
        for f in names:
            self.update(cloud, grads, f)


def exponential_lr(step: int, lr_init: float, lr_final: float, max_steps: int) -> float:
    """optim.py:68-73."""
    if step >= max_steps:
        return lr_final
    t = max(step, 0) / max_steps
    return float(math.exp((1.0 - t) * math.log(lr_init) + t * math.log(lr_final)))
