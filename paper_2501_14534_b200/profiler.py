"""CUDA-event stage timing for the bench (tracing).

`with stage("blend_fwd"): ...` records a start/end event pair on the current
stream (the stream every libtgs call is launched on) when a StageTimer is
active, and costs nothing otherwise.  Durations are device time, read after the
timed region's closing synchronize.
"""

from __future__ import annotations

import contextlib

import torch

_active = None


class StageTimer:
    def __init__(self):
        self.pairs: dict[str, list] = {}

    def __enter__(self):
        global _active
        self._prev, _active = _active, self
        return self

    def __exit__(self, *a):
        global _active
        _active = self._prev

    def durations_ms(self) -> dict:
        return {k: sum(s.elapsed_time(e) for s, e in v) for k, v in self.pairs.items()}

    def counts(self) -> dict:
        return {k: len(v) for k, v in self.pairs.items()}


@contextlib.contextmanager
def stage(name: str):
    t = _active
    if t is None:
        yield
        return
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    try:
        yield
    finally:
        e.record()
        t.pairs.setdefault(name, []).append((s, e))
