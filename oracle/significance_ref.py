"""Significance scoring and pruning restated on the CPU — TEST INFRASTRUCTURE ONLY.

Follows the reference's significance.py:

    count_hits             significance.py:31-42   per-Gaussian ray hits summed over views
    significance_scores    significance.py:45-78   hits * alpha_hat * min(V / V90, 1) ** power,
                                                   V = 4/3 pi prod(masked scales), V90 the
                                                   nearest-rank 90th percentile (0 -> V > 0)
    prune_keep             significance.py:81-99   drop the floor(rate N) lowest (score, index)
    prune_schedule         significance.py:100-104 first_rate * decay ** k

Pinned to the reference's own outputs by tests/golden/significance.npz
(tests/golden/make_golden.py: significance_golden) in tests/test_oracle_golden.py.
Only tests/ import this module.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

from . import oracle


def _expit(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def count_hits(fields, cams, settings) -> np.ndarray:
    """significance.py:31-42 on the float64 oracle renderer."""
    if not cams:
        raise ValueError("count_hits needs at least one camera")
    s = SimpleNamespace(**{k: getattr(settings, k) for k in (
        "lowpass_s", "active_sh_degree", "background", "tile_size", "near", "mask_threshold",
        "sh_mask_threshold", "compute_sh_rest_grads")}, record_hits=True)
    total = None
    for cam in cams:
        h = oracle.render_forward(fields, cam, s, "f64")["hit_counts"]
        total = h.copy() if total is None else total + h
    return total


def rank90(n: int) -> int:
    """Nearest-rank index of the 90th percentile (significance.py:65)."""
    return max(int(np.ceil(0.9 * n)) - 1, 0)


def significance_scores(hits, fields, mask_threshold: float, volume_power: float = 0.5) -> dict:
    """significance.py:45-78 in float64: masks = sigmoid(m) > eps (masking.py:21-25),
    alpha_hat = sigmoid(o) M, masked scales e^ls M (masking.py:34-43)."""
    m = np.asarray(fields["mask_logits"], dtype=np.float64)
    n = m.shape[0]
    mask = (_expit(m) > mask_threshold).astype(np.float64)
    alphas = _expit(fields["opacity_logits"]) * mask
    scales = np.exp(np.asarray(fields["log_scales"], dtype=np.float64)) * mask[:, None]
    volumes = (4.0 / 3.0) * np.pi * scales.prod(axis=1)
    v90 = np.sort(volumes)[rank90(n)]
    if v90 > 0:
        v_norm = np.minimum(volumes / v90, 1.0) ** volume_power
    else:
        v_norm = (volumes > 0).astype(np.float64)
    scores = np.asarray(hits).astype(np.float64) * alphas * v_norm
    return dict(volumes=volumes, v_norm=v_norm, scores=scores, v90=v90)


def prune_keep(scores, rate: float) -> np.ndarray:
    """significance.py:81-99: kept row indices (ascending) after dropping the
    floor(rate N) lowest scores, ties pruned from the lower index first."""
    if not 0.0 < rate < 1.0:
        raise ValueError("prune rate must lie in (0, 1)")
    scores = np.asarray(scores)
    n = scores.shape[0]
    k = int(math.floor(rate * n))
    if k >= n:
        raise ValueError("significance pruning would remove every Gaussian")
    if k == 0:
        return np.arange(n)
    order = np.lexsort((np.arange(n), scores))
    return np.sort(order[k:])


def prune_schedule(event_index: int, first_rate: float, decay: float) -> float:
    """significance.py:100-104."""
    if event_index < 0:
        raise ValueError("event index must be >= 0")
    return first_rate * decay ** event_index
