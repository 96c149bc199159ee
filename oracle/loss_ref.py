"""float64 restatement of the reference loss image terms — TEST INFRASTRUCTURE ONLY.

Follows training.total_loss (training.py:76-89) and metrics.ssim_fast
(metrics.py:120-188): separable 11-tap sigma-1.5 window over the symmetric-
padded image, analytic gradient with the padded border folded back onto its
source pixels.  Used by tests and by bench.py's CPU baseline / reference arm.
"""

from __future__ import annotations

import numpy as np
from scipy.ndimage import correlate1d


def _taps(size=11, sigma=1.5):
    x = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    t = np.exp(-0.5 * (x / sigma) ** 2)
    return t / t.sum()


def _win(p, taps, r):  # metrics.py:120-123
    return correlate1d(correlate1d(p, taps, axis=0, mode="constant"), taps, axis=1, mode="constant")[r:-r, r:-r]


def _adj(u, taps, idx, r):  # metrics.py:126-135
    h, w = u.shape
    c = np.zeros((h + 2 * r, w + 2 * r))
    c[r:r + h, r:r + w] = u
    c = correlate1d(correlate1d(c, taps, axis=0, mode="constant"), taps, axis=1, mode="constant")
    out = np.zeros(h * w)
    np.add.at(out, idx.ravel(), c.ravel())
    return out.reshape(h, w)


def ssim_and_grad(a, b, k1=0.01, k2=0.03):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    taps, r = _taps(), 5
    h, w, ch = a.shape
    idx = np.pad(np.arange(h * w).reshape(h, w), r, mode="symmetric")
    c1, c2 = k1 * k1, k2 * k2
    inv = 1.0 / (h * w * ch)
    total, grad = 0.0, np.zeros_like(a)
    for c in range(ch):
        ac, bc = a[:, :, c], b[:, :, c]
        ap, bp = ac.ravel()[idx], bc.ravel()[idx]
        mu_a, mu_b = _win(ap, taps, r), _win(bp, taps, r)
        saa, sbb, sab = _win(ap * ap, taps, r), _win(bp * bp, taps, r), _win(ap * bp, taps, r)
        a1, a2 = 2 * mu_a * mu_b + c1, 2 * (sab - mu_a * mu_b) + c2
        b1, b2 = mu_a ** 2 + mu_b ** 2 + c1, (saa - mu_a ** 2) + (sbb - mu_b ** 2) + c2
        smap = a1 * a2 / (b1 * b2)
        total += smap.sum() * inv
        den = b1 * b2
        d_mu = 2 * mu_b * (a2 - a1) / den - 2 * mu_a * smap * (1.0 / b1 - 1.0 / b2)
        grad[:, :, c] = (_adj(d_mu, taps, idx, r) + 2 * ac * _adj(-smap / b2, taps, idx, r)
                         + bc * _adj(2 * a1 / den, taps, idx, r)) * inv
    return total, grad


def total_loss_image(render, target, lam=0.2):
    """(l1, d_ssim, dL/drender) of training.total_loss's image terms."""
    diff = np.asarray(render, np.float64) - np.asarray(target, np.float64)
    l1 = float(np.abs(diff).mean())
    s, g = ssim_and_grad(render, target)
    return l1, (1.0 - s) / 2.0, (1.0 - lam) * np.sign(diff) / diff.size - lam * 0.5 * g
