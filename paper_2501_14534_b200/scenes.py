"""Seeded synthetic workloads c1..c5 (BASELINE.json `configs`).

The reference's headline numbers come from real datasets (Mip-NeRF 360 etc.)
that are not available here; these generators stand in for them with the
shapes, sizes and attribute distributions BASELINE.json states.  All values
are produced in float64 by numpy's PCG64 and rounded to float32 once, so the
CUDA path, the fp32 oracle and the fp64 reference (fed the same float32-valued
inputs) see identical parameters.

Config choices that BASELINE.json leaves open are pinned here and listed in
DESIGN.md ("Synthetic workloads"):
  * positions are radially clamped (scaled back onto the sphere), not dropped;
  * c2 clamps its N(0, 3) positions to radius 2 (the survey's choice);
  * fov 60 degrees is horizontal, fy = fx, principal point at the image centre
    with the integer-pixel-centre convention ((W-1)/2, (H-1)/2);
  * every camera looks at the origin with up = +z (cameras.look_at).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .cameras import Camera, look_at

PARAM_FIELDS = (
    "positions", "log_scales", "rotations", "opacity_logits",
    "sh_dc", "sh_rest", "mask_logits", "sh_mask_logits",
)
FIELD_SHAPES = {
    "positions": (3,), "log_scales": (3,), "rotations": (4,), "opacity_logits": (),
    "sh_dc": (3,), "sh_rest": (15, 3), "mask_logits": (), "sh_mask_logits": (3,),
}


@dataclass
class Scene:
    name: str
    fields: dict                      # PARAM_FIELDS -> float32 numpy arrays
    cameras: list                     # [Camera]
    targets: list = field(default_factory=list)   # float32 (H, W, 3) per camera
    settings: dict = field(default_factory=dict)  # RenderSettings kwargs

    @property
    def n(self) -> int:
        return int(self.fields["positions"].shape[0])


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


def _clamp_ball(p: np.ndarray, radius: float) -> np.ndarray:
    r = np.linalg.norm(p, axis=1, keepdims=True)
    return p * np.minimum(1.0, radius / np.maximum(r, 1e-30))


def random_fields(rng, n, pos_std=1.0, pos_radius=2.0, ls_mean=-4.0, ls_std=0.5, positions=None) -> dict:
    """Attribute distributions of BASELINE.json configs[0]."""
    pos = positions if positions is not None else _clamp_ball(rng.normal(0.0, pos_std, (n, 3)), pos_radius)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return {
        "positions": _f32(pos),
        "log_scales": _f32(rng.normal(ls_mean, ls_std, (n, 3))),
        "rotations": _f32(q),
        "opacity_logits": _f32(rng.normal(0.0, 1.0, n)),
        "sh_dc": _f32(rng.normal(0.5, 0.2, (n, 3))),
        "sh_rest": _f32(rng.normal(0.0, 0.05, (n, 15, 3))),
        "mask_logits": _f32(rng.normal(2.0, 1.0, n)),
        "sh_mask_logits": _f32(rng.normal(2.0, 1.0, (n, 3))),
    }


def pinhole(position, width, height, fov_deg=60.0, target=(0.0, 0.0, 0.0), name="") -> Camera:
    f = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    R, t = look_at(np.asarray(position, dtype=np.float64), np.asarray(target, dtype=np.float64))
    return Camera(fx=f, fy=f, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0, R=R, t=t,
                  width=width, height=height, name=name)


def _unit(rng):
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


def config1(seed: int = 1, n: int = 10_000, size: int = 256) -> Scene:
    """c1: CPU-runnable parity case, one 256x256 view, L1 against U[0,1]."""
    rng = np.random.default_rng(seed)
    fields = random_fields(rng, n)
    cam = pinhole(4.0 * _unit(rng), size, size, name="c1")
    target = _f32(rng.uniform(0.0, 1.0, (size, size, 3)))
    return Scene("c1", fields, [cam], [target], dict(near=0.2, tile_size=16))


def config2(seed: int = 2, n: int = 200_000, width: int = 1280, height: int = 720) -> Scene:
    """c2: forward + binning at 720p, positions N(0,3) clamped to radius 2."""
    rng = np.random.default_rng(seed)
    fields = random_fields(rng, n, pos_std=3.0, pos_radius=2.0, ls_mean=-4.5, ls_std=0.7)
    cam = pinhole(4.0 * _unit(rng), width, height, name="c2")
    return Scene("c2", fields, [cam], [], dict(near=0.2, tile_size=16))


def config3(seed: int = 3, n: int = 1_000_000, width: int = 1920, height: int = 1080, views: int = 8) -> Scene:
    """c3: the training-step workload, 8 views on a radius U(4,6) sphere."""
    rng = np.random.default_rng(seed)
    fields = random_fields(rng, n)
    cams, targets = [], []
    for k in range(views):
        cams.append(pinhole(rng.uniform(4.0, 6.0) * _unit(rng), width, height, name=f"c3v{k}"))
        targets.append(_f32(rng.uniform(0.0, 1.0, (height, width, 3))))
    return Scene("c3", fields, cams, targets,
                 dict(near=0.2, tile_size=16, mask_threshold=0.01, sh_mask_threshold=0.1))


def config4(seed: int = 4, n: int = 3_000_000, width: int = 3840, height: int = 2160, frames: int = 200,
            clusters: int = 64, radius: float = 10.0, orbit_radius: float = 16.0) -> Scene:
    """c4: render-only 4K orbit over 64 anisotropic clusters in a radius-10 scene."""
    rng = np.random.default_rng(seed)
    centers = _clamp_ball(rng.uniform(-radius, radius, (clusters, 3)), radius)
    which = rng.integers(0, clusters, n)
    std = rng.uniform(0.1, 1.0, (clusters, 3))
    q = rng.normal(size=(clusters, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    rot = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], 1)
    local = rng.normal(size=(n, 3)) * std[which]
    pos = centers[which] + np.einsum("nij,nj->ni", rot[which], local)
    fields = random_fields(rng, n, positions=_clamp_ball(pos, radius))
    cams = []
    for k in range(frames):
        th = 2.0 * math.pi * k / frames
        cams.append(pinhole((orbit_radius * math.cos(th), orbit_radius * math.sin(th), 0.3 * orbit_radius),
                            width, height, name=f"c4f{k}"))
    return Scene("c4", fields, cams, [], dict(near=0.2, tile_size=16))


def config5(seed: int = 5, n: int = 1_000_000, width: int = 1920, height: int = 1080, views: int = 8) -> Scene:
    """c5: the progressive-schedule sweep's scene — the c1 attribute distributions on a thin
    radius-2 shell (a surface, as reconstructed scenes concentrate their Gaussians on
    surfaces) rather than c3's solid ball, whose interior no camera sees: every row lies on
    a surface some of the 8 cameras (radius U(4, 6), as c3) look at.  log-scales
    N(-4.5, 0.3), so the shell is a few Gaussians thick."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pos = d * (2.0 + rng.normal(0.0, 0.01, (n, 1)))
    fields = random_fields(rng, n, ls_mean=-4.5, ls_std=0.3, positions=pos)
    cams = [pinhole(rng.uniform(4.0, 6.0) * _unit(rng), width, height, name=f"c5v{k}") for k in range(views)]
    return Scene("c5", fields, cams, [], dict(near=0.2, tile_size=16, mask_threshold=0.01, sh_mask_threshold=0.1))


def small_scene(seed: int, n: int, width: int, height: int, dist: float = 4.0, **settings) -> Scene:
    """c1 distributions at a reduced size (parity tests)."""
    rng = np.random.default_rng(seed)
    fields = random_fields(rng, n)
    cam = pinhole(dist * _unit(rng), width, height, name="small")
    target = _f32(rng.uniform(0.0, 1.0, (height, width, 3)))
    s = dict(near=0.2, tile_size=16)
    s.update(settings)
    return Scene("small", fields, [cam], [target], s)
