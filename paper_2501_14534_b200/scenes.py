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


def config5_sfm(seed: int = 5, n: int = 1_000_000, n_gt: int = 50_000, width: int = 1920, height: int = 1080,
                views: int = 8) -> tuple[Scene, dict]:
    """c5 the way the reference builds its own training scenes (synthetic.py make_scene +
    schedule.py seed_from_sfm, restated): a ground-truth cloud of n_gt Gaussians on the
    radius-2 shell (opacities U(0.55, 0.95), colours U(0.2, 0.9), mild view dependence
    fading with band order) whose renders are the targets, and the TRAINED cloud seeded
    from n SfM-like points — noisy samples around ground-truth centres (offset N(0, 1) x
    the owner's scale x U(0.2, 2)) — with isotropic scales from the mean distance to the
    3 nearest seeds, identity rotations, opacity 0.1, the owner's colour (+ N(0, 0.02))
    and mask logits 2.0.  Returns (scene with the seed cloud, ground-truth fields)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    c0 = 0.28209479177387814  # SH band-0 constant: dc = (rgb - 0.5) / c0
    d = rng.normal(size=(n_gt, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    q = rng.normal(size=(n_gt, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    spacing = math.sqrt(4.0 * math.pi * 4.0 / n_gt)  # mean distance between shell centres
    ls = np.log(rng.uniform(0.5 * spacing, 1.5 * spacing, (n_gt, 3)))
    rgb = rng.uniform(0.2, 0.9, (n_gt, 3))
    rest = np.zeros((n_gt, 15, 3))
    rest[:, 0:3] = rng.normal(0.0, 0.08, (n_gt, 3, 3))
    rest[:, 3:8] = rng.normal(0.0, 0.04, (n_gt, 5, 3))
    rest[:, 8:15] = rng.normal(0.0, 0.02, (n_gt, 7, 3))
    op = rng.uniform(0.55, 0.95, n_gt)
    gt = {"positions": _f32(2.0 * d), "log_scales": _f32(ls), "rotations": _f32(q),
          "opacity_logits": _f32(np.log(op / (1.0 - op))), "sh_dc": _f32((rgb - 0.5) / c0), "sh_rest": _f32(rest),
          "mask_logits": _f32(np.full(n_gt, 2.0)), "sh_mask_logits": _f32(np.full((n_gt, 3), 2.0))}
    owner = rng.integers(0, n_gt, n)
    xyz = 2.0 * d[owner] + rng.normal(size=(n, 3)) * np.exp(ls[owner]) * rng.uniform(0.2, 2.0, (n, 1))
    dist, _ = cKDTree(xyz).query(xyz, k=4)
    mean_d = np.maximum(dist[:, 1:].mean(axis=1), 1e-7)
    prgb = np.clip(rgb[owner] + rng.normal(0.0, 0.02, (n, 3)), 0.0, 1.0)
    rot = np.zeros((n, 4))
    rot[:, 0] = 1.0
    fields = {"positions": _f32(xyz), "log_scales": _f32(np.log(mean_d)[:, None].repeat(3, axis=1)),
              "rotations": _f32(rot), "opacity_logits": _f32(np.full(n, math.log(0.1 / 0.9))),
              "sh_dc": _f32((prgb - 0.5) / c0), "sh_rest": _f32(np.zeros((n, 15, 3))),
              "mask_logits": _f32(np.full(n, 2.0)), "sh_mask_logits": _f32(np.full((n, 3), 2.0))}
    cams = [pinhole(rng.uniform(4.0, 6.0) * _unit(rng), width, height, name=f"c5v{k}") for k in range(views)]
    sc = Scene("c5", fields, cams, [], dict(near=0.2, tile_size=16, mask_threshold=0.01, sh_mask_threshold=0.1))
    return sc, gt


def small_scene(seed: int, n: int, width: int, height: int, dist: float = 4.0, **settings) -> Scene:
    """c1 distributions at a reduced size (parity tests)."""
    rng = np.random.default_rng(seed)
    fields = random_fields(rng, n)
    cam = pinhole(dist * _unit(rng), width, height, name="small")
    target = _f32(rng.uniform(0.0, 1.0, (height, width, 3)))
    s = dict(near=0.2, tile_size=16)
    s.update(settings)
    return Scene("small", fields, [cam], [target], s)
