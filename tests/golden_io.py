"""Loaders for the committed golden fixtures (tests/golden/*.npz).

The fixtures were produced by the unmodified reference (tests/golden/make_golden.py);
this module only turns them back into (fields, camera, settings) triples.
"""

from __future__ import annotations

import hashlib
import os
from types import SimpleNamespace

import numpy as np

from paper_2501_14534_b200 import scenes
from paper_2501_14534_b200.cameras import Camera

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELDS = scenes.PARAM_FIELDS
CASES = ["loop24", "fd16", "dense32", "masked72x40", "deg1_norest", "deg2_tile8", "kat_single", "kat_two",
         "kat_walls", "edges", "empty", "c1"]


def digest(fields) -> str:
    h = hashlib.sha256()
    for f in FIELDS:
        h.update(np.ascontiguousarray(np.asarray(fields[f], dtype=np.float32)).tobytes())
    return h.hexdigest()


def load(name: str):
    z = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    if "in_digest" in z:
        sc = {"c1": scenes.config1}[name]()
        fields = sc.fields
        assert digest(fields) == str(z["in_digest"]), "seeded generator no longer reproduces the fixture inputs"
    else:
        fields = {f: z[f"in_{f}"] for f in FIELDS}
    fx, fy, cx, cy = (float(v) for v in z["cam_intr"])
    w, h = (int(v) for v in z["cam_size"])
    cam = Camera(fx=fx, fy=fy, cx=cx, cy=cy, R=z["cam_R"], t=z["cam_t"], width=w, height=h)
    settings = SimpleNamespace(
        lowpass_s=float(z["set_lowpass"]), active_sh_degree=int(z["set_degree"]),
        background=tuple(float(v) for v in z["set_bg"]), tile_size=int(z["set_tile"]), near=float(z["set_near"]),
        record_hits=bool(int(z["set_hits"])), mask_threshold=float(z["set_mask"]),
        sh_mask_threshold=float(z["set_shmask"]), compute_sh_rest_grads=bool(int(z["set_rest"])),
    )
    return SimpleNamespace(name=name, fields=fields, cam=cam, settings=settings, z=z)


def load_significance():
    """tests/golden/significance.npz: two scenes ("a": regular, "z": v90 == 0) with
    three cameras each, the reference's hits / volumes / v_norm / scores / kept rows."""
    z = dict(np.load(os.path.join(GOLDEN, "significance.npz")))
    out = {}
    for tag in ("a", "z"):
        fields = {f: z[f"{tag}_in_{f}"] for f in FIELDS}
        cams = []
        for k in range(z[f"{tag}_cam_intr"].shape[0]):
            fx, fy, cx, cy = (float(v) for v in z[f"{tag}_cam_intr"][k])
            w, h = (int(v) for v in z[f"{tag}_cam_size"][k])
            cams.append(Camera(fx=fx, fy=fy, cx=cx, cy=cy, R=z[f"{tag}_cam_R"][k], t=z[f"{tag}_cam_t"][k],
                               width=w, height=h))
        settings = SimpleNamespace(lowpass_s=0.3, active_sh_degree=3, background=(0.0, 0.0, 0.0), tile_size=16,
                                   near=0.2, record_hits=True, mask_threshold=float(z["mask_threshold"]),
                                   sh_mask_threshold=0.1, compute_sh_rest_grads=True)
        out[tag] = SimpleNamespace(fields=fields, cams=cams, settings=settings,
                                   **{k: z[f"{tag}_{k}"] for k in ("hits", "volumes", "v_norm", "scores", "keep")})
    return out, z
