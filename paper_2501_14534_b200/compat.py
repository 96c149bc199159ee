"""numpy-in / numpy-out adaptor with the reference's exact conventions.

Lets the reference's own call sites (`training.py:296,309,430`,
`significance.py:40`, `synthetic.py:115`, `cli.py:135-248`) run on the B200
path unchanged:

    import slimsplat.rasterizer as R, slimsplat.training as T
    from paper_2501_14534_b200 import compat
    R.render_forward = T.render_forward = compat.render_forward
    R.render_backward = T.render_backward = compat.render_backward
    R.bin_tiles = compat.bin_tiles

Inputs are the reference's float64 numpy objects (any object with the
GaussianCloud / Camera / RenderSettings attribute names); outputs are float64
numpy arrays with the reference's shapes, and `RenderOutput._tiles.indices`
index the compacted visible subset exactly like `bin_tiles` does in
`_prepare` (rasterizer.py:177-200).  Each call uploads the cloud and downloads
the results — the host<->device cost of a literal drop-in; a training loop
that keeps the cloud on the GPU should use the tensor API (rasterizer.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import rasterizer as _r
from .cloud import GaussianCloud

FIELDS = ("positions", "log_scales", "rotations", "opacity_logits", "sh_dc", "sh_rest", "mask_logits",
          "sh_mask_logits")


@dataclass
class TileBinsNP:
    offsets: np.ndarray
    indices: np.ndarray
    tiles_x: int
    tiles_y: int


@dataclass
class RenderOutputNP:
    image: np.ndarray
    transmittance: np.ndarray
    weight_sum: np.ndarray
    n_contrib: np.ndarray
    last_pos: np.ndarray
    visible: np.ndarray
    screen_areas: np.ndarray
    hit_counts: np.ndarray | None = None
    hit_records: list | None = None
    _tiles: TileBinsNP | None = field(default=None, repr=False)
    _device: object = field(default=None, repr=False)


@dataclass
class CloudGradsNP:
    positions: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    opacity_logits: np.ndarray
    sh_dc: np.ndarray
    sh_rest: np.ndarray
    mask_logits: np.ndarray
    sh_mask_logits: np.ndarray
    mean2d_screen: np.ndarray

    def finite(self) -> bool:
        return all(np.isfinite(getattr(self, f)).all() for f in self.__dataclass_fields__)


def _settings(s) -> _r.RenderSettings:
    d = _r.RenderSettings()
    return _r.RenderSettings(**{k: getattr(s, k, getattr(d, k)) for k in _r.RenderSettings.__dataclass_fields__})


def _np64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _upload(cloud) -> GaussianCloud:
    return GaussianCloud.from_fields({f: np.asarray(getattr(cloud, f)) for f in FIELDS})


def render_forward(cloud, cam, settings) -> RenderOutputNP:
    dev_cloud = _upload(cloud)
    out = _r.render_forward(dev_cloud, cam, _settings(settings))
    vis = out.visible.cpu().numpy()
    # reference TileBins index the compacted visible set (rasterizer.py:177-188)
    remap = np.cumsum(vis) - 1
    ids = out._tiles.indices.cpu().numpy().astype(np.int64)
    bins = TileBinsNP(out._tiles.offsets.cpu().numpy().astype(np.int64), remap[ids], out._tiles.tiles_x,
                      out._tiles.tiles_y)
    return RenderOutputNP(
        image=_np64(out.image), transmittance=_np64(out.transmittance), weight_sum=_np64(out.weight_sum),
        n_contrib=out.n_contrib.cpu().numpy(), last_pos=out.last_pos.cpu().numpy(), visible=vis,
        screen_areas=_np64(out.screen_areas),
        hit_counts=out.hit_counts.cpu().numpy() if out.hit_counts is not None else None,
        hit_records=out.hit_records, _tiles=bins, _device=(dev_cloud, out))


def render_backward(cloud, cam, settings, dimage, output) -> CloudGradsNP:
    from .errors import ContractViolationError
    if output is None or output.transmittance is None or output.last_pos is None:
        raise ContractViolationError("render_backward needs the forward pass auxiliaries")
    if getattr(output, "_device", None) is not None:
        dev_cloud, dev_out = output._device
    else:  # an output built elsewhere: recompute the device state from the host aux
        dev_cloud = _upload(cloud)
        dev_out = _r.RenderOutput(image=None, transmittance=torch.from_numpy(np.asarray(output.transmittance)),
                                  weight_sum=None, n_contrib=None,
                                  last_pos=torch.from_numpy(np.asarray(output.last_pos)), visible=None,
                                  screen_areas=None)
    g = _r.render_backward(dev_cloud, cam, _settings(settings), np.asarray(dimage), dev_out)
    return CloudGradsNP(**{f: _np64(getattr(g, f)) for f in FIELDS + ("mean2d_screen",)})


def bin_tiles(means2d, radii, depths, width, height, tile_size) -> TileBinsNP:
    b = _r.bin_tiles(np.asarray(means2d), np.asarray(radii), np.asarray(depths), width, height, tile_size)
    return TileBinsNP(b.offsets.cpu().numpy().astype(np.int64), b.indices.cpu().numpy().astype(np.int64),
                      b.tiles_x, b.tiles_y)
