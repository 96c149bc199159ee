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
the results — the host<->device cost of a literal drop-in (bench.py
`compat_drop_in`); a training loop that keeps the cloud on the GPU should use the
tensor API (rasterizer.py, train.Trainer).  The float64 <-> float32 conversions run
on the GPU (the copies carry float64), the tile lists are remapped only when read.
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
    _tiles_np: TileBinsNP | None = field(default=None, repr=False)
    _device: object = field(default=None, repr=False)

    @property
    def _tiles(self) -> TileBinsNP | None:
        """The reference's TileBins (rasterizer.py:177-200), made on first access: the
        device lists' ids remapped to the compacted visible subset."""
        if self._tiles_np is None and self._device is not None:
            out = self._device[1]
            remap = np.cumsum(self.visible) - 1
            ids = out._tiles.indices.cpu().numpy()
            self._tiles_np = TileBinsNP(out._tiles.offsets.cpu().numpy().astype(np.int64), remap[ids],
                                        out._tiles.tiles_x, out._tiles.tiles_y)
        return self._tiles_np


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


def _host(tensors: dict) -> dict:
    """Device tensors to numpy, float32 ones widened to float64 on the GPU, through pinned
    blocks of torch's caching host allocator (a pageable .cpu() of the ~0.5 GB of gradients
    ran at ~2 GB/s): every copy is issued, then one synchronisation.  The returned arrays
    own their pinned blocks, which return to the allocator's cache when released."""
    out = {}
    for k, t in tensors.items():
        if t is None:
            out[k] = None
            continue
        src = t.detach()
        if src.dtype == torch.float32:
            src = src.double()
        buf = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
        buf.copy_(src, non_blocking=True)
        out[k] = buf
    torch.cuda.current_stream().synchronize()
    return {k: (v.numpy() if v is not None else None) for k, v in out.items()}


def _upload(cloud) -> GaussianCloud:
    """The reference cloud's float64 fields copied as they are and rounded to float32 on
    the GPU, into the flat parameter buffer."""
    arrs = {f: np.asarray(getattr(cloud, f)) for f in FIELDS}
    n = int(arrs["positions"].shape[0])
    dev = GaussianCloud(n, "cuda")
    for f in FIELDS:
        dst = getattr(dev, f)
        src = torch.from_numpy(np.ascontiguousarray(arrs[f])).to(dst.device)
        if tuple(src.shape) != tuple(dst.shape):
            from .errors import ContractViolationError
            raise ContractViolationError(f"field {f} has shape {tuple(src.shape)}, expected {tuple(dst.shape)}")
        dst.copy_(src)
    return dev


def render_forward(cloud, cam, settings) -> RenderOutputNP:
    dev_cloud = _upload(cloud)
    out = _r.render_forward(dev_cloud, cam, _settings(settings))
    h = _host(dict(image=out.image, transmittance=out.transmittance, weight_sum=out.weight_sum,
                   n_contrib=out.n_contrib, last_pos=out.last_pos, visible=out.visible, screen_areas=out.screen_areas,
                   hit_counts=out.hit_counts))
    # the reference TileBins (indexing the compacted visible set, rasterizer.py:177-188)
    # are made from the device lists on first access (RenderOutputNP._tiles)
    return RenderOutputNP(**h, hit_records=out.hit_records, _device=(dev_cloud, out))


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
    flat = _host({"g": g.flat})["g"]  # one transfer of every field (widened on the GPU), then views
    out = {}
    for f in FIELDS + ("mean2d_screen",):
        o, size = g._layout_map[f]
        out[f] = flat[o:o + size].reshape(tuple(getattr(g, f).shape))
    return CloudGradsNP(**out)


def bin_tiles(means2d, radii, depths, width, height, tile_size) -> TileBinsNP:
    b = _r.bin_tiles(np.asarray(means2d), np.asarray(radii), np.asarray(depths), width, height, tile_size)
    return TileBinsNP(b.offsets.cpu().numpy().astype(np.int64), b.indices.cpu().numpy().astype(np.int64),
                      b.tiles_x, b.tiles_y)
