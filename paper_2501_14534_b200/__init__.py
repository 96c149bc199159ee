"""B200-native Trick-GS rasterizer hot path (drop-in for slimsplat.rasterizer).

Public API mirrors the reference package's (`slimsplat/__init__.py:3-28`) for
the rasterizer path; the compute runs in libtgs.so (hand-written sm_100a CUDA,
include/tgs.h).  Importing the package does not touch the GPU.
"""

from .cameras import Camera, look_at
from .cloud import CloudGrads, GaussianCloud
from .errors import (ContractViolationError, DegenerateRotationError, DivergenceError, EmptySceneError,
                     NativeLibraryError, SingularCovarianceError, SlimsplatError)
from .rasterizer import (RenderOutput, RenderSettings, TileBins, bin_tiles, render_backward, render_forward,
                         render_views, sh_rest_update_step)

__version__ = "0.1.0"

__all__ = [
    "Camera", "CloudGrads", "GaussianCloud", "RenderOutput", "RenderSettings", "TileBins", "bin_tiles",
    "look_at", "render_backward", "render_forward", "render_views", "sh_rest_update_step", "SlimsplatError",
    "DegenerateRotationError", "SingularCovarianceError", "ContractViolationError", "EmptySceneError",
    "DivergenceError", "NativeLibraryError",
]
