"""A few c4 frames (3M Gaussians, 4K) through render_forward — the command profiled by
`ncu -k regex:k_blend_fwd16w` for the 4K forward blend."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, render_forward, scenes

sc = scenes.config4()
cloud = GaussianCloud.from_fields(sc.fields)
st = RenderSettings(near=0.2, tile_size=16)
for k in range(3):
    render_forward(cloud, sc.cameras[20 + k], st)
torch.cuda.synchronize()
print("ok")
