"""cProfile of the literal drop-in (compat.py) for one c3 view iteration: where the host
time of render_forward + render_backward with float64 numpy in / out goes.
    python profiles/compat_prof.py"""
import cProfile
import os
import pstats
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import bench
from paper_2501_14534_b200 import RenderSettings, compat, scenes

sc = scenes.config3()
st = RenderSettings(**bench.settings_kwargs())
cloud64 = types.SimpleNamespace(**{k: np.asarray(v, dtype=np.float64) for k, v in sc.fields.items()})
cam = sc.cameras[0]
dimg = np.random.default_rng(0).standard_normal((cam.height, cam.width, 3))
for _ in range(2):
    compat.render_backward(cloud64, cam, st, dimg, compat.render_forward(cloud64, cam, st))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    out = compat.render_forward(cloud64, cam, st)
    compat.render_backward(cloud64, cam, st, dimg, out)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
