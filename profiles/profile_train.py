"""Two c3 training steps (8 views) through train.Trainer — the command profiled by
`ncu -k regex:<kernel>` for the per-step kernels (preprocess backward, Adam)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
sc = scenes.config3(n=n, views=8)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
tr = Trainer(cloud, sc.cameras, targets, st)
for _ in range(2):
    tr.step()
torch.cuda.synchronize()
print("ok", tr.terms.sum().item())
