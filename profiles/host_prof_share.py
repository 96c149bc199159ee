"""Host side of rank 0's 1-view share of an 8-rank step (Trainer(views=[0], zero_sim=(0, 8))):
wall vs device time per step and a cProfile of the host work.
    python profiles/host_prof_share.py [zero|gaussians]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer

sc = scenes.config3()
st = RenderSettings(**bench.settings_kwargs())
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(sc.targets[0]).cuda()] + [None] * 7
mode = sys.argv[1] if len(sys.argv) > 1 else "zero"
kw = (dict(dp_mode="gaussians", gshard_sim=(0, 8), all_views=[[d] for d in range(8)]) if mode == "gaussians"
      else dict(zero_sim=(0, 8)))
tr = Trainer(cloud, sc.cameras, targets, st, bench.LAMBDA_SSIM, views=[0], **kw)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for _ in range(20):
    tr.step()
b.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 20 * 1e3
print(f"device {a.elapsed_time(b) / 20:.3f} ms/step, wall {wall:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    tr.step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
