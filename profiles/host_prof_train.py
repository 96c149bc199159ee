"""cProfile of the host side of Trainer.step on a small scene (host-bound):
PYTHONPATH=. python profiles/host_prof_train.py"""
import cProfile
import pstats

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer

sc = scenes.config3(n=50_000, views=8, width=240, height=135)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
tr = Trainer(cloud, sc.cameras, targets, st)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    tr.step()
b.record()
torch.cuda.synchronize()
print(f"{a.elapsed_time(b) / 20:.3f} ms per step (host-bound scene)")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    tr.step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
