"""Training-step throughput vs the number of view streams in train.Trainer (c3)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer
sc = scenes.config3(views=8)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
base = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
for ns in (1, 2, 3, 4, 6, 8):
    cloud = GaussianCloud.from_fields(sc.fields)
    tr = Trainer(cloud, sc.cameras, targets, st, streams=ns)
    for _ in range(3): tr.step()
    torch.cuda.synchronize()
    # reset params so the workload is comparable
    cloud.flat.copy_(base.flat); tr.opt.m.zero_(); tr.opt.v.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): tr.step()
    e.record(); torch.cuda.synchronize()
    print(ns, "streams:", round(5000.0 / s.elapsed_time(e), 2), "step/s")
