"""How much of the c3 training step is binning?  Times the native pipelined step (static
scene: every learning rate 0, so the tile lists stay exact) with the stock library and
with an experiment build whose batch driver reuses the previous step's tile lists after
three batches (binning skipped; NOT valid training, it only measures the step without
the binning kernels).
    bash profiles/scripts/build_variant.sh skipbin driver.cu TGS_EXP_SKIP_BIN
    python profiles/binning_cost_exp.py            (stock)
    TGS_LIB=profiles/variants/libtgs_skipbin.so python profiles/binning_cost_exp.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer

sc = scenes.config3(views=8)
st = RenderSettings(**bench.settings_kwargs())
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
tr = Trainer(cloud, sc.cameras, targets, st, bench.LAMBDA_SSIM)
for f in list(tr.opt.lrs):
    tr.opt.set_lr(f, 0.0)
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k = 20
a.record()
for _ in range(k):
    tr.step()
b.record()
torch.cuda.synchronize()
tr.check_divergence()
print(f"{os.environ.get('TGS_LIB') or 'stock'}: c3 static-scene step {a.elapsed_time(b) / k:.3f} ms, "
      f"loss terms {tr.terms.sum().item():.6f}")
