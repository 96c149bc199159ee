"""Host latency at the start of a training step (the fixed-workload bench synchronizes
before every timed step, so the host's time to its first heavy launch is GPU idle inside
the step): host time of each phase of Trainer._step up to the views' driver call, and the
allocator's device-malloc count per step.
    python profiles/step_host_latency.py            (one GPU, the bench's 8-view step)
    python profiles/step_host_latency.py gaussians  (rank 0's share of an 8-rank Gaussian-sharded step)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, rasterizer, scenes
from paper_2501_14534_b200 import train as train_mod
from paper_2501_14534_b200.train import Trainer

sc = scenes.config3()
st = RenderSettings(**bench.settings_kwargs())
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
if len(sys.argv) > 1 and sys.argv[1] == "gaussians":
    tr = Trainer(cloud, sc.cameras, targets, st, bench.LAMBDA_SSIM, views=[0], dp_mode="gaussians",
                 gshard_sim=(0, 8), all_views=[[d] for d in range(8)])
else:
    tr = Trainer(cloud, sc.cameras, targets, st, bench.LAMBDA_SSIM)
for _ in range(4):
    tr.step()
torch.cuda.synchronize()
marks = []
orig_pv, orig_ex, orig_nat = train_mod.preprocess_views, train_mod.exact_records, Trainer._views_native


def pv(*a, **k):
    marks.append(("preprocess_views in", time.perf_counter()))
    r = orig_pv(*a, **k)
    marks.append(("preprocess_views out", time.perf_counter()))
    return r


def ex(*a, **k):
    r = orig_ex(*a, **k)
    marks.append(("exact_records out", time.perf_counter()))
    return r


def nat(self, *a, **k):
    marks.append(("views_native in", time.perf_counter()))
    r = orig_nat(self, *a, **k)
    marks.append(("views_native out", time.perf_counter()))
    return r


train_mod.preprocess_views, train_mod.exact_records, Trainer._views_native = pv, ex, nat
from paper_2501_14534_b200 import _lib
_L = _lib.load()
_orig_tv = _L.tgs_train_views


def tv(*a):
    marks.append(("driver call", time.perf_counter()))
    return _orig_tv(*a)


_L.tgs_train_views = tv
for it in range(5):
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    marks.clear()
    t0 = time.perf_counter()
    tr.step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    m1 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    print(f"step {it}: host {1e3 * (t1 - t0):.3f} ms, to idle {1e3 * (t2 - t0):.3f} ms, device mallocs {m1 - m0}; " +
          ", ".join(f"{k} {1e6 * (t - t0):.0f}us" for k, t in marks))
