"""Where rank 0's share of an N-rank step goes (bench.py --rank-share N measures its total):
a CUPTI kernel trace (torch.profiler) of 4 share steps — per-kernel time per step, the
GPU-busy union and the idle gaps, and the host time per step.
Usage: python profiles/rank_share_trace.py [N] [zero|gaussians]"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sc = scenes.config3()
st = RenderSettings(**bench.settings_kwargs())
cloud = GaussianCloud.from_fields(sc.fields)
views = list(range(0, 8, N))
targets = [torch.from_numpy(t).cuda() if v in views else None for v, t in enumerate(sc.targets)]
mode = sys.argv[2] if len(sys.argv) > 2 else "zero"
kw = (dict(dp_mode="gaussians", gshard_sim=(0, N), all_views=[list(range(d, 8, N)) for d in range(N)])
      if mode == "gaussians" else dict(zero_sim=(0, N)))
tr = Trainer(cloud, sc.cameras, targets, st, bench.LAMBDA_SSIM, views=views, **kw)
for _ in range(3):
    tr.step()
torch.cuda.synchronize()
K = 4
host = []
for _ in range(K):  # host time of a step (enqueue only), GPU idle at its start
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.step()
    host.append((time.perf_counter() - t0) * 1e6)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(K):
        tr.step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
per = collections.defaultdict(float)
for s, e, n in iv:
    per[n.split("(")[0].replace("void ", "")[:60]] += (e - s) / K
busy, cs, ce, gaps = 0.0, iv[0][0], iv[0][1], []
for s, e, n in iv[1:]:
    if s > ce:
        busy += ce - cs
        gaps.append((s - ce, n[:50]))
        cs, ce = s, e
    else:
        ce = max(ce, e)
busy += ce - cs
span = iv[-1][1] - iv[0][0]
print(f"N={N} {mode} views {views}: span {span / K:.0f} us/step, busy {busy / K:.0f} us/step "
      f"({100 * busy / span:.1f}%), idle {(span - busy) / K:.0f} us/step; host enqueue {sorted(host)[K // 2]:.0f} us/step")
for k, v in sorted(per.items(), key=lambda x: -x[1])[:22]:
    print(f"  {v:8.1f} us/step  {k}")
gaps.sort(reverse=True)
for g, n in gaps[:8]:
    print(f"  gap {g:7.1f} us before {n}")
