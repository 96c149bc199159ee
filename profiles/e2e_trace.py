"""Where the end-to-end c3 step (targets H2D from pinned memory every step) loses time
against the device-resident step: a CUPTI trace (torch.profiler) of 3 steps of each,
with each target copy's completion time against the start of its view's loss.
    python profiles/e2e_trace.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.train import Trainer

sc = scenes.config3()
st = RenderSettings(**bench.settings_kwargs())
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
host = [torch.from_numpy(t).pin_memory() for t in sc.targets]
tr = Trainer(cloud, sc.cameras, targets, st, bench.LAMBDA_SSIM)
for _ in range(3):
    tr.step(host_targets=host)
torch.cuda.synchronize()
for label, fn in (("device", lambda: tr.step()), ("e2e", lambda: tr.step(host_targets=host))):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
    ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0)
    t0 = ev[0][0]
    span = ev[-1][1] - t0
    cp = [(s - t0, e - t0, n) for s, e, n in ev if "Memcpy" in n and "HtoD" in n]
    loss = [(s - t0, n) for s, e, n in ev if "k_ssim_fwd" in n]
    print(f"{label}: span {span / 3:.0f} us/step; {len(cp)} H2D copies; first 8: " +
          ", ".join(f"[{a:.0f}-{b:.0f}]" for a, b, _ in cp[:8]))
    print("   ssim_fwd starts (first 8): " + ", ".join(f"{a:.0f}" for a, _ in loss[:8]))
    seen = set()
    for s_, e_, n in ev:
        k = n.split("(")[0].replace("void ", "")[:40]
        if k not in seen and (s_ - t0) < 3000:
            seen.add(k)
            print(f"   first {k:40s} {s_ - t0:8.0f} - {e_ - t0:8.0f}")
