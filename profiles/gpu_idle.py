"""GPU busy/idle accounting of the c3 render batch and training step from a CUPTI
kernel trace (torch.profiler; nsys is not in the image).  Prints the wall span of
one batch, the union of kernel intervals (GPU busy), and the largest idle gaps.
Usage: PYTHONPATH=. python profiles/gpu_idle.py [render|train]"""

import sys

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.rasterizer import preprocess_views, render_forward
from paper_2501_14534_b200.train import Trainer

mode = sys.argv[1] if len(sys.argv) > 1 else "render"
sc = scenes.config3(views=8)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
dev = cloud.device
streams = [torch.cuda.Stream(device=dev) for _ in range(2)]

if mode == "render":
    from paper_2501_14534_b200.rasterizer import render_views

    def work():  # the batch API (native tgs_render_views once the counts are known)
        render_views(cloud, sc.cameras, st)
else:
    targets = [torch.from_numpy(t).to(dev) for t in sc.targets]
    tr = Trainer(cloud, sc.cameras, targets, st)
    work = tr.step

for _ in range(3):
    work()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        work()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev if "Memcpy" not in e.name and "Memset" not in e.name)
if not iv:
    print("no kernel events")
    sys.exit(0)
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
busy, cur_s, cur_e, gaps = 0.0, iv[0][0], iv[0][1], []
for s, e, name in iv[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, cur_e - t0, name))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = t1 - t0
print(f"{mode}: 3 batches, span {span:.0f} us, GPU busy (union of kernels) {busy:.0f} us = {100 * busy / span:.1f}%, "
      f"idle {span - busy:.0f} us in {len(gaps)} gaps")
gaps.sort(reverse=True)
for g, at, name in gaps[:12]:
    print(f"  gap {g:7.1f} us at +{at:8.0f} before {name[:60]}")
hist = {}
for g, _, _ in gaps:
    k = "<5" if g < 5 else "5-20" if g < 20 else "20-100" if g < 100 else ">=100"
    hist[k] = hist.get(k, 0.0) + g
print("  idle by gap size (us):", {k: round(v) for k, v in sorted(hist.items())})
