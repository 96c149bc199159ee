"""One c3 view forward + loss + backward after warm-up — the command profiled by
`ncu --set full -k regex:<kernel>` (profiles/README.md)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, loss, render_backward, render_forward, scenes

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
sc = scenes.config3(n=n, views=1)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
target = torch.from_numpy(sc.targets[0]).cuda()
for it in range(3):
    if it == 2:  # ncu --profile-from-start off captures the last (warm) iteration only
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    out = render_forward(cloud, sc.cameras[0], st)
    terms, d = loss.l1_ssim(out.image, target)
    g = render_backward(cloud, sc.cameras[0], st, d, out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", terms)
