"""Blend backward with the forward's exception lists vs re-resolving bracket pairs in
float64, on one c3 view (training-loss upstream gradient): per-launch time (CUDA events),
exception / overflow-tile counts, and the max partials difference.

    python profiles/exc_ab.py            (ncu: add --ncu to run each variant once)"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, loss, rasterizer, scenes

sc = scenes.config3()
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
once = "--ncu" in sys.argv
res = {}
for v in range(2 if once else len(sc.cameras)):
    cam = sc.cameras[v]
    out = rasterizer.render_forward(cloud, cam, st)
    _, d = loss.l1_ssim(out.image, torch.from_numpy(sc.targets[v]).cuda())
    s = out._state
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    ovf = s.exc_overflow.cpu().numpy().view(np.uint32)
    plain = dataclasses.replace(out, _state=dataclasses.replace(s, exceptions=None, exc_overflow=None))
    ds = {}
    times = {}
    for name, o in (("exceptions", out), ("float64", plain)):
        ds[name] = torch.zeros((len(cloud), 9), device="cuda")
        reps = 1 if once else 20
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        rasterizer.blend_backward(cloud, cam, st, d, o, dsplats=ds[name])
        ds[name].zero_()
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(reps):
            rasterizer.blend_backward(cloud, cam, st, d, o, dsplats=ds[name])
        ev[1].record()
        torch.cuda.synchronize()
        times[name] = ev[0].elapsed_time(ev[1]) / reps
    a, b = ds["exceptions"].cpu().numpy(), ds["float64"].cpu().numpy()
    res[v] = {"ms_exceptions": times["exceptions"], "ms_float64": times["float64"],
              "pixels_with_exception": int((s.exceptions > 0).sum()), "overflow_tiles": int(ovf[0]),
              "tiles": nt, "max_rel_diff": float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))}
print(json.dumps(res, indent=1))
