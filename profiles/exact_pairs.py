"""How many (pixel, splat) pairs the blend kernels decide in float64 (the exact-decision
cold path) at c3: one view's forward + backward with a -DTGS_COUNT_EXACT build.

    TGS_LIB=profiles/variants/libtgs_count.so python profiles/exact_pairs.py
Build: see profiles/scripts/build_count_variant.sh."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, _lib, loss, render_backward, render_forward, scenes

lib = _lib.load()
sc = scenes.config3()
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
res = {}
for v in range(len(sc.cameras)):
    cam = sc.cameras[v]
    cnt = ctypes.c_ulonglong(0)
    lib.tgs_debug_exact_pairs(None, 1)
    out = render_forward(cloud, cam, st)
    torch.cuda.synchronize()
    lib.tgs_debug_exact_pairs(ctypes.byref(cnt), 1)
    fwd = cnt.value
    _, d = loss.l1_ssim(out.image, torch.from_numpy(sc.targets[v]).cuda())
    render_backward(cloud, cam, st, d, out)
    torch.cuda.synchronize()
    lib.tgs_debug_exact_pairs(ctypes.byref(cnt), 1)
    pairs = int(out.last_pos.to(torch.int64).sum())
    res[v] = {"forward_exact_pairs": fwd, "backward_exact_pairs": cnt.value, "pairs_walked": pairs,
              "fraction": fwd / max(pairs, 1)}
print(json.dumps(res, indent=1))
