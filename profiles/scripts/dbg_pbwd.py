"""Debug: GPU preprocess backward vs the float64 oracle's on the SAME screen-space partials."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2501_14534_b200 as tgs
from paper_2501_14534_b200 import scenes
from paper_2501_14534_b200.rasterizer import blend_backward, preprocess_backward_views
from oracle import oracle
v = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sc = scenes.config3()
st = tgs.RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = tgs.GaussianCloud.from_fields(sc.fields)
cam = sc.cameras[v]
out = tgs.render_forward(cloud, cam, st)
d = np.random.default_rng(1).standard_normal((cam.height, cam.width, 3))
ds, state = blend_backward(cloud, cam, st, torch.from_numpy(d.astype(np.float32)).cuda(), out)
g = preprocess_backward_views(cloud, [cam], st, [state.visible_u8], [ds], tgs.CloudGrads.zeros(len(cloud)))
ref = oracle.preprocess_backward(sc.fields, cam, st, ds.cpu().numpy().astype(np.float64), "f64")
res = {}
for f in ("positions", "log_scales", "rotations", "opacity_logits", "sh_dc", "mask_logits", "mean2d_screen"):
    a = getattr(g, f).cpu().numpy().astype(np.float64).reshape(len(cloud), -1)
    b = ref[f].reshape(len(cloud), -1)
    e = np.abs(a - b).max(1)
    worst = np.argsort(-e)[:5]
    res[f] = {"rel": float(np.linalg.norm(a - b) / np.linalg.norm(b)),
              "worst": [{"row": int(r), "gpu": a[r].tolist(), "ref": b[r].tolist(),
                         "pos": sc.fields["positions"][r].tolist(), "ls": sc.fields["log_scales"][r].tolist(),
                         "rot": sc.fields["rotations"][r].tolist(), "vis": int(state.visible_u8[r]),
                         "ds": ds[r].tolist(), "splat": state.splats[r].tolist()} for r in worst]}
print(json.dumps(res, indent=1))
