"""Debug: per-view GPU render_backward vs the float64 oracle at c3, and the Trainer's
8-view gradient vs the sum of single-view GPU gradients."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
import paper_2501_14534_b200 as tgs
from paper_2501_14534_b200 import scenes, loss
from paper_2501_14534_b200.train import Trainer
from oracle import oracle
F = ("positions", "log_scales", "opacity_logits", "sh_dc", "mask_logits", "mean2d_screen")
sc = scenes.config3()
st = tgs.RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = tgs.GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
singles, dimgs = [], []
for v, cam in enumerate(sc.cameras):
    out = tgs.render_forward(cloud, cam, st)
    _, d = loss.l1_ssim(out.image, targets[v], 0.2)
    g = tgs.render_backward(cloud, cam, st, d, out)
    singles.append({f: getattr(g, f).cpu().numpy().astype(np.float64) for f in F})
    dimgs.append(d.cpu().numpy().astype(np.float64))
tr = Trainer(cloud, sc.cameras, targets, st, 0.2, lambda_m=0.0, lambda_sh=0.0, streams=int(sys.argv[1]) if len(sys.argv) > 1 else 4)
tr.step(); torch.cuda.synchronize()
rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
res = {"trainer_vs_sum_singles": {f: rel(tr.grads.__getattribute__(f).cpu().numpy().astype(np.float64), sum(s[f] for s in singles)) for f in F}}
def view64(v):
    f = oracle.render_forward(sc.fields, sc.cameras[v], st, "f64")
    return oracle.render_backward(sc.fields, sc.cameras[v], st, dimgs[v], f, "f64")
with ThreadPoolExecutor(8) as ex:
    parts = list(ex.map(view64, range(8)))
res["single_vs_oracle"] = {v: {f: rel(singles[v][f], parts[v][f]) for f in F} for v in range(8)}
p0 = view64(3)
res["oracle_thread_vs_serial_view3"] = {f: rel(parts[3][f], p0[f]) for f in F}
print(json.dumps(res, indent=1))
