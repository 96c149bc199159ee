"""Debug: c3 view 4, GPU blend-backward partials vs the float64 oracle's, per column."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2501_14534_b200 as tgs
from paper_2501_14534_b200 import scenes
from paper_2501_14534_b200.rasterizer import blend_backward
from oracle import oracle
v = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sc = scenes.config3()
st = tgs.RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = tgs.GaussianCloud.from_fields(sc.fields)
cam = sc.cameras[v]
out = tgs.render_forward(cloud, cam, st)
if len(sys.argv) > 2 and sys.argv[2] == "loss":
    from paper_2501_14534_b200 import loss
    _, dt = loss.l1_ssim(out.image, torch.from_numpy(sc.targets[v]).cuda(), 0.2)
    d = dt.cpu().numpy().astype(np.float64)
else:
    d = np.random.default_rng(1).standard_normal((cam.height, cam.width, 3))
ds, state = blend_backward(cloud, cam, st, torch.from_numpy(d.astype(np.float32)).cuda(), out)
ds = ds.cpu().numpy().astype(np.float64)
f = oracle.render_forward(sc.fields, cam, st, "f64")
ref = oracle.blend_backward(f["splats"], f["offsets"], f["ids"], cam.width, cam.height, 16, st.background,
                            f["transmittance"], f["last_pos"], d, "f64")
res = {"image_err": float(np.abs(out.image.cpu().numpy() - f["image"]).max()),
       "T_err": float(np.abs(out.transmittance.cpu().numpy() - f["transmittance"]).max()),
       "lastpos_mismatch": int((out.last_pos.cpu().numpy() != f["last_pos"]).sum())}
err = np.abs(ds - ref)
res["col_rel"] = [float(np.linalg.norm(ds[:, k] - ref[:, k]) / max(np.linalg.norm(ref[:, k]), 1e-30)) for k in range(9)]
rel_row = err[:, :6].max(1) / (np.abs(ref[:, :6]).max(1) + 1e-30)
rows = np.argsort(-err[:, :6].max(1))[:6]
sp = state.splats.cpu().numpy()
res["worst"] = [{"row": int(r), "gpu": ds[r].tolist(), "ref": ref[r].tolist(), "splat": sp[r].tolist()} for r in rows]
# rows with large relative error
bad = err[:, 0] > 1e-3 * np.abs(ref[:, 0]) + 1e-5
res["bad_rows"] = int(bad.sum())
res["dimage_absmax"] = float(np.abs(d).max())
res["ref_col_norm"] = [float(np.linalg.norm(ref[:, k])) for k in range(9)]
res["gpu_col_norm"] = [float(np.linalg.norm(ds[:, k])) for k in range(9)]
res["bad_radius_stats"] = [float(np.percentile(sp[bad, 10], q)) for q in (0, 50, 100)] if bad.any() else None
res["all_radius_stats"] = [float(np.percentile(sp[:, 10], q)) for q in (0, 50, 99, 100)]
print(json.dumps(res, indent=1))
