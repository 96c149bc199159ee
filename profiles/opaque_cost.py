"""Cost of exact decisions on opaque scenes: one c3 view's blend forward / backward with the
stock opacities (N(0,1) logits) and with every logit +6 (alpha ~0.997, above the 0.99
clamp: trained scenes saturate), exact decisions vs float32 (TGS_EXACT=0 in a subprocess).
    python profiles/opaque_cost.py"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch

    import bench
    from paper_2501_14534_b200 import GaussianCloud, RenderSettings, loss, rasterizer, scenes
    shift = float(sys.argv[2])
    sc = scenes.config3()
    f = dict(sc.fields)
    f["opacity_logits"] = (f["opacity_logits"] + shift).astype("float32")
    st = RenderSettings(**bench.settings_kwargs())
    cloud = GaussianCloud.from_fields(f)
    cam = sc.cameras[0]
    tgt = torch.from_numpy(sc.targets[0]).cuda()
    out = rasterizer.render_forward(cloud, cam, st)
    _, d = loss.l1_ssim(out.image, tgt)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ds = torch.zeros((len(cloud), 9), device="cuda")
    for _ in range(2):
        out = rasterizer.render_forward(cloud, cam, st)
        rasterizer.blend_backward(cloud, cam, st, d, out, dsplats=ds)
    torch.cuda.synchronize()
    tf = tb = 0.0
    for _ in range(5):
        pre = rasterizer.preprocess(cloud, cam, st)
        bins = rasterizer._bin(pre[0], pre[2], len(cloud), cam.width, cam.height, 16, 0,
                               rasterizer._tiles_y(cam, 16), pre[4], pre[3])
        torch.cuda.synchronize()
        ev[0].record()
        out = rasterizer.render_forward(cloud, cam, st, pre=pre, bins=bins)
        ev[1].record()
        rasterizer.blend_backward(cloud, cam, st, d, out, dsplats=ds)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1]) / 5
        tb += ev[1].elapsed_time(ev[2]) / 5
    s = out._state
    flagged = int(s.exc_overflow[0].item()) if s.exc_overflow is not None else None
    print(json.dumps({"shift": shift, "exact": rasterizer.EXACT_DECISIONS, "ms_forward": round(tf, 4),
                      "ms_backward": round(tb, 4), "flagged_tiles": flagged}))
    sys.exit(0)
res = []
for shift in (0.0, 6.0):
    for exact in ("1", "0"):
        r = subprocess.run([sys.executable, __file__, "run", str(shift)], capture_output=True, text=True,
                           env={**os.environ, "TGS_EXACT": exact})
        res.append(r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:])
print("\n".join(res))
