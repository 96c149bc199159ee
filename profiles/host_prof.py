import cProfile, pstats, sys
import torch
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.rasterizer import render_views
sc = scenes.config3(views=8)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields({k: v[:2000] for k, v in sc.fields.items()})
for _ in range(5):
    render_views(cloud, sc.cameras, st)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    render_views(cloud, sc.cameras, st)
torch.cuda.synchronize()
pr.disable()
ps = pstats.Stats(pr).sort_stats("tottime")
ps.print_stats(28)
