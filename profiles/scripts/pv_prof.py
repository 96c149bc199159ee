import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes, _lib
from paper_2501_14534_b200.rasterizer import preprocess_views
sc = scenes.config3()
st = RenderSettings(**bench.settings_kwargs())
cloud = GaussianCloud.from_fields(sc.fields)
cache = {}
for _ in range(5): preprocess_views(cloud, sc.cameras, st, exact=False, cache=cache)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); preprocess_views(cloud, sc.cameras, st, exact=False, cache=cache); ts.append(time.perf_counter() - t0)
print("host us per call", sorted(ts)[25] * 1e6)
import ctypes
c_cloud, c_set = cloud.native(), _lib.make_settings(st)
c_cams = (_lib.TgsCamera * 8)(*[_lib.make_camera(c) for c in sc.cameras])
ent = list(cache.values())[0]
ptrs, err = ent[1], ent[2]
h = _lib.stream_handle(cloud.device)
fn = _lib.load().tgs_preprocess_forward_views
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(ctypes.byref(c_cloud), c_cams, ctypes.byref(c_set), 8, ptrs[0], ptrs[1], ptrs[2], ptrs[3], err.data_ptr(), None, None, h); ts.append(time.perf_counter() - t0)
print("raw C call us", sorted(ts)[25] * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    preprocess_views(cloud, sc.cameras, st, exact=False, cache=cache)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
