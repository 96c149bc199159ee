"""How much of the c3 training step is binning?  Times the pipelined step as is, then
with every view's tile lists replayed from the first step (binning skipped; results
are NOT valid training, this only measures the step without the binning kernels).
Usage: PYTHONPATH=. python profiles/binning_cost_exp.py"""

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, rasterizer, scenes
from paper_2501_14534_b200 import train as train_mod
from paper_2501_14534_b200.train import Trainer

sc = scenes.config3(views=8)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
targets = [torch.from_numpy(t).cuda() for t in sc.targets]
tr = Trainer(cloud, sc.cameras, targets, st)
for f in list(tr.opt.lrs):  # a static scene: cached tile lists stay exact (same work every step)
    tr.opt.set_lr(f, 0.0)


def timed(k=10):
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        tr.step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


base = timed()
cache = {}
orig_begin, orig_end = rasterizer._bin_begin, rasterizer._bin_end


def begin(splats, tiles, n, w, h, ts, rb, re, err=None, keys=None, cs=None):
    key = (w, h, len(cache) % 8)
    return ("cached", key) if key in cache else (key, orig_begin(splats, tiles, n, w, h, ts, rb, re, err, keys, cs))


def end(p):
    if p[0] == "cached":
        cache["_n"] = cache.get("_n", 0) + 1
        return cache[p[1]]
    bins = orig_end(p[1])
    cache[p[0]] = bins
    return bins


# one view per key slot: the Trainer binds views in order, so slot = view index
counter = {"i": 0}


def begin_slot(*a, **k):
    i = counter["i"] % 8
    counter["i"] += 1
    key = ("v", i)
    if key in cache:
        return ("cached", key)
    return (key, orig_begin(*a, **k))


train_mod._bin_begin = begin_slot
train_mod._bin_end = end
no_bin = timed()
print(f"c3 step: {base:.3f} ms with binning, {no_bin:.3f} ms with cached tile lists "
      f"-> binning costs {base - no_bin:.3f} ms of the step ({100 * (base - no_bin) / base:.1f}%)")
