"""Render-loop experiments: device time per frame for the per-view path and for
render_views (one multi-view preprocess pass + N-stream pipeline) at several batch
sizes.  Usage:
    PYTHONPATH=. python profiles/render_exp.py c3|c4 [frames]"""

import sys
import time

import torch

from paper_2501_14534_b200 import GaussianCloud, RenderSettings, scenes
from paper_2501_14534_b200.rasterizer import render_forward, render_views

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 48
if cfg == "c3":
    sc = scenes.config3(views=8)
    st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
else:
    sc = scenes.config4()
    st = RenderSettings(near=0.2, tile_size=16)
cams = sc.cameras
cloud = GaussianCloud.from_fields(sc.fields)
dev = cloud.device
pstreams = [torch.cuda.Stream(device=dev) for _ in range(2)]


def per_view(k0, count):
    main = torch.cuda.current_stream(dev)
    for s_ in pstreams:
        s_.wait_stream(main)
    for j in range(count):
        with torch.cuda.stream(pstreams[j % 2]):
            render_forward(cloud, cams[(k0 + j) % len(cams)], st)
    for s_ in pstreams:
        main.wait_stream(s_)


def batched(bs, ns):
    def run(k0, count):
        for b in range(0, count, bs):
            render_views(cloud, [cams[(k0 + b + j) % len(cams)] for j in range(min(bs, count - b))], st, streams=ns)
    return run


def timed(fn):
    fn(0, 8)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    m0 = torch.cuda.memory_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    fn(8, frames)
    h1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    m1 = torch.cuda.memory_stats()
    timed.mem = (m1.get("num_alloc_retries", 0) - m0.get("num_alloc_retries", 0),
                 m1.get("num_device_alloc", 0) - m0.get("num_device_alloc", 0),
                 m1.get("allocated_bytes.all.peak", 0) / 2**30, m1.get("reserved_bytes.all.current", 0) / 2**30)
    return a.elapsed_time(b) / frames * 1e3, (h1 - h0) / frames * 1e6


print(f"{cfg}: {len(cloud)} Gaussians, {cams[0].width}x{cams[0].height}, {frames} frames")
for name, fn in (("per-view, 2 streams", per_view),
                 ("render_views bs=8, 2 streams", batched(8, 2)),
                 ("render_views bs=8, 3 streams", batched(8, 3)),
                 ("render_views bs=4, 3 streams", batched(4, 3)),
                 ("render_views bs=16, 3 streams", batched(16, 3))):
    dev_us, host_us = timed(fn)
    r, na, pk, rs = timed.mem
    print(f"  {name:32s} {dev_us:8.1f} us/frame ({1e6 / dev_us:7.1f} FPS), host {host_us:8.1f} us/frame; "
          f"alloc retries {r}, cudaMallocs {na}, peak {pk:.1f} GiB, reserved {rs:.1f} GiB")
