"""Generate golden vectors from the UNMODIFIED reference (slimsplat, fp64).

Run in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed here
as small .npz fixtures.  They pin the CPU oracle (oracle/oracle.cpp, float64
instantiation) — tests/test_oracle_golden.py — and through it the CUDA path.

Every input parameter is rounded to float32 BEFORE it is handed to the
reference, so the fp64 reference, the fp32 oracle and the CUDA kernels all
consume identical values.  Scenes follow the reference's own test fixtures
(pkg/tests/conftest.py:26-60, test_rasterizer.py:25-247) plus c1-distribution
scenes from paper_2501_14534_b200.scenes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from scipy.special import logit  # noqa: E402
from slimsplat.cameras import Camera, look_at  # noqa: E402
from slimsplat.cloud import GaussianCloud  # noqa: E402
from slimsplat.rasterizer import RenderSettings, bin_tiles, render_backward, render_forward  # noqa: E402
from slimsplat.training import total_loss  # noqa: E402
from slimsplat.config import TrainConfig  # noqa: E402

from paper_2501_14534_b200 import scenes  # noqa: E402

FIELDS = scenes.PARAM_FIELDS


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def cloud_from(fields: dict) -> GaussianCloud:
    return GaussianCloud(**{f: f32(fields[f]) for f in FIELDS})


def ref_camera(fx, fy, cx, cy, R, t, w, h):
    return Camera(fx=fx, fy=fy, cx=cx, cy=cy, R=R, t=t, width=w, height=h)


def make_camera(size=32, dist=3.5, fx=40.0, fy=42.0):  # conftest.py:42-47 scene
    R, t = look_at(np.array([0.0, -dist, 1.0]), np.zeros(3))
    return ref_camera(fx, fy, (size - 1) / 2.0, (size - 1) / 2.0, R, t, size, size)


def random_cloud(rng, n, alpha_range=(0.1, 0.32), spread=0.8, scale_range=(0.08, 0.3)):
    """Same distributions as conftest.random_cloud (conftest.py:26-39)."""
    c = GaussianCloud.zeros(n)
    c.positions = rng.uniform(-spread, spread, (n, 3))
    c.log_scales = np.log(rng.uniform(scale_range[0], scale_range[1], (n, 3)))
    q = rng.normal(size=(n, 4))
    c.rotations = q / np.linalg.norm(q, axis=1, keepdims=True)
    c.opacity_logits = logit(rng.uniform(alpha_range[0], alpha_range[1], n))
    c.sh_dc = (rng.uniform(0.3, 0.8, (n, 3)) - 0.5) / 0.28209479177387814
    c.sh_rest = rng.normal(0.0, 0.05, (n, 15, 3))
    c.mask_logits = rng.uniform(1.0, 3.0, n)
    c.sh_mask_logits = rng.uniform(1.0, 3.0, (n, 3))
    return {f: getattr(c, f) for f in FIELDS}


def single(color=(1.0, 0.0, 0.0), alpha=0.9, z=0.0, scale=0.4):  # test_rasterizer.py:25-31
    c = GaussianCloud.zeros(1)
    c.positions = np.array([[0.0, 0.0, z]])
    c.log_scales = np.full((1, 3), np.log(scale))
    c.opacity_logits = np.array([logit(alpha)])
    c.sh_dc = (np.array([color]) - 0.5) / 0.28209479177387814
    return c


def cam_arrays(cam):
    return dict(cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]), cam_R=cam.R, cam_t=cam.t,
                cam_size=np.array([cam.width, cam.height]))


def settings_arrays(s: RenderSettings):
    return dict(set_lowpass=s.lowpass_s, set_degree=s.active_sh_degree, set_bg=np.array(s.background, float),
                set_tile=s.tile_size, set_near=s.near, set_mask=s.mask_threshold, set_shmask=s.sh_mask_threshold,
                set_rest=int(s.compute_sh_rest_grads), set_hits=int(s.record_hits))


def input_digest(fields) -> str:
    import hashlib
    h = hashlib.sha256()
    for f in FIELDS:
        h.update(np.ascontiguousarray(np.asarray(fields[f], dtype=np.float32)).tobytes())
    return h.hexdigest()


def run_case(name, cloud: GaussianCloud, cam, settings, dimage=None, full=True, grad_rows=None, records=False,
             store_inputs=True):
    out = render_forward(cloud, cam, settings)
    tiles = out._tiles
    d = dict(**cam_arrays(cam), **settings_arrays(settings))
    if store_inputs:
        d.update({f"in_{f}": getattr(cloud, f).astype(np.float32) for f in FIELDS})
    else:  # regenerated from the seeded generator by the tests; digest pins it
        d["in_digest"] = np.array(input_digest({f: getattr(cloud, f) for f in FIELDS}))
    d.update(image=out.image, transmittance=out.transmittance, weight_sum=out.weight_sum,
             n_contrib=out.n_contrib, last_pos=out.last_pos, visible=out.visible,
             screen_areas=out.screen_areas, tile_offsets=tiles.offsets, tile_ids=tiles.indices)
    if out.hit_counts is not None:
        d["hit_counts"] = out.hit_counts
    if records and out.hit_records is not None:
        cnt = np.array([len(r) for r in out.hit_records], dtype=np.int64)
        d["rec_count"] = cnt
        d["rec_gauss"] = np.array([g for r in out.hit_records for g, _ in r], dtype=np.int64)
        d["rec_weight"] = np.array([w for r in out.hit_records for _, w in r], dtype=np.float64)
    if not full:  # large case: keep float outputs in float32 to bound the fixture size
        for k in ("image", "transmittance", "weight_sum", "screen_areas"):
            d[k] = d[k].astype(np.float32)
    if dimage is not None:
        grads = render_backward(cloud, cam, settings, dimage, out)
        d["dimage"] = dimage
        rows = np.arange(len(cloud)) if grad_rows is None else grad_rows
        d["grad_rows"] = rows
        for f in FIELDS + ("mean2d_screen",):
            g = getattr(grads, f)[rows]
            d[f"grad_{f}"] = g if full else g.astype(np.float32)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **d)
    print(f"{name}: N={len(cloud)} {cam.width}x{cam.height} visible={int(out.visible.sum())} "
          f"instances={tiles.indices.size} -> {os.path.getsize(path) / 1024:.0f} KiB")


def main():
    rng = np.random.default_rng(1234)  # conftest.py:133-135 seed

    # 1. blend vs untiled loop scene (test_rasterizer.py:68-82), large splats
    cam = make_camera(24)
    c = cloud_from(random_cloud(rng, 30, alpha_range=(0.2, 0.9)))
    st = RenderSettings(background=(0.1, 0.2, 0.3), record_hits=True, record_full=True)
    run_case("loop24", c, cam, st, dimage=rng.standard_normal((24, 24, 3)), records=True)

    # 2. finite-difference scene (test_rasterizer.py:210-238)
    cam = make_camera(16, dist=3.5)
    c = cloud_from(random_cloud(rng, 10))
    st = RenderSettings(background=(0.1, 0.2, 0.3))
    run_case("fd16", c, cam, st, dimage=rng.standard_normal((16, 16, 3)))

    # 3. conservation / opaque scenes (test_rasterizer.py:84-89), high alpha -> clamp + termination
    cam = make_camera(32)
    c = cloud_from(random_cloud(rng, 60, alpha_range=(0.3, 0.999)))
    run_case("dense32", c, cam, RenderSettings(), dimage=rng.standard_normal((32, 32, 3)))

    # 4. masks active: Gaussian and SH-band masks cut a large fraction (masking.py:21-43,84-86)
    sc = scenes.small_scene(seed=11, n=400, width=72, height=40, dist=3.0)
    c = cloud_from(sc.fields)
    cam = ref_camera(*[getattr(sc.cameras[0], k) for k in ("fx", "fy", "cx", "cy", "R", "t", "width", "height")])
    st = RenderSettings(near=0.2, mask_threshold=0.85, sh_mask_threshold=0.85, lowpass_s=0.5,
                        background=(0.3, 0.1, 0.2))
    run_case("masked72x40", c, cam, st, dimage=rng.standard_normal((40, 72, 3)))

    # 5. decimated SH-rest grads at active degree 1 (sh.py:202-214, test_rasterizer.py:240-247)
    st = RenderSettings(near=0.2, active_sh_degree=1, compute_sh_rest_grads=False, mask_threshold=0.3)
    run_case("deg1_norest", c, cam, st, dimage=rng.standard_normal((40, 72, 3)))

    # 6. degree 2, tile 8, non-square, lowpass 0 edge (geometry.py:150,176)
    st = RenderSettings(near=0.2, active_sh_degree=2, tile_size=8, lowpass_s=0.0)
    run_case("deg2_tile8", c, cam, st, dimage=rng.standard_normal((40, 72, 3)))

    # 7. known answers (test_rasterizer.py:40-66, 185-199)
    cam17 = make_camera(17, dist=3.0)
    run_case("kat_single", cloud_from({f: getattr(single(alpha=0.999, scale=1.2), f) for f in FIELDS}), cam17,
             RenderSettings())
    axis = -cam17.center / np.linalg.norm(cam17.center)
    front, back = single((1.0, 0.0, 0.0), 0.5, scale=2.0), single((0.0, 0.0, 1.0), 0.9999, scale=2.0)
    front.positions[0] = cam17.center + 2.7 * axis
    back.positions[0] = cam17.center + 3.3 * axis
    two = front.concat(back)
    run_case("kat_two", cloud_from({f: getattr(two, f) for f in FIELDS}), cam17,
             RenderSettings(background=(0.25, 0.5, 0.75)))
    walls = [single(alpha=0.999, z=0.5 - 0.05 * k, scale=3.0) for k in range(6)]
    cl = walls[0]
    for w_ in walls[1:]:
        cl = cl.concat(w_)
    cl = cl.concat(single(color=(0.0, 1.0, 0.0), alpha=0.5, z=-1.5, scale=0.5))
    run_case("kat_walls", cloud_from({f: getattr(cl, f) for f in FIELDS}), cam17, RenderSettings(),
             dimage=np.ones((17, 17, 3)))

    # 8. edge cases: behind camera, off-screen-but-visible (0 tiles), alpha-skipped, masked
    c = GaussianCloud.zeros(6)
    c.positions = np.array([[0, 0, 0], [0, -5, 1.0], [30.0, 0, 0], [0.2, 0.1, 0], [0.1, 0, 0.2], [-0.2, 0, 0]])
    c.log_scales = np.full((6, 3), np.log(0.1))
    c.opacity_logits = np.array([0.0, 0.0, 0.0, -6.0, 0.0, 1.0])   # row 3: sigmoid < 1/255
    c.mask_logits = np.array([2.0, 2.0, 2.0, 2.0, -4.0, 2.0])      # row 4: masked off
    c.sh_dc = np.full((6, 3), 0.7)
    cam = make_camera(32)
    run_case("edges", cloud_from({f: getattr(c, f) for f in FIELDS}), cam, RenderSettings(near=0.2),
             dimage=np.ones((32, 32, 3)))

    # 9. empty cloud
    run_case("empty", cloud_from({f: getattr(GaussianCloud.zeros(0), f) for f in FIELDS}), make_camera(16),
             RenderSettings(background=(0.2, 0.4, 0.6)))

    # 10. c1 (BASELINE configs[0]) with its L1 upstream gradient; float outputs stored as fp32,
    #     gradients for 512 seeded rows
    sc = scenes.config1()
    c = cloud_from(sc.fields)
    cam = ref_camera(*[getattr(sc.cameras[0], k) for k in ("fx", "fy", "cx", "cy", "R", "t", "width", "height")])
    st = RenderSettings(near=0.2)
    out = render_forward(c, cam, st)
    target = sc.targets[0].astype(np.float64)
    dimage = np.sign(out.image - target) / out.image.size   # L1 term of total_loss (training.py:80-82)
    rows = np.sort(np.random.default_rng(99).choice(len(c), 512, replace=False))
    run_case("c1", c, cam, st, dimage=dimage, full=False, grad_rows=rows, store_inputs=False)

    # 11. bin_tiles on raw arrays (test_rasterizer.py:128-172)
    means = rng.uniform(-10, 58, (60, 2))
    radii = rng.uniform(0.5, 20.0, 60)
    depths = rng.uniform(0.1, 5.0, 60)
    means, radii, depths = f32(means), f32(radii), f32(depths)
    b = bin_tiles(means, radii, depths, 48, 40, 16)
    tie_means = np.full((30, 2), 8.0)
    tie_r = np.full(30, 2.0)
    tie_d = rng.integers(1, 4, 30).astype(np.float64)
    tb = bin_tiles(tie_means, tie_r, tie_d, 16, 16, 16)
    np.savez_compressed(os.path.join(HERE, "bins.npz"), means=means, radii=radii, depths=depths,
                        offsets=b.offsets, indices=b.indices, tie_means=tie_means, tie_radii=tie_r,
                        tie_depths=tie_d, tie_offsets=tb.offsets, tie_indices=tb.indices)
    print("bins: ok")

    # 12. loss: total_loss image terms (training.py:61-106, metrics.py:138-188) on a 40x56 pair
    img = rng.uniform(0, 1, (40, 56, 3)).astype(np.float32).astype(np.float64)
    tgt = rng.uniform(0, 1, (40, 56, 3)).astype(np.float32).astype(np.float64)
    cfg = TrainConfig()
    terms, dimg, _, _ = total_loss(img, tgt, GaussianCloud.zeros(1), cfg)
    np.savez_compressed(os.path.join(HERE, "loss.npz"), image=img, target=tgt, l1=terms.l1, d_ssim=terms.d_ssim,
                        lambda_ssim=cfg.lambda_ssim, dimage=dimg)
    print(f"loss: lambda={cfg.lambda_ssim} l1={terms.l1:.6f} d_ssim={terms.d_ssim:.6f}")




def schedule_and_images():
    """Progressive hooks (schedule.py:107-170,218-247) and target ops (images.py:58-102)."""
    from slimsplat.schedule import BlurSpec, Timeline, blur_at, default_blur_decay, lowpass_s_at, phase_at, resolution_at
    from slimsplat.images import area_resize, gaussian_blur
    rows = []
    for mode in ("linear", "logarithmic"):
        for i in (0, 1, 7, 100, 977, 5000, 9999, 19499, 19500, 25000):
            for rs, re_ in ((135, 1080), (240, 1920), (6, 48), (48, 48)):
                rows.append((0 if mode == "linear" else 1, i, rs, re_, 19500, resolution_at(i, rs, re_, 19500, mode)))
    res = np.array(rows, dtype=np.int64)
    lp = np.array([(n, h, w, lowpass_s_at(n, h, w)) for n in (1, 10, 1000, 100000, 1000000)
                   for h, w in ((1080, 1920), (135, 240), (48, 48))], dtype=np.float64)
    blur = []
    spec0 = BlurSpec(9, 2.4)
    decay = default_blur_decay(2.4, 100, 19500, 0.3)
    for i in (0, 50, 100, 1000, 5000, 10000, 19000, 19499, 19500):
        for down in (1.0, 2.0, 8.0, 3.5):
            b = blur_at(i, spec0, 100, decay, 19500, down)
            blur.append((i, down, b.size, b.sigma))
    blur = np.array(blur, dtype=np.float64)
    tl = Timeline()
    names = ["standard_densify", "late_densify", "mask_prune", "significance_prune", "sh_full_update",
             "progressive_scale_active"]
    its = np.array([0, 16, 500, 600, 9999, 10000, 15500, 16000, 20000, 20100, 20500, 21000, 29999])
    phases = np.array([[n in phase_at(int(i), tl) for n in names] for i in its], dtype=np.uint8)
    rng = np.random.default_rng(77)
    img = rng.uniform(0, 1, (61, 83, 3))
    np.savez_compressed(os.path.join(HERE, "schedule.npz"), res=res, lowpass=lp, blur=blur, decay=decay,
                        phase_its=its, phases=phases, phase_names=np.array(names), img=img,
                        area_17x29=area_resize(img, 17, 29), area_61x40=area_resize(img, 61, 40),
                        blur_7_1p3=gaussian_blur(img, 7, 1.3), blur_9_2p4=gaussian_blur(img, 9, 2.4))
    print("schedule: ok")


def significance_golden():
    """Significance scoring and pruning (significance.py:31-104): hits over several
    views, volumes, the nearest-rank 90th-percentile normaliser, scores, the pruned
    set for a rate, the event schedule; plus the v90 == 0 branch (most rows masked)."""
    from slimsplat.significance import count_hits, prune_by_significance, prune_schedule, significance_scores
    rng = np.random.default_rng(4242)
    d = {}
    for tag, n, mask_mean in (("a", 700, 2.0), ("z", 300, -6.0)):
        fields = scenes.random_fields(rng, n, ls_mean=-2.6, ls_std=0.5)
        if tag == "z":  # all but ~5% of the rows masked off -> v90 == 0
            m = np.full(n, mask_mean)
            m[rng.choice(n, n // 20, replace=False)] = 3.0
            fields["mask_logits"] = m
        cloud = cloud_from(fields)
        cams = [scenes.pinhole(3.2 * scenes._unit(rng), 64, 48) for _ in range(3)]
        rcams = [ref_camera(c.fx, c.fy, c.cx, c.cy, c.R, c.t, c.width, c.height) for c in cams]
        st = RenderSettings(near=0.2, mask_threshold=0.3)
        hits = count_hits(cloud, rcams, st)
        rep = significance_scores(hits, cloud, mask_threshold=0.3, volume_power=0.5)
        _, keep = prune_by_significance(cloud, rep.scores, 0.35)
        d.update({f"{tag}_in_{f}": getattr(cloud, f).astype(np.float32) for f in FIELDS})
        d[f"{tag}_cam_intr"] = np.array([[c.fx, c.fy, c.cx, c.cy] for c in cams])
        d[f"{tag}_cam_R"] = np.stack([c.R for c in cams])
        d[f"{tag}_cam_t"] = np.stack([c.t for c in cams])
        d[f"{tag}_cam_size"] = np.array([[c.width, c.height] for c in cams])
        d.update({f"{tag}_hits": hits, f"{tag}_volumes": rep.volumes, f"{tag}_v_norm": rep.v_norm,
                  f"{tag}_scores": rep.scores, f"{tag}_keep": keep})
        print(f"significance {tag}: n={n} hits>0={int((hits > 0).sum())} kept={keep.size}")
    d["schedule"] = np.array([[k, prune_schedule(k, 0.6, 0.5)] for k in range(5)])
    d["mask_threshold"], d["volume_power"], d["rate"] = 0.3, 0.5, 0.35
    np.savez_compressed(os.path.join(HERE, "significance.npz"), **d)


if __name__ == "__main__":
    if len(sys.argv) == 1:
        main()
    if len(sys.argv) == 1 or "schedule" in sys.argv:
        schedule_and_images()
    if len(sys.argv) == 1 or "significance" in sys.argv:
        significance_golden()
