"""CUDA path vs the reference (golden vectors) and vs the oracle (GPU only).

Bars (BASELINE.json north star):
  * bit-exact vs the float32 oracle: visibility, every column of the projected
    record (means, conic, alpha, colour, depth, radius, area), tiles_touched,
    sorted tile lists and CSR offsets;
  * image / transmittance / weight_sum within 1e-4 absolute of the float64
    reference;
  * gradients within 1e-3 relative / 1e-5 absolute, the absolute floor scaled by
    the field's largest entry under O(1) upstream gradients.
"""

import numpy as np
import pytest
import torch

import golden_io
from oracle import oracle

pytestmark = pytest.mark.gpu

GRAD_FIELDS = golden_io.FIELDS + ("mean2d_screen",)


@pytest.fixture(scope="module")
def tgs():
    import paper_2501_14534_b200 as p
    from paper_2501_14534_b200 import _lib
    _lib.load()
    return p


def _settings(tgs, s):
    return tgs.RenderSettings(lowpass_s=s.lowpass_s, active_sh_degree=s.active_sh_degree, background=s.background,
                              tile_size=s.tile_size, near=s.near, record_hits=s.record_hits,
                              mask_threshold=s.mask_threshold, sh_mask_threshold=s.sh_mask_threshold,
                              compute_sh_rest_grads=s.compute_sh_rest_grads)


def _np(t):
    return t.detach().cpu().numpy()


def _grad_close(got, ref, name):
    """Gradients under an O(1) upstream gradient (the golden fixtures and c1 use N(0, 1), as
    the reference's own tests do): 1e-3 relative, and an absolute floor of 1e-5 times the
    field's largest entry.  Such a gradient is a float32 sum of O(1)..O(10) per-pixel terms
    that can cancel to ~1e-3, where float32 reassociation alone moves it by ~1e-5 (measured:
    1 entry in 1,200 at masked72x40 and deg1_norest, |err| 1.2e-5 / 2.5e-5).  The plain
    1e-3 / 1e-5 bar holds for every entry under the training loss's own upstream gradient
    at c3 (tests/test_gpu_c3_parity.py::test_c3_gradients_vs_fp64_oracle[l1_ssim])."""
    atol = 1e-5 * max(1.0, float(np.abs(ref).max()) if ref.size else 1.0)
    np.testing.assert_allclose(got, ref, rtol=1e-3, atol=atol, err_msg=name)


@pytest.mark.parametrize("name", golden_io.CASES)
def test_forward_backward_vs_reference_golden(tgs, name):
    case = golden_io.load(name)
    z = case.z
    st = _settings(tgs, case.settings)
    cloud = tgs.GaussianCloud.from_fields(case.fields)
    out = tgs.render_forward(cloud, case.cam, st)
    assert np.array_equal(_np(out.visible), z["visible"])
    np.testing.assert_allclose(_np(out.screen_areas), z["screen_areas"], rtol=1e-5, atol=1e-6)
    assert np.array_equal(_np(out._tiles.offsets), z["tile_offsets"])
    valid = np.flatnonzero(z["visible"])
    ref_ids = valid[z["tile_ids"]] if z["tile_ids"].size else z["tile_ids"]
    assert np.array_equal(_np(out._tiles.indices), ref_ids)
    np.testing.assert_allclose(_np(out.image), z["image"], atol=1e-4, rtol=0)
    np.testing.assert_allclose(_np(out.transmittance), z["transmittance"], atol=1e-4, rtol=0)
    np.testing.assert_allclose(_np(out.weight_sum), z["weight_sum"], atol=1e-4, rtol=0)
    if name != "kat_walls":  # T hits exactly 1e-4 there (see test_oracle_golden)
        assert np.array_equal(_np(out.n_contrib), z["n_contrib"])
        assert np.array_equal(_np(out.last_pos), z["last_pos"])
    if "dimage" not in z:
        return
    g = tgs.render_backward(cloud, case.cam, st, torch.from_numpy(z["dimage"].astype(np.float32)).cuda(), out)
    if name == "kat_walls":
        for f in ("positions", "sh_dc", "opacity_logits"):
            assert np.all(_np(getattr(g, f))[-1] == 0.0)
        return
    rows = z["grad_rows"]
    for f in GRAD_FIELDS:
        _grad_close(_np(getattr(g, f))[rows], z[f"grad_{f}"], f)


@pytest.mark.parametrize("cfg", ["c1", "c2", "masked", "deg1", "tile8", "tile32", "uhd", "uhd_c4", "plane"])
def test_preprocess_and_sort_bit_exact_vs_fp32_oracle(tgs, cfg):
    from paper_2501_14534_b200 import scenes
    kw = {}
    if cfg == "c1":
        sc = scenes.config1()
    elif cfg == "c2":
        sc = scenes.config2()
    elif cfg == "uhd":  # 3840x2160: 32,400 tiles -> two count slabs, C > 512 is not needed
        sc = scenes.small_scene(seed=22, n=150_000, width=3840, height=2160, dist=3.0)
    elif cfg == "uhd_c4":  # c4 cluster scene, fewer Gaussians, 4K, frame 37 of the orbit
        sc = scenes.config4(n=300_000, frames=200)
        sc.cameras[0] = sc.cameras[37]
    elif cfg == "plane":  # 12k Gaussians at exactly one depth: overflows a value bucket -> LSD fallback
        sc = scenes.small_scene(seed=23, n=24_000, width=320, height=240, dist=4.0)
        sc.fields["positions"][:12_000, 0] = 0.0
        sc.cameras[0] = scenes.pinhole((4.0, 0.0, 0.0), 320, 240)
    else:
        sc = scenes.small_scene(seed=21, n=30_000, width=333, height=207, dist=3.0)
        kw = {"masked": dict(mask_threshold=0.85, sh_mask_threshold=0.85, lowpass_s=0.5),
              "deg1": dict(active_sh_degree=1, lowpass_s=0.0), "tile8": dict(tile_size=8),
              "tile32": dict(tile_size=32, active_sh_degree=2)}[cfg]
    st = tgs.RenderSettings(near=0.2, **kw)
    cam = sc.cameras[0]
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    out = tgs.render_forward(cloud, cam, st)
    ref = oracle.preprocess(sc.fields, cam, st, "f32")
    st_state = out._state
    sp = _np(st_state.splats)[: len(cloud)]
    assert np.array_equal(_np(out.visible), ref["visible"])
    assert np.array_equal(sp.view(np.uint32), ref["splats"].view(np.uint32)), \
        f"splat columns differ: {np.unique(np.nonzero(sp.view(np.uint32) != ref['splats'].view(np.uint32))[1])}"
    assert np.array_equal(_np(st_state.tiles_touched)[: len(cloud)], ref["tiles_touched"])
    off, ids, _, _ = oracle.bin_tiles(ref["splats"], ref["tiles_touched"], cam.width, cam.height, st.tile_size, "f32",
                                      ref["depth_key"])
    assert np.array_equal(_np(out._tiles.offsets).astype(np.int64), off)
    assert np.array_equal(_np(out._tiles.indices).astype(np.int64), ids)


def test_c2_image_vs_fp64_oracle(tgs):
    """c2 (200k Gaussians, 720p) forward within 1e-4 of the float64 restatement."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.config2()
    st = tgs.RenderSettings(near=0.2)
    out = tgs.render_forward(tgs.GaussianCloud.from_fields(sc.fields), sc.cameras[0], st)
    ref = oracle.render_forward(sc.fields, sc.cameras[0], st, "f64")
    assert np.array_equal(_np(out.visible), ref["visible"])
    # the blend decisions at alpha = 1/255 and e = -4.5 are the float64 ones (exact
    # blend-decision records), so every pixel is within the north-star 1e-4 (a float32
    # decision flips 57 of 921,600 pixels here by up to 5.1e-3)
    for got, want in ((out.image, ref["image"]), (out.transmittance, ref["transmittance"]),
                      (out.weight_sum, ref["weight_sum"])):
        err = np.abs(_np(got) - want)
        assert err.max() <= 1e-4, f"max err {err.max():.3e}, {(err > 1e-4).sum()} entries above 1e-4"
    np.testing.assert_allclose(_np(out.weight_sum) + _np(out.transmittance), 1.0, atol=1e-5)


def test_blend_exception_lists_equal_float64_resolution(tgs):
    """The backward deciding bracket pairs from the forward's exception lists gives the
    same partials as re-resolving them in float64: at c2 with 2% clampable Gaussians
    (alpha > 0.9899: the backward decides their clamp in float64 near their centres), with
    the per-pixel exceptions and the overflow tiles (float64 body) exercised; and with
    every tile flagged."""
    import dataclasses
    from paper_2501_14534_b200 import scenes
    sc = scenes.config2()
    fields = dict(sc.fields)
    rng = np.random.default_rng(11)
    ol = fields["opacity_logits"].copy()
    ol[rng.choice(ol.size, ol.size // 50, replace=False)] = 6.0
    fields["opacity_logits"] = ol
    st = tgs.RenderSettings(near=0.2)
    cam = sc.cameras[0]
    cloud = tgs.GaussianCloud.from_fields(fields)
    out = tgs.render_forward(cloud, cam, st)
    state = out._state
    assert state.exceptions is not None and state.exc_overflow is not None
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    ovf = _np(state.exc_overflow).view(np.uint32)
    cnt, flags = int(ovf[0]), ovf[1:1 + nt]
    assert 0 < cnt < nt and int(flags.sum()) == cnt and set(np.unique(flags)) <= {0, 1}
    word, lp = _np(state.exceptions), _np(out.last_pos)
    exc = word & 0x7FFFFFFF  # 1-based list position | clamped << 31
    assert (exc <= lp).all()
    assert (exc > 0).sum() > 0 and (word < 0).sum() > 0  # both kinds: blended in the bracket, clamped
    dimg = torch.from_numpy(rng.standard_normal((cam.height, cam.width, 3)).astype(np.float32)).cuda()
    ds_exc, _ = tgs.rasterizer.blend_backward(cloud, cam, st, dimg, out)
    plain = dataclasses.replace(out, _state=dataclasses.replace(state, exceptions=None, exc_overflow=None))
    ds_chk, _ = tgs.rasterizer.blend_backward(cloud, cam, st, dimg, plain)
    a, b = _np(ds_exc), _np(ds_chk)
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6 * np.abs(b).max())
    every = torch.from_numpy(np.concatenate([[nt], np.ones(nt)]).astype(np.int32)).cuda()
    forced = dataclasses.replace(out, _state=dataclasses.replace(state, exc_overflow=every))
    ds_all, _ = tgs.rasterizer.blend_backward(cloud, cam, st, dimg, forced)
    np.testing.assert_allclose(_np(ds_all), b, rtol=1e-5, atol=1e-6 * np.abs(b).max())


@pytest.mark.parametrize("shift", [3.0, 6.0])
def test_opaque_scene_vs_fp64_oracle(tgs, shift):
    """A trained scene's Gaussians saturate: a c2-like scene (100k, 640x480) with every opacity
    logit raised (shift 6: most
    alpha > 0.99, so the 0.99 clamp decides whether dL/dalpha flows, _kernels.py:157-168;
    shift 3: alpha around 0.95, the clamp boundary inside many footprints).  Image within
    1e-4 of the float64 reference, every gradient field within the north-star bar outside
    the T = 1e-4 termination flips (see test_c1_gradients_vs_fp64_oracle_full)."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.config2(n=100_000, width=640, height=480)
    fields = dict(sc.fields)
    fields["opacity_logits"] = (fields["opacity_logits"] + np.float32(shift)).astype(np.float32)
    st = tgs.RenderSettings(near=0.2)
    cam = sc.cameras[0]
    dimg = np.random.default_rng(19).standard_normal((cam.height, cam.width, 3)).astype(np.float32)
    cloud = tgs.GaussianCloud.from_fields(fields)
    out = tgs.render_forward(cloud, cam, st)
    g = tgs.render_backward(cloud, cam, st, torch.from_numpy(dimg).cuda(), out)
    ref_f = oracle.render_forward(fields, cam, st, "f64")
    ref_g = oracle.render_backward(fields, cam, st, dimg.astype(np.float64), ref_f, "f64")
    for got, want in ((out.image, ref_f["image"]), (out.transmittance, ref_f["transmittance"])):
        err = np.abs(_np(got) - want)
        assert err.max() <= 1e-4, err.max()
    from test_gpu_c3_parity import flip_rows
    flipped, npix = flip_rows(out, ref_f, cam, st.tile_size)
    keep = np.ones(len(cloud), dtype=bool)
    keep[flipped] = False
    assert npix <= 1e-3 * out.last_pos.numel() + 5, (npix, flipped.size)
    for f in GRAD_FIELDS:
        got, ref = _np(getattr(g, f)), ref_g[f]
        _grad_close(got[keep], ref[keep], f)


def test_c1_gradients_vs_fp64_oracle_full(tgs):
    """All N rows at c1 with an O(1) upstream gradient (dimage ~ N(0,1))."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.config1()
    st = tgs.RenderSettings(near=0.2)
    cam = sc.cameras[0]
    dimg = np.random.default_rng(7).standard_normal((cam.height, cam.width, 3)).astype(np.float32)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    out = tgs.render_forward(cloud, cam, st)
    g = tgs.render_backward(cloud, cam, st, torch.from_numpy(dimg).cuda(), out)
    ref_f = oracle.render_forward(sc.fields, cam, st, "f64")
    ref_g = oracle.render_backward(sc.fields, cam, st, dimg.astype(np.float64), ref_f, "f64")
    # rows between the two stopping positions of a pixel whose transmittance crosses
    # T = 1e-4 one entry apart in float32 and float64 (see test_gpu_c3_parity.flip_rows)
    from test_gpu_c3_parity import flip_rows
    flipped, npix = flip_rows(out, ref_f, cam, st.tile_size)
    keep = np.ones(len(cloud), dtype=bool)
    keep[flipped] = False
    assert npix <= 1e-4 * out.last_pos.numel() + 5, (npix, flipped.size)
    for f in GRAD_FIELDS:
        got, ref = _np(getattr(g, f)), ref_g[f]
        rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
        assert rel < 1e-4, (f, rel)
        _grad_close(got[keep], ref[keep], f)


def test_hits_and_records_vs_reference(tgs):
    case = golden_io.load("loop24")
    st = _settings(tgs, case.settings)
    st.record_hits = True
    st.record_full = True
    out = tgs.render_forward(tgs.GaussianCloud.from_fields(case.fields), case.cam, st)
    assert np.array_equal(_np(out.hit_counts), case.z["hit_counts"])
    recs = out.hit_records
    assert [len(r) for r in recs] == case.z["rec_count"].tolist()
    flat_g = np.array([g for r in recs for g, _ in r])
    flat_w = np.array([w for r in recs for _, w in r])
    assert np.array_equal(flat_g, case.z["rec_gauss"])
    np.testing.assert_allclose(flat_w, case.z["rec_weight"], atol=1e-5)


def test_bin_tiles_raw_arrays(tgs):
    z = dict(np.load(f"{golden_io.GOLDEN}/bins.npz"))
    b = tgs.bin_tiles(z["means"], z["radii"], z["depths"], 48, 40, 16)
    assert np.array_equal(_np(b.offsets), z["offsets"]) and np.array_equal(_np(b.indices), z["indices"])
    b = tgs.bin_tiles(z["tie_means"], z["tie_radii"], z["tie_depths"], 16, 16, 16)
    assert np.array_equal(_np(b.offsets), z["tie_offsets"]) and np.array_equal(_np(b.indices), z["tie_indices"])


def test_row_bands_compose_to_full_render(tgs):
    """Tile-row sharding: rendering disjoint bands reproduces the full image bitwise."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.small_scene(seed=3, n=20_000, width=320, height=200)
    st = tgs.RenderSettings(near=0.2)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    cam = sc.cameras[0]
    full = tgs.render_forward(cloud, cam, st)
    ty = (cam.height + 15) // 16
    img = torch.zeros_like(full.image)
    for rb, re in ((0, 3), (3, 4), (4, ty)):
        part = tgs.render_forward(cloud, cam, st, row_band=(rb, re))
        rows = slice(rb * 16, min(re * 16, cam.height))
        img[rows] = part.image[rows]
    assert torch.equal(img, full.image)
    # the band's tile lists are exactly the full lists of its tiles
    fo, fi = _np(full._tiles.offsets), _np(full._tiles.indices)
    tx = (cam.width + 15) // 16
    for rb, re in ((0, 3), (3, 4), (4, ty), (1, ty - 1)):
        part = tgs.render_forward(cloud, cam, st, row_band=(rb, re))
        po, pi = _np(part._tiles.offsets), _np(part._tiles.indices)
        want_o = fo[rb * tx: re * tx + 1] - fo[rb * tx]
        assert np.array_equal(po, want_o)
        assert np.array_equal(pi, fi[fo[rb * tx]: fo[re * tx]])


def test_errors_and_edges(tgs):
    from paper_2501_14534_b200 import scenes
    sc = scenes.small_scene(seed=4, n=50, width=32, height=32)
    cam = sc.cameras[0]
    st = tgs.RenderSettings(near=0.2)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    out = tgs.render_forward(cloud, cam, st)
    with pytest.raises(tgs.ContractViolationError):
        tgs.render_backward(cloud, cam, st, torch.zeros((31, 32, 3), device="cuda"), out)
    out.last_pos = None
    with pytest.raises(tgs.ContractViolationError):
        tgs.render_backward(cloud, cam, st, torch.zeros((32, 32, 3), device="cuda"), out)
    bad = dict(sc.fields)
    bad["rotations"] = bad["rotations"].copy()
    bad["rotations"][7] = 0.0
    with pytest.raises(tgs.DegenerateRotationError):
        tgs.render_forward(tgs.GaussianCloud.from_fields(bad), cam, st)
    with pytest.raises(tgs.ContractViolationError):
        tgs.render_forward(cloud, cam, tgs.RenderSettings(mask_threshold=1.5))
    with pytest.raises(tgs.ContractViolationError):
        tgs.render_forward(cloud, cam, tgs.RenderSettings(lowpass_s=-1.0))
    # zero upstream gradient -> zero gradients (test_rasterizer.py:176-183)
    out = tgs.render_forward(cloud, cam, st)
    g = tgs.render_backward(cloud, cam, st, torch.zeros((32, 32, 3), device="cuda"), out)
    assert float(g.flat.abs().max()) == 0.0
    # decimated SH-rest gradients (test_rasterizer.py:240-247)
    st2 = tgs.RenderSettings(near=0.2, compute_sh_rest_grads=False)
    out = tgs.render_forward(cloud, cam, st2)
    g = tgs.render_backward(cloud, cam, st2, torch.randn((32, 32, 3), device="cuda"), out)
    assert float(g.sh_rest.abs().max()) == 0.0 and float(g.sh_mask_logits.abs().max()) == 0.0
    assert float(g.sh_dc.abs().max()) > 0.0


def test_loss_vs_reference_golden(tgs):
    from paper_2501_14534_b200 import loss
    z = dict(np.load(f"{golden_io.GOLDEN}/loss.npz"))
    img = torch.from_numpy(z["image"].astype(np.float32)).cuda()
    tgt = torch.from_numpy(z["target"].astype(np.float32)).cuda()
    terms, dimg = loss.l1_ssim(img, tgt, float(z["lambda_ssim"]))
    assert abs(terms["l1"] - float(z["l1"])) < 1e-6
    assert abs(terms["d_ssim"] - float(z["d_ssim"])) < 1e-5
    ref = z["dimage"]
    np.testing.assert_allclose(_np(dimg), ref, rtol=1e-3, atol=1e-4 * np.abs(ref).max())


def test_fused_loss_vs_fp64_restatement_multi_tile(tgs):
    """Fused SSIM kernel over many 32x32 tiles incl. ragged borders vs oracle/loss_ref.py."""
    from oracle import loss_ref
    from paper_2501_14534_b200 import loss
    rng = np.random.default_rng(3)
    img = rng.uniform(0, 1, (150, 203, 3)).astype(np.float32)
    tgt = np.clip(img + rng.normal(0, 0.2, img.shape), 0, 1).astype(np.float32)
    terms, d = loss.l1_ssim(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), 0.2)
    l1, dssim, dref = loss_ref.total_loss_image(img, tgt, 0.2)
    assert abs(terms["l1"] - l1) < 1e-6 and abs(terms["d_ssim"] - dssim) < 1e-5
    np.testing.assert_allclose(_np(d), dref, rtol=1e-3, atol=1e-4 * np.abs(dref).max())


def test_c3_scale_properties(tgs):
    """Size-independent properties at the full c3 size (1M Gaussians, 1080p)."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.config3(views=1)
    st = tgs.RenderSettings(near=0.2, mask_threshold=0.01)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    out = tgs.render_forward(cloud, sc.cameras[0], st)
    ws, T = _np(out.weight_sum), _np(out.transmittance)
    np.testing.assert_allclose(ws + T, 1.0, atol=2e-5)         # conservation (test_rasterizer.py:84-89)
    nc, lp = _np(out.n_contrib), _np(out.last_pos)
    assert (nc <= lp).all() and ((nc == 0) == (lp == 0)).all()
    off = _np(out._tiles.offsets)
    assert off[0] == 0 and (np.diff(off) >= 0).all() and off[-1] == out._tiles.indices.numel()
    # sortedness: within every tile, float64 depth keys ascend (ties by index)
    keys = _np(out._state.depth_keys).view(np.uint64)
    ids = _np(out._tiles.indices).astype(np.int64)
    k = keys[ids]
    tile_of = np.repeat(np.arange(off.size - 1), np.diff(off))
    same = tile_of[1:] == tile_of[:-1]
    assert ((k[1:] > k[:-1]) | ((k[1:] == k[:-1]) & (ids[1:] > ids[:-1])))[same].all()
    # completeness: every Gaussian sits in exactly the tiles of its rect, once each
    sp = _np(out._state.splats)[: len(cloud)]
    tt = _np(out._state.tiles_touched)[: len(cloud)]
    assert np.array_equal(np.bincount(ids, minlength=len(cloud)), np.maximum(tt, 0))
    mx, my, r = sp[ids, 0], sp[ids, 1], sp[ids, 10]
    f16 = np.float32(16)
    tx_, ty_ = tile_of % 120, tile_of // 120
    x0 = np.clip(np.floor((mx - r) / f16), 0, 119)
    x1 = np.clip(np.floor((mx + r) / f16), 0, 119)
    y0 = np.clip(np.floor((my - r) / f16), 0, 67)
    y1 = np.clip(np.floor((my + r) / f16), 0, 67)
    assert ((tx_ >= x0) & (tx_ <= x1) & (ty_ >= y0) & (ty_ <= y1)).all()
    # determinism: a second render is bitwise identical
    out2 = tgs.render_forward(cloud, sc.cameras[0], st)
    assert torch.equal(out.image, out2.image) and torch.equal(out._tiles.indices, out2._tiles.indices)


def test_multiview_backward_equals_sum_of_views(tgs):
    """tgs_preprocess_backward_views (one pass over the parameters, 11 views -> two
    chunks of <= 8) equals the sum of per-view render_backward gradients."""
    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.rasterizer import blend_backward, preprocess_backward_views
    sc = scenes.small_scene(seed=12, n=5000, width=96, height=80, dist=3.5)
    st = tgs.RenderSettings(near=0.2, mask_threshold=0.3)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    rng = np.random.default_rng(5)
    cams = [scenes.pinhole(rng.uniform(3.0, 4.5) * d / np.linalg.norm(d), 96, 80)
            for d in rng.normal(size=(11, 3))]
    want = tgs.CloudGrads.zeros(len(cloud))
    vis, parts = [], []
    for cam in cams:
        dimg = torch.from_numpy(rng.standard_normal((80, 96, 3)).astype(np.float32)).cuda()
        out = tgs.render_forward(cloud, cam, st)
        tgs.render_backward(cloud, cam, st, dimg, out, grads=want, accumulate=True)
        ds, state = blend_backward(cloud, cam, st, dimg, out)
        vis.append(state.visible_u8)
        parts.append(ds)
    got = preprocess_backward_views(cloud, cams, st, vis, parts, tgs.CloudGrads.zeros(len(cloud)))
    for f in GRAD_FIELDS:
        a, b = _np(getattr(got, f)), _np(getattr(want, f))
        _grad_close(a, b, f)


def test_target_ops_vs_reference(tgs):
    from paper_2501_14534_b200 import images
    z = dict(np.load(f"{golden_io.GOLDEN}/schedule.npz"))
    img = torch.from_numpy(z["img"].astype(np.float32)).cuda()
    np.testing.assert_allclose(_np(images.area_resize(img, 17, 29)), z["area_17x29"], atol=2e-6)
    np.testing.assert_allclose(_np(images.area_resize(img, 61, 40)), z["area_61x40"], atol=2e-6)
    np.testing.assert_allclose(_np(images.gaussian_blur(img, 7, 1.3)), z["blur_7_1p3"], atol=2e-6)
    np.testing.assert_allclose(_np(images.gaussian_blur(img, 9, 2.4)), z["blur_9_2p4"], atol=2e-6)
    assert torch.equal(images.area_resize(img, 61, 83), img)


def test_prune_compaction_and_adam(tgs):
    """masking.prune_by_mask (masking.py:70-81) + Adam row compaction (optim.py:51-55)."""
    from paper_2501_14534_b200 import optim, pruning
    case = golden_io.load("masked72x40")
    cloud = tgs.GaussianCloud.from_fields(case.fields)
    opt = optim.Adam(cloud, {f: 1e-2 for f in golden_io.FIELDS})
    g = tgs.CloudGrads.zeros(len(cloud))
    g.flat.normal_()
    opt.step(cloud, g)
    old = cloud
    new, keep = pruning.prune_by_mask(cloud, 0.85)
    s = 1.0 / (1.0 + np.exp(-_np(old.mask_logits).astype(np.float64)))  # logits after the Adam step
    want = np.flatnonzero(s > 0.85)                       # reference: hard_mask(m, eps) > 0
    assert np.array_equal(_np(keep), want)
    for f in golden_io.FIELDS:
        assert np.array_equal(_np(getattr(new, f)), _np(getattr(old, f))[want])
    mo = {f: _np(opt.m[old.field_range(f)[0]:][: old.field_range(f)[1]]) for f in golden_io.FIELDS}
    pruning.compact_adam(opt, old, new, keep)
    for f in golden_io.FIELDS:
        o, size = new.field_range(f)
        got = _np(opt.m[o:o + size]).reshape((len(new),) + tuple(getattr(new, f).shape[1:]))
        assert np.array_equal(got, mo[f].reshape((len(old),) + tuple(getattr(old, f).shape[1:]))[want])
    with pytest.raises(tgs.EmptySceneError):
        pruning.prune_by_mask(new, 0.9999)


def test_adam_matches_reference_formula(tgs):
    """optim.Adam.update (optim.py:37-49) in float64 vs the kernel."""
    from paper_2501_14534_b200 import optim
    rng = np.random.default_rng(0)
    sc = golden_io.load("fd16")
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    opt = optim.Adam(cloud, {f: 1e-2 for f in golden_io.FIELDS}, eps=1e-15)
    p = _np(cloud.positions).astype(np.float64)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for step in range(1, 4):
        grad = rng.standard_normal(p.shape).astype(np.float32)
        g = tgs.CloudGrads.zeros(len(cloud))
        g.positions.copy_(torch.from_numpy(grad))
        opt.update(cloud, g, "positions")
        m = 0.9 * m + 0.1 * grad
        v = 0.999 * v + 0.001 * grad * grad
        p -= 1e-2 * (m / (1 - 0.9 ** step)) / (np.sqrt(v / (1 - 0.999 ** step)) + 1e-15)
    np.testing.assert_allclose(_np(cloud.positions), p, rtol=1e-5, atol=1e-6)


def test_compat_adaptor_reference_conventions(tgs):
    """numpy in/out with V'-space tile ids, as the reference's RenderOutput (rasterizer.py:177-200)."""
    from paper_2501_14534_b200 import compat
    case = golden_io.load("masked72x40")
    from types import SimpleNamespace
    cloud = SimpleNamespace(**{f: case.fields[f].astype(np.float64) for f in golden_io.FIELDS})
    out = compat.render_forward(cloud, case.cam, case.settings)
    z = case.z
    assert out.image.dtype == np.float64 and out.image.shape == z["image"].shape
    np.testing.assert_allclose(out.image, z["image"], atol=1e-4)
    assert np.array_equal(out._tiles.offsets, z["tile_offsets"])
    assert np.array_equal(out._tiles.indices, z["tile_ids"])
    g = compat.render_backward(cloud, case.cam, case.settings, z["dimage"], out)
    for f in golden_io.FIELDS:
        _grad_close(getattr(g, f), z[f"grad_{f}"], f)
    b = compat.bin_tiles(z["image"][:0, 0, :2].reshape(0, 2), np.zeros(0), np.zeros(0), 16, 16, 16)
    assert b.indices.size == 0 and np.all(b.offsets == 0)


def test_render_sharded_single_rank_nccl(tgs):
    """parallel.render_sharded through a real NCCL group (world size 1 on this box)."""
    import socket

    import torch.distributed as dist

    from paper_2501_14534_b200 import parallel, scenes
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        sc = scenes.small_scene(seed=8, n=20_000, width=300, height=170)
        st = tgs.RenderSettings(near=0.2)
        cloud = tgs.GaussianCloud.from_fields(sc.fields)
        img = parallel.render_sharded(cloud, sc.cameras[0], st)
        ref = tgs.render_forward(cloud, sc.cameras[0], st).image
        assert torch.equal(img, ref)
        # a sequence through one renderer (bands from the previous batch's histogram)
        rng = np.random.default_rng(9)
        orbit = [scenes.pinhole(3.0 * scenes._unit(rng), 300, 170, name=f"o{k}") for k in range(5)]
        r = parallel.ShardedRenderer(cloud, st)
        got = r.render(orbit[:3]) + r.render(orbit[3:])
        for cam, im in zip(orbit, got):
            assert torch.equal(im, tgs.render_forward(cloud, cam, st).image)
        from paper_2501_14534_b200 import rasterizer
        splats, _, tiles, _, _, _ = rasterizer.preprocess(cloud, sc.cameras[0], st)
        counts = parallel.row_histogram(splats, tiles, len(cloud), sc.cameras[0], 16)
        out = tgs.render_forward(cloud, sc.cameras[0], st)
        per_tile = np.diff(_np(out._tiles.offsets)).reshape(-1, out._tiles.tiles_x).sum(axis=1)
        assert np.array_equal(_np(counts), per_tile)
        # the data-parallel training step (bucketed NCCL all-reduce on a communication
        # stream, per-bucket Adam) equals the single-process step (one fused Adam)
        from paper_2501_14534_b200.train import Trainer
        rng = np.random.default_rng(8)
        cams = [sc.cameras[0]] + [scenes.pinhole(3.0 * scenes._unit(rng), 160, 96, name=f"d{k}") for k in range(2)]
        tg = [torch.rand((c.height, c.width, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(k))
              for k, c in enumerate(cams)]
        res = []
        for pg in (dist.group.WORLD, None):
            c2 = tgs.GaussianCloud.from_fields(sc.fields)
            tr = Trainer(c2, cams, [t.clone() for t in tg], st, process_group=pg, deterministic=True)
            tr.step()
            tr.step()
            torch.cuda.synchronize()
            res.append((tr.cloud.flat.clone(), tr.terms.clone(), dict(tr.opt.steps)))
        assert torch.equal(res[0][1], res[1][1]) and res[0][2] == res[1][2]
        np.testing.assert_allclose(_np(res[0][0]), _np(res[1][0]), rtol=1e-6, atol=1e-10)
    finally:
        dist.destroy_process_group()


def test_depth_sort_fallback_path_runs_only_on_bucket_overflow(tgs):
    """The value-bucket depth sort hands over to the ticketed LSD chain exactly when a
    bucket overflows; the chain's per-ticket trace shows which path ran."""
    import ctypes
    from paper_2501_14534_b200 import _lib, scenes
    lib = _lib.load()
    st = tgs.RenderSettings(near=0.2)
    buf = torch.zeros(8 * 4096, dtype=torch.int64, device="cuda")
    ran = {}
    for name in ("random", "plane"):
        sc = scenes.small_scene(seed=23, n=24_000, width=320, height=240, dist=4.0)
        cam = sc.cameras[0]
        if name == "plane":
            sc.fields["positions"][:12_000, 0] = 0.0
            cam = scenes.pinhole((4.0, 0.0, 0.0), 320, 240)
        cloud = tgs.GaussianCloud.from_fields(sc.fields)
        buf.zero_()
        lib.tgs_debug_trace_depth_sort(ctypes.c_void_p(buf.data_ptr()))
        try:
            out = tgs.render_forward(cloud, cam, st)
            torch.cuda.synchronize()
        finally:
            lib.tgs_debug_trace_depth_sort(ctypes.c_void_p(0))
        ran[name] = bool((buf != 0).any())
        ref = oracle.preprocess(sc.fields, cam, st, "f32")
        off, ids, _, _ = oracle.bin_tiles(ref["splats"], ref["tiles_touched"], cam.width, cam.height, st.tile_size,
                                          "f32", ref["depth_key"])
        assert np.array_equal(_np(out._tiles.offsets).astype(np.int64), off)
        assert np.array_equal(_np(out._tiles.indices).astype(np.int64), ids)
    assert ran == {"random": False, "plane": True}


def test_fused_adam_all_groups_with_mask_penalties(tgs):
    """tgs_adam_step_groups: every group in one launch + the mask penalties of total_loss
    (masking.py:60-67) vs optim.py:37-49 per group in float64."""
    from paper_2501_14534_b200 import optim
    from paper_2501_14534_b200.loss import SH_BAND_WEIGHTS
    rng = np.random.default_rng(1)
    sc = golden_io.load("fd16")
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    n = len(cloud)
    lrs = {f: 10 ** rng.uniform(-4, -1) for f in golden_io.FIELDS}
    opt = optim.Adam(cloud, lrs, eps=1e-15)
    lam_m, lam_sh = 0.05, 0.07
    p = {f: _np(getattr(cloud, f)).astype(np.float64) for f in golden_io.FIELDS}
    m = {f: np.zeros_like(p[f]) for f in golden_io.FIELDS}
    v = {f: np.zeros_like(p[f]) for f in golden_io.FIELDS}
    for step in range(1, 4):
        g = tgs.CloudGrads.zeros(n)
        grads = {}
        for f in golden_io.FIELDS:
            grads[f] = rng.standard_normal(p[f].shape).astype(np.float32)
            getattr(g, f).copy_(torch.from_numpy(grads[f]))
        opt.step(cloud, g, lambda_m=lam_m, lambda_sh=lam_sh)
        for f in golden_io.FIELDS:
            gr = grads[f].astype(np.float64)
            s = 1.0 / (1.0 + np.exp(-p[f]))
            if f == "mask_logits":
                gr = gr + lam_m * s * (1 - s) / n
            elif f == "sh_mask_logits":
                gr = gr + lam_sh * s * (1 - s) * np.asarray(SH_BAND_WEIGHTS) / n
            if f in ("mask_logits", "sh_mask_logits"):
                np.testing.assert_allclose(_np(getattr(g, f)), gr, rtol=1e-5, atol=1e-7, err_msg=f)
            m[f] = 0.9 * m[f] + 0.1 * gr
            v[f] = 0.999 * v[f] + 0.001 * gr * gr
            p[f] = p[f] - lrs[f] * (m[f] / (1 - 0.9 ** step)) / (np.sqrt(v[f] / (1 - 0.999 ** step)) + 1e-15)
    for f in golden_io.FIELDS:
        np.testing.assert_allclose(_np(getattr(cloud, f)), p[f], rtol=2e-5, atol=2e-6, err_msg=f)


def test_bin_tiles_huge_grid_multi_slab(tgs):
    """Raw-array bin_tiles on a 16384 x 16384 image (1,048,576 tiles, 128 x 128 super-tiles):
    the chunk x super-tile counts run in two row slabs.  Bit-exact vs the float32 oracle."""
    rng = np.random.default_rng(7)
    n, W, H, ts = 3000, 16384, 16384, 16
    means = rng.uniform(-300, W + 300, (n, 2)).astype(np.float32)
    radii = rng.uniform(2.0, 400.0, n).astype(np.float32)
    depths = rng.uniform(1.0, 10.0, n).astype(np.float32)
    b = tgs.bin_tiles(means, radii, depths, W, H, ts)
    sp = np.zeros((n, 12), dtype=np.float32)
    sp[:, 0:2], sp[:, 9], sp[:, 10] = means, depths, radii
    f16 = np.float32(ts)
    tx, ty = W // ts, H // ts
    x0 = np.clip(np.floor((means[:, 0] - radii) / f16), 0, tx - 1)
    x1 = np.clip(np.floor((means[:, 0] + radii) / f16), 0, tx - 1)
    y0 = np.clip(np.floor((means[:, 1] - radii) / f16), 0, ty - 1)
    y1 = np.clip(np.floor((means[:, 1] + radii) / f16), 0, ty - 1)
    on = ((means[:, 0] + radii >= 0) & (means[:, 0] - radii <= W - 1) & (means[:, 1] + radii >= 0) &
          (means[:, 1] - radii <= H - 1) & (radii > 0))
    tt = np.where(on, (x1 - x0 + 1) * (y1 - y0 + 1), 0).astype(np.int32)
    off, ids, _, _ = oracle.bin_tiles(sp, tt, W, H, ts, "f32")
    assert np.array_equal(_np(b.offsets).astype(np.int64), off)
    assert np.array_equal(_np(b.indices).astype(np.int64), ids)


def test_deterministic_backward_reproducible_and_exact(tgs):
    """deterministic=True: bitwise identical gradients run to run, within the north-star
    tolerance of the float64 oracle, and equal (up to reassociation) to the atomic path."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.config1()
    st = tgs.RenderSettings(near=0.2)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    cam = sc.cameras[0]
    dimg = np.random.default_rng(3).standard_normal((cam.height, cam.width, 3)).astype(np.float32)
    dt = torch.from_numpy(dimg).cuda()
    out = tgs.render_forward(cloud, cam, st)
    g1 = tgs.render_backward(cloud, cam, st, dt, out, deterministic=True)
    g2 = tgs.render_backward(cloud, cam, st, dt, out, deterministic=True)
    ga = tgs.render_backward(cloud, cam, st, dt, out)
    assert torch.equal(g1.flat, g2.flat)
    ref = oracle.render_forward(sc.fields, cam, st, "f64")
    rg = oracle.render_backward(sc.fields, cam, st, dimg.astype(np.float64), ref, "f64")
    for f in golden_io.FIELDS:
        a, b = _np(getattr(g1, f)), rg[f]
        assert np.linalg.norm(a - b) <= 1e-4 * max(np.linalg.norm(b), 1e-30), f
        np.testing.assert_allclose(a, _np(getattr(ga, f)), rtol=1e-4, atol=1e-6 * max(1.0, np.abs(b).max()),
                                   err_msg=f)


def test_trainer_deterministic_steps_bitwise_reproducible(tgs):
    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.train import Trainer
    sc = scenes.small_scene(seed=31, n=20_000, width=160, height=120, dist=3.5)
    rng = np.random.default_rng(4)
    cams = [scenes.pinhole(rng.uniform(3.0, 4.5) * d / np.linalg.norm(d), 160, 120) for d in rng.normal(size=(4, 3))]
    targets = [torch.from_numpy(rng.uniform(0, 1, (120, 160, 3)).astype(np.float32)).cuda() for _ in cams]
    st = tgs.RenderSettings(near=0.2, mask_threshold=0.01)
    flats = []
    for _ in range(2):
        cloud = tgs.GaussianCloud.from_fields(sc.fields)
        tr = Trainer(cloud, cams, targets, st, deterministic=True)
        for _ in range(3):
            tr.step()
        torch.cuda.synchronize()
        flats.append(cloud.flat.clone())
    assert torch.equal(flats[0], flats[1])


def test_multiview_preprocess_bitwise_equals_single_view(tgs):
    """tgs_preprocess_forward_views == tgs_preprocess_forward per view, bit for bit."""
    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.rasterizer import preprocess, preprocess_views
    sc = scenes.small_scene(seed=41, n=30_000, width=200, height=150, dist=3.0)
    rng = np.random.default_rng(2)
    cams = [scenes.pinhole(rng.uniform(2.5, 4.5) * d / np.linalg.norm(d), 200, 150) for d in rng.normal(size=(11, 3))]
    for deg in (0, 3):
        st = tgs.RenderSettings(near=0.2, active_sh_degree=deg, mask_threshold=0.3)
        cloud = tgs.GaussianCloud.from_fields(sc.fields)
        many = preprocess_views(cloud, cams, st)
        for cam, got in zip(cams, many):
            want = preprocess(cloud, cam, st)
            for a, b in zip(got[:4] + got[5:], want[:4] + want[5:]):
                assert torch.equal(a.view(torch.int32) if a.dtype == torch.float32 else a,
                                   b.view(torch.int32) if b.dtype == torch.float32 else b)


def test_significance_vs_reference_golden(tgs):
    """significance.py:31-99 on the CUDA path against the reference's own outputs
    (tests/golden/significance.npz) and the oracle restatement."""
    from oracle import significance_ref as sig_ref
    from paper_2501_14534_b200 import significance as sig
    cases, z = golden_io.load_significance()
    for tag, c in cases.items():
        cloud = tgs.GaussianCloud.from_fields(c.fields)
        st = _settings(tgs, c.settings)
        hits = sig.count_hits(cloud, c.cams, st)
        ref32 = sig_ref.count_hits(c.fields, c.cams, c.settings)  # float64 oracle == golden (pinned on CPU)
        assert np.array_equal(_np(hits), c.hits), tag
        assert np.array_equal(ref32, c.hits)
        rep = sig.significance_scores(hits, cloud, mask_threshold=float(z["mask_threshold"]),
                                      volume_power=float(z["volume_power"]))
        vol, vn, sc = _np(rep.volumes), _np(rep.v_norm), _np(rep.scores)
        np.testing.assert_allclose(vol, c.volumes, rtol=2e-6, atol=0)
        np.testing.assert_allclose(vn, c.v_norm, rtol=2e-6, atol=0)
        np.testing.assert_allclose(sc, c.scores, rtol=4e-6, atol=0)
        # V90 is exactly the nearest-rank order statistic of the device volumes, and
        # v_norm follows from it in float32 (IEEE division and square root)
        v90 = np.sort(vol)[sig_ref.rank90(vol.size)]
        want = np.sqrt(np.minimum(vol / v90, np.float32(1))) if v90 > 0 else (vol > 0).astype(np.float32)
        assert np.array_equal(vn, want.astype(np.float32)), tag
        # the kept rows: exactly the reference's lexsort rule applied to these scores,
        # and the reference's own set
        _, keep = sig.prune_by_significance(cloud, rep.scores, float(z["rate"]))
        assert np.array_equal(_np(keep), sig_ref.prune_keep(sc, float(z["rate"]))), tag
        assert np.array_equal(_np(keep), c.keep), tag


def test_significance_selection_ties_and_edges(tgs):
    """Radix selection at 1M rows with heavy ties (lexsort tie break by index),
    all-equal scores, k == 0, n == 1, and the reference's error conditions."""
    from oracle import significance_ref as sig_ref
    from paper_2501_14534_b200 import significance as sig
    rng = np.random.default_rng(5)
    for n, levels, rate in ((1_000_000, 37, 0.3), (100_003, 2, 0.5), (4097, 1, 0.9), (10, 1000, 0.05)):
        s = (rng.integers(0, levels, n) * 0.25).astype(np.float32)
        got = _np(sig.prune_keep_indices(torch.from_numpy(s).cuda(), rate))
        assert np.array_equal(got, sig_ref.prune_keep(s, rate)), (n, levels, rate)
    s = rng.random(1_000_000, dtype=np.float32) * 1e-3  # distinct values, tiny magnitudes
    assert np.array_equal(_np(sig.prune_keep_indices(torch.from_numpy(s).cuda(), 0.77)), sig_ref.prune_keep(s, 0.77))
    one = torch.ones(1, device="cuda")
    assert _np(sig.prune_keep_indices(one, 0.5)).tolist() == [0]  # floor(0.5) == 0: nothing pruned
    with pytest.raises(tgs.ContractViolationError):
        sig.prune_keep_indices(one, 1.0)
    with pytest.raises(tgs.ContractViolationError):
        sig.prune_schedule(-1, 0.6, 0.5)
    with pytest.raises(tgs.ContractViolationError):
        sig.count_hits(tgs.GaussianCloud.from_fields(golden_io.load("fd16").fields), [], tgs.RenderSettings())
    empty = tgs.GaussianCloud.from_fields({k: v[:0] for k, v in golden_io.load("fd16").fields.items()})
    with pytest.raises(tgs.EmptySceneError):
        sig.significance_scores(torch.zeros(0, dtype=torch.int64), empty)


def test_trainer_densify_stats_and_significance_event(tgs):
    """Densification statistics (training.py:333-338) accumulated inside the
    multi-view preprocess kernels equal the per-view formula on the step's own
    partials; pruning compacts them with the cloud; a significance event
    (training.py:369-401) prunes floor(rate N) rows."""
    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.rasterizer import preprocess_views
    from paper_2501_14534_b200.train import Trainer
    sc = scenes.small_scene(seed=31, n=3000, width=96, height=64, dist=3.5)
    rng = np.random.default_rng(31)
    cams = [sc.cameras[0]] + [scenes.pinhole(3.5 * scenes._unit(rng), 80 + 16 * k, 64, name=f"v{k}")
                              for k in range(2)]
    st = tgs.RenderSettings(near=0.2, mask_threshold=0.05, sh_mask_threshold=0.1)
    sc.fields["mask_logits"][:200] = -6.0  # masked rows: never visible, count stays 0
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    targets = [torch.rand((c.height, c.width, 3), device="cuda") for c in cams]
    tr = Trainer(cloud, cams, targets, st, densify_stats=True)
    tr.clear_partials = False  # keep the step's partials readable below
    before = tgs.GaussianCloud.from_fields(sc.fields)
    pres = preprocess_views(before, cams, st)
    tr.step()
    torch.cuda.synchronize()
    acc = np.zeros(len(cloud), np.float64)
    cnt = np.zeros(len(cloud), np.int64)
    amax = np.zeros(len(cloud), np.float32)
    for v, cam in enumerate(cams):
        vis = _np(pres[v][1]).astype(bool)
        ds = _np(tr.dsplats[v])
        norm = np.sqrt((ds[:, 0] * (cam.width / 2.0)) ** 2 + (ds[:, 1] * (cam.height / 2.0)) ** 2)
        acc[vis] += norm[vis]
        cnt[vis] += 1
        amax = np.maximum(amax, np.where(vis, _np(pres[v][0])[:, 11], 0.0).astype(np.float32))
    assert cnt.max() == len(cams) and (cnt == 0).any()
    assert np.array_equal(_np(tr.stats.grad_count), cnt)
    assert np.array_equal(_np(tr.stats.area_max), amax)
    np.testing.assert_allclose(_np(tr.stats.grad_accum), acc, rtol=1e-5, atol=1e-9)
    mg = _np(tr.stats.mean_grad())
    np.testing.assert_allclose(mg, np.where(cnt > 0, acc / np.maximum(cnt, 1), 0.0), rtol=1e-5, atol=1e-9)
    # mask pruning compacts the statistics with the cloud
    old = (_np(tr.stats.grad_accum), _np(tr.stats.grad_count), _np(tr.stats.area_max))
    keep = np.flatnonzero(_np(tr.cloud.mask_logits) > 0.0)
    tr.prune(0.5)  # sigmoid(m) > 0.5 <=> m > 0
    assert len(tr.cloud) == keep.size < len(cloud)
    for got, ref in zip((tr.stats.grad_accum, tr.stats.grad_count, tr.stats.area_max), old):
        assert np.array_equal(_np(got), ref[keep])
    n0 = len(tr.cloud)
    tr.step()  # the compacted state steps
    rep = tr.significance_prune(cams, st, rate=0.25)
    assert rep.scores.numel() == n0 and len(tr.cloud) == n0 - int(np.floor(0.25 * n0))
    assert tr.stats.grad_count.numel() == len(tr.cloud)
    tr.step()
    torch.cuda.synchronize()
    assert np.isfinite(_np(tr.terms)).all()


def test_render_views_equals_render_forward(tgs):
    """render_views (one multi-view preprocess pass, three streams) returns, view for
    view, exactly what render_forward returns."""
    from paper_2501_14534_b200 import scenes
    sc = scenes.small_scene(seed=41, n=20000, width=160, height=96, dist=3.0)
    rng = np.random.default_rng(41)
    cams = [sc.cameras[0]] + [scenes.pinhole(3.0 * scenes._unit(rng), 96 + 32 * (k % 3), 96, name=f"v{k}")
                              for k in range(6)]
    st = tgs.RenderSettings(near=0.2, record_hits=True)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    outs = tgs.render_views(cloud, cams, st)
    outs_again = tgs.render_views(cloud, cams, st, streams=2)
    for cam, o, o2 in zip(cams, outs, outs_again):
        ref = tgs.render_forward(cloud, cam, st)
        for f in ("image", "transmittance", "weight_sum", "n_contrib", "last_pos", "visible", "screen_areas",
                  "hit_counts"):
            assert torch.equal(getattr(o, f), getattr(ref, f)), f
            assert torch.equal(getattr(o2, f), getattr(ref, f)), f
        assert torch.equal(o._tiles.indices, ref._tiles.indices) and torch.equal(o._tiles.offsets, ref._tiles.offsets)
    assert tgs.render_views(cloud, [], st) == []
    # the native batch path (tgs_render_views, used once a geometry's counts are known)
    # recovers from a too-small id capacity: grow, retry, same results
    from paper_2501_14534_b200 import rasterizer
    sizes = tuple((int(c.width), int(c.height)) for c in cams)
    geom = next(k for k in rasterizer._RV_CAP if k[1] == len(cloud) and k[3] == sizes)
    rasterizer._RV_CAP[geom] = 1024
    outs3 = tgs.render_views(cloud, cams, st)
    assert rasterizer._RV_CAP[geom] >= max(o._tiles.indices.numel() for o in outs3)
    for cam, o in zip(cams, outs3):
        ref = tgs.render_forward(cloud, cam, st)
        for f in ("image", "transmittance", "n_contrib", "last_pos", "visible", "hit_counts"):
            assert torch.equal(getattr(o, f), getattr(ref, f)), f


def test_tile_order_is_a_heaviest_first_permutation_and_changes_nothing(tgs):
    """Blend launch orders (centre-out default, heaviest-first tgs_tile_order): both
    are permutations of the tiles, the LPT one with non-increasing
    floor(log2(list length)); the forward blend gives the same bits under any order
    and without one (the order only schedules CTAs)."""
    import ctypes
    from paper_2501_14534_b200 import _lib, scenes
    sc = scenes.small_scene(seed=51, n=30000, width=200, height=136, dist=3.0)
    st = tgs.RenderSettings(near=0.2)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    cam = sc.cameras[0]
    from paper_2501_14534_b200 import rasterizer
    out = tgs.render_forward(cloud, cam, st)  # default launch order (centre-out)
    bins = out._tiles
    nt = bins.offsets.numel() - 1
    assert np.array_equal(np.sort(_np(bins.order)), np.arange(nt))
    prev = rasterizer.BLEND_ORDER
    rasterizer.BLEND_ORDER = "lpt"
    try:
        out_lpt = tgs.render_forward(cloud, cam, st)
    finally:
        rasterizer.BLEND_ORDER = prev
    for f in ("image", "transmittance", "weight_sum", "n_contrib", "last_pos"):
        assert torch.equal(getattr(out_lpt, f), getattr(out, f))
    order = _np(out_lpt._tiles.order[:nt])
    assert np.array_equal(np.sort(order), np.arange(nt))
    lens = np.diff(_np(bins.offsets))[order]
    cls = np.floor(np.log2(np.maximum(lens, 1)))
    assert (np.diff(cls) <= 0).all() and lens[0] == lens.max()
    # raw ABI: same image without an order
    h, w = cam.height, cam.width
    bufs = [torch.empty((h, w, 3), device="cuda"), torch.empty((h, w), device="cuda"),
            torch.empty((h, w), device="cuda"), torch.empty((h, w), dtype=torch.int32, device="cuda"),
            torch.empty((h, w), dtype=torch.int32, device="cuda")]
    c_cam, c_set = _lib.make_camera(cam), _lib.make_settings(st)
    _lib.call("tgs_blend_forward", _lib.ptr(out._state.splats), _lib.ptr(out._state.exact), _lib.ptr(bins.offsets),
              _lib.ptr(bins.indices),
              ctypes.byref(c_cam), ctypes.byref(c_set), 0, bins.tiles_y, *[_lib.ptr(b) for b in bufs], None, None,
              None, None, _lib.stream_handle())
    for got, ref in zip(bufs, (out.image, out.transmittance, out.weight_sum, out.n_contrib, out.last_pos)):
        assert torch.equal(got, ref)
    # random offsets with empty tiles and a single huge tile
    rng = np.random.default_rng(3)
    ln = rng.integers(0, 3000, 40000).astype(np.int32)
    ln[rng.choice(40000, 5000, replace=False)] = 0
    ln[123] = 1 << 22
    offs = torch.from_numpy(np.concatenate([[0], np.cumsum(ln)]).astype(np.int32)).cuda()
    o = torch.empty(40000 + 64, dtype=torch.int32, device="cuda")
    _lib.call("tgs_tile_order", _lib.ptr(offs), 40000, _lib.ptr(o), _lib.stream_handle())
    oo = _np(o[:40000])
    assert np.array_equal(np.sort(oo), np.arange(40000)) and oo[0] == 123
    c2 = np.floor(np.log2(np.maximum(ln[oo], 1)))  # lengths 0 and 1 share the lightest class
    assert (np.diff(c2) <= 0).all()


def test_render_views_native_mixed_batches_and_errors(tgs):
    """tgs_render_views (native batch driver) on batches mixing resolutions, 8-px tiles,
    a cloud that grows after its capacities were learned (retry on TGS_ERR_CAPACITY),
    degenerate rotations (DegenerateRotationError through the driver) and an empty cloud."""
    from paper_2501_14534_b200 import rasterizer, scenes
    sc = scenes.small_scene(seed=71, n=15000, width=160, height=96, dist=3.0)
    rng = np.random.default_rng(71)
    cams = [scenes.pinhole(3.0 * scenes._unit(rng), (96, 160, 200)[k % 3], (64, 96, 80)[k % 3], name=f"m{k}")
            for k in range(7)]
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    for ts in (16, 8):
        st = tgs.RenderSettings(near=0.2, tile_size=ts)
        for _ in range(2):  # first call learns the capacities (Python pipeline), second is native
            outs = tgs.render_views(cloud, cams, st)
        geom = (0, len(cloud), ts, tuple((c.width, c.height) for c in cams))
        assert geom in rasterizer._RV_CAP
        for cam, o in zip(cams, outs):
            ref = tgs.render_forward(cloud, cam, st)
            assert torch.equal(o.image, ref.image) and torch.equal(o.last_pos, ref.last_pos)
            assert torch.equal(o._tiles.indices, ref._tiles.indices)
    # grow the splats after the capacity was learned: more instances than the capacity
    st = tgs.RenderSettings(near=0.2)
    tgs.render_views(cloud, cams, st)
    big = dict(sc.fields)
    big["log_scales"] = sc.fields["log_scales"] + 1.2
    cloud_big = tgs.GaussianCloud.from_fields(big)
    outs = tgs.render_views(cloud_big, cams, st)  # same geometry key (n, sizes): retries natively
    for cam, o in zip(cams, outs):
        ref = tgs.render_forward(cloud_big, cam, st)
        assert torch.equal(o.image, ref.image) and o._tiles.indices.numel() == ref._tiles.indices.numel()
    # a degenerate rotation raises through the driver
    bad = dict(sc.fields)
    bad["rotations"] = sc.fields["rotations"].copy()
    bad["rotations"][5] = 0.0
    with pytest.raises(tgs.DegenerateRotationError):
        tgs.render_views(tgs.GaussianCloud.from_fields(bad), cams, st)
    empty = tgs.GaussianCloud.from_fields({k: v[:0] for k, v in sc.fields.items()})
    outs = tgs.render_views(empty, cams[:2], st)
    assert all(float(o.transmittance.min()) == 1.0 for o in outs)


def test_adam_subset_of_groups_leaves_other_fields_untouched(tgs):
    """tgs_adam_step_groups on groups that do not start at offset 0 (the data-parallel
    buckets: sh_rest alone, the two mask groups): only those groups move."""
    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.cloud import PARAM_FIELDS, CloudGrads
    from paper_2501_14534_b200.optim import Adam
    sc = scenes.small_scene(seed=91, n=3000, width=64, height=64)
    for names in (("sh_rest",), ("mask_logits", "sh_mask_logits"), ("rotations", "sh_dc")):
        cloud = tgs.GaussianCloud.from_fields(sc.fields)
        before = cloud.flat.clone()
        g = CloudGrads(len(cloud), cloud.device)
        g.flat.normal_()
        opt = Adam(cloud, {f: 0.01 for f in PARAM_FIELDS})
        opt.step(cloud, g, names=names, lambda_m=0.05, lambda_sh=0.05)
        torch.cuda.synchronize()
        for f in PARAM_FIELDS:
            o, n = cloud.field_range(f)
            moved = not torch.equal(cloud.flat[o:o + n], before[o:o + n])
            assert moved == (f in names), (names, f)
            if f not in names:
                assert float(opt.m[o:o + n].abs().max()) == 0.0, (names, f)


def test_trainer_host_targets_equal_device_targets(tgs):
    """Trainer.step(host_targets=...) (per-view copies from pinned host memory on a copy
    stream, each view's loss waiting only for its own copy: the bench's e2e path) gives
    the same step as device-resident targets, bit for bit (deterministic reduction)."""
    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.train import Trainer
    sc = scenes.small_scene(seed=93, n=8000, width=128, height=96, dist=3.0)
    rng = np.random.default_rng(93)
    cams = [sc.cameras[0]] + [scenes.pinhole(3.0 * scenes._unit(rng), 128, 96, name=f"h{k}") for k in range(3)]
    host = {v: torch.rand((c.height, c.width, 3), generator=torch.Generator().manual_seed(v)).pin_memory()
            for v, c in enumerate(cams)}
    st = tgs.RenderSettings(near=0.2)
    out = []
    for use_host in (True, False):
        cloud = tgs.GaussianCloud.from_fields(sc.fields)
        dev_t = [torch.zeros((c.height, c.width, 3), device="cuda") if use_host else host[v].cuda()
                 for v, c in enumerate(cams)]
        tr = Trainer(cloud, cams, dev_t, st, deterministic=True)
        for _ in range(2):
            tr.step(host_targets=host if use_host else None)
        torch.cuda.synchronize()
        out.append((tr.cloud.flat.clone(), tr.terms.clone()))
    assert torch.equal(out[0][1], out[1][1])
    assert torch.equal(out[0][0], out[1][0])


@pytest.mark.parametrize("hw", [(11, 11), (13, 17), (33, 40), (31, 64), (45, 19)])
def test_loss_small_and_odd_images(tgs, hw):
    """The loss on images smaller than one 32x32 tile or one TMA halo box (42 x 44/48),
    odd widths (padded partial row pitch): vs oracle/loss_ref.py."""
    from oracle import loss_ref
    from paper_2501_14534_b200 import loss
    h, w = hw
    rng = np.random.default_rng(h * 100 + w)
    img = rng.uniform(0, 1, (h, w, 3)).astype(np.float32)
    tgt = np.clip(img + rng.normal(0, 0.2, img.shape), 0, 1).astype(np.float32)
    terms, d = loss.l1_ssim(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), 0.2)
    l1, dssim, dref = loss_ref.total_loss_image(img, tgt, 0.2)
    assert abs(terms["l1"] - l1) < 1e-6 and abs(terms["d_ssim"] - dssim) < 1e-5
    np.testing.assert_allclose(_np(d), dref, rtol=1e-3, atol=1e-4 * np.abs(dref).max())


def test_preprocess_row_shards_equal_full_cloud(tgs):
    """dp_mode="gaussians" runs the multi-view preprocess forward, the exact records and the
    preprocess backward over a rank's rows only: the shards' outputs, gradients and
    densification statistics put together equal the whole-cloud calls bit for bit
    (4,999 rows in 3 shards, the last uneven)."""
    from paper_2501_14534_b200 import parallel, scenes
    from paper_2501_14534_b200.rasterizer import exact_records, preprocess_backward_views, preprocess_views
    from paper_2501_14534_b200.train import DensifyStats
    sc = scenes.small_scene(seed=41, n=4999, width=96, height=64, dist=3.5)
    rng = np.random.default_rng(41)
    cams = [sc.cameras[0]] + [scenes.pinhole(3.5 * scenes._unit(rng), 80, 64, name=f"s{k}") for k in range(2)]
    st = tgs.RenderSettings(near=0.2, mask_threshold=0.05, sh_mask_threshold=0.1)
    cloud = tgs.GaussianCloud.from_fields(sc.fields)
    n = len(cloud)
    st_full = DensifyStats(n, cloud.device)
    full = preprocess_views(cloud, cams, st, stats=st_full, exact=False)
    exact_records(cloud, cams, st, full)
    g = torch.Generator("cuda").manual_seed(41)
    ds = [torch.randn((n, 9), device="cuda", generator=g) for _ in cams]
    gr_full = preprocess_backward_views(cloud, cams, st, [p[1] for p in full], ds, tgs.CloudGrads.zeros(n),
                                        stats=st_full)
    st_sh = DensifyStats(n, cloud.device)
    gr_sh = tgs.CloudGrads.zeros(n)
    for a, b in parallel.shard_rows(n, 3):
        sub = preprocess_views(cloud, cams, st, stats=st_sh, exact=False, rows=(a, b))
        exact_records(cloud, cams, st, sub, rows=(a, b))
        for v in range(len(cams)):
            for kind in (0, 1, 2, 3, 5):
                assert torch.equal(sub[v][kind], full[v][kind][a:b]), (a, v, kind)
        preprocess_backward_views(cloud, cams, st, [p[1] for p in sub], [d[a:b].contiguous() for d in ds], gr_sh,
                                  stats=st_sh, rows=(a, b), local=True)
    assert torch.equal(gr_sh.flat, gr_full.flat)
    for f in ("grad_accum", "grad_count", "area_max"):
        assert torch.equal(getattr(st_sh, f), getattr(st_full, f)), f


def test_gaussian_sharded_trainer_single_rank_nccl(tgs):
    """Trainer(dp_mode="gaussians") through a real NCCL group (world size 1 on this box:
    the all-to-alls deliver every row): the step's loss terms equal the one-GPU step's
    bit for bit and its gradient agrees to float32 atomics-order noise; with learning
    rates the parameters after two steps agree likewise."""
    import socket

    import torch.distributed as dist

    from paper_2501_14534_b200 import scenes
    from paper_2501_14534_b200.train import Trainer
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        sc = scenes.small_scene(seed=43, n=20_000, width=200, height=120, dist=3.0)
        rng = np.random.default_rng(43)
        cams = [sc.cameras[0]] + [scenes.pinhole(3.0 * scenes._unit(rng), 160, 96, name=f"g{k}") for k in range(3)]
        st = tgs.RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
        tg = [torch.rand((c.height, c.width, 3), device="cuda", generator=torch.Generator("cuda").manual_seed(k))
              for k, c in enumerate(cams)]
        res = {}
        for mode in ("gaussians", "one_gpu"):
            c2 = tgs.GaussianCloud.from_fields(sc.fields)
            kw = dict(process_group=dist.group.WORLD, dp_mode="gaussians") if mode == "gaussians" else {}
            tr = Trainer(c2, cams, [t.clone() for t in tg], st, densify_stats=True, **kw)
            lrs = dict(tr.opt.lrs)
            for f in lrs:
                tr.opt.set_lr(f, 0.0)
            tr.step()
            torch.cuda.synchronize()
            terms, grads = tr.terms.clone(), tr.grads.flat.clone()
            # the same step with the targets streamed from pinned host memory (the e2e path)
            host = {v: t.cpu().pin_memory() for v, t in enumerate(tg)}
            tr.step(host_targets=host)
            torch.cuda.synchronize()
            assert torch.equal(tr.terms, terms), mode
            for f, lr in lrs.items():
                tr.opt.set_lr(f, lr)
            tr.step()
            tr.step()
            tr.check_divergence()
            torch.cuda.synchronize()
            res[mode] = (terms, grads, tr.cloud.flat.clone(), tr.stats.grad_count.clone())
        a, b = res["gaussians"], res["one_gpu"]
        assert torch.equal(a[0], b[0])
        scale = float(b[1].abs().max())
        torch.testing.assert_close(a[1], b[1], rtol=1e-3, atol=1e-5 * scale)
        torch.testing.assert_close(a[2], b[2], rtol=1e-4, atol=1e-4)
        assert torch.equal(a[3], b[3])
    finally:
        dist.destroy_process_group()
