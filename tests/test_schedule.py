"""Progressive hooks vs the reference's outputs (CPU only, tests/golden/schedule.npz)."""

import numpy as np
import pytest

import golden_io
from paper_2501_14534_b200 import schedule as S

Z = dict(np.load(f"{golden_io.GOLDEN}/schedule.npz"))


def test_resolution_at_matches_reference():
    for mode, i, rs, re_, tau, want in Z["res"]:
        assert S.resolution_at(int(i), int(rs), int(re_), int(tau), "linear" if mode == 0 else "logarithmic") == want


def test_lowpass_s_at_matches_reference():
    for n, h, w, want in Z["lowpass"]:
        assert S.lowpass_s_at(int(n), int(h), int(w)) == pytest.approx(want, rel=0, abs=0)


def test_blur_at_matches_reference():
    decay = S.default_blur_decay(2.4, 100, 19500, 0.3)
    assert decay == float(Z["decay"])
    for i, down, size, sigma in Z["blur"]:
        b = S.blur_at(int(i), S.BlurSpec(9, 2.4), 100, decay, 19500, float(down))
        assert b.size == int(size) and b.sigma == pytest.approx(sigma, rel=1e-15)


def test_phase_at_matches_reference():
    tl = S.Timeline()
    names = [str(n) for n in Z["phase_names"]]
    for i, row in zip(Z["phase_its"], Z["phases"]):
        got = S.phase_at(int(i), tl)
        assert [n in got for n in names] == [bool(v) for v in row]


def test_contracts():
    with pytest.raises(S.ConfigError):
        S.resolution_at(0, 0, 10, 5)
    with pytest.raises(S.ContractViolationError):
        S.lowpass_s_at(0, 4, 4)
    with pytest.raises(S.ContractViolationError):
        S.BlurSpec(4, 1.0)
    assert S.active_sh_degree(0) == 0 and S.active_sh_degree(2500) == 2 and S.active_sh_degree(10**6) == 3
    assert S.Timeline().scaled(3000).mask_prune_interval == 50


def test_config5_sfm_follows_the_reference_seeding_recipe():
    """scenes.config5_sfm restates synthetic.make_scene + schedule.seed_from_sfm: seeds
    near ground-truth centres, isotropic kNN scales, identity rotations, opacity 0.1,
    mask logits 2.0."""
    import numpy as np
    from scipy.spatial import cKDTree

    from paper_2501_14534_b200 import scenes
    sc, gt = scenes.config5_sfm(n=3000, n_gt=150, width=64, height=48, views=2)
    f = sc.fields
    assert f["positions"].shape == (3000, 3) and gt["positions"].shape == (150, 3)
    d, _ = cKDTree(gt["positions"]).query(f["positions"])
    assert np.quantile(d, 0.9) < 4.0 * np.exp(gt["log_scales"]).max()
    assert np.all(f["log_scales"][:, 0] == f["log_scales"][:, 2])
    assert np.all(f["rotations"] == np.array([1, 0, 0, 0], dtype=np.float32))
    assert np.allclose(1.0 / (1.0 + np.exp(-f["opacity_logits"])), 0.1)
    assert np.all(f["mask_logits"] == 2.0) and np.all(f["sh_mask_logits"] == 2.0)
    op = 1.0 / (1.0 + np.exp(-gt["opacity_logits"]))
    assert op.min() >= 0.55 - 1e-6 and op.max() <= 0.95 + 1e-6
    assert len(sc.cameras) == 2 and sc.cameras[0].width == 64
