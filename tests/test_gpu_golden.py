"""The device path against the frozen oracle goldens (tests/golden/lvigs_crop.npz): a crop of
the bench's synthetic workload (4000 Gaussians, 160x128, colourised-LiDAR training map).
Bars as elsewhere: depth order, projected depths, tile lists and contributor counts exact;
images <= 1e-4; gradients within 1e-3 (group-normwise, tests/_common.py); training steps track
the oracle's losses and stay within a few Adam steps of its parameters."""
import os

import numpy as np
import pytest

from tests._common import grad_errors

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "lvigs_crop.npz")
LR = np.array([1.6e-4] * 3 + [1e-3] * 4 + [5e-3] * 3 + [5e-2] + [2.5e-3] * 48)


def G():
    from paper_2411_02703_b200 import gsmap
    return gsmap


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def setup(gold):
    from oracle import pyoracle as O
    gs = O.empty_gaussians(len(gold["train_p"]))
    gs["p"] = gold["train_p"]
    gs["degree"] = gold["train_degree"]
    fx, fy, cx, cy, w, h = gold["camera"]
    cam = G().Camera(fx, fy, cx, cy, int(w), int(h))
    pose = G().Pose(*gold["pose0"])
    return gs, cam, pose


def test_render_matches_goldens(gold):
    gs, cam, pose = setup(gold)
    m = G().GaussianMap(None, gs)
    out = G().render(m, pose, cam)
    pr = out.projected()
    np.testing.assert_array_equal(pr["index"], gold["order"])
    np.testing.assert_array_equal(pr["depth"], gold["depth_sorted"])
    off, ent = out.tiles()
    np.testing.assert_array_equal(off, gold["tile_off"])
    np.testing.assert_array_equal(ent, gold["tile_gid"])
    nc, _ = out.pixel_state()
    np.testing.assert_array_equal(nc, gold["n_contrib"])
    for k, g in (("color", out.color), ("depth", out.depth), ("visibility", out.visibility)):
        assert np.abs(g - gold[k].astype(np.float64)).max() <= 1e-4, k


def test_backward_matches_goldens(gold):
    gs, cam, pose = setup(gold)
    m = G().GaussianMap(None, gs)
    out = G().render(m, pose, cam)
    H, W = gold["color"].shape[:2]
    gg = G().render_backward(m, pose, cam, out, gold["c1_dl_dcolor"].astype(np.float64), np.zeros((H, W))).read()
    e, ge = grad_errors(gg, gold["c1_grads"], gs)
    assert (ge <= 1e-3).mean() >= 0.999 and ge.max() < 1e-2, ge.max()
    assert (e <= 1e-3).mean() >= 0.995, (e > 1e-3).sum()


@pytest.mark.parametrize("which", ["c1", "c3"])
def test_training_tracks_goldens(gold, which):
    gs, cam, pose = setup(gold)
    m = G().GaussianMap(None, gs)
    extent = m.scene_extent
    gt = gold["gt_color"].astype(np.float64)
    sparse = gold["sparse_depth"].astype(np.float64)
    if which == "c1":
        kf = G().Keyframe(pose, gt, sparse, 3, 0)
        cfg = G().TrainConfig.make(0.0, 0.0, 0)
        reps = [G().train_keyframe_step(m, kf, cfg, cam) for _ in range(3)]
        for r, lo in zip(reps, gold["c1_step_losses"]):
            assert r["loss"] == pytest.approx(lo, rel=2e-3)
        final, steps = gold["c1_params"], 3
    else:
        kf = G().Keyframe(pose, gt, sparse, 6, 2)
        cfg = G().TrainConfig.make(0.2, 0.5, 2, 2)
        reps = [G().train_keyframe_step(m, kf, cfg, cam) for _ in range(6)]
        assert [r["level"] for r in reps] == list(gold["c3_step_levels"])
        for r, lo in zip(reps, gold["c3_step_losses"]):
            assert r["loss"] == pytest.approx(lo, rel=2e-3)
        final, steps = gold["c3_params"], 6
    lr = LR.copy()
    lr[:3] *= extent
    d = np.abs(m.gaussians["p"] - final)
    assert np.all(d <= steps * 2 * lr + 1e-6)
    assert np.mean(d <= 0.05 * lr + 1e-6) > 0.95
