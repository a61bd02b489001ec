"""Checkpoint v1 (io/checkpoint.cpp) and per-frame evaluation (pipeline.cpp:34-64) on the device
map, against the CPU oracle's restatement (test_io.cpp:190-207, test_pipeline.cpp:128-146)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from tests._common import gpu_cam, gpu_pose, pair, random_scene, round32

pytestmark = pytest.mark.gpu


def G():
    from paper_2411_02703_b200 import gsmap
    return gsmap


def q8(img):
    return np.floor(np.clip(img, 0.0, 1.0) * 255.0 + 0.5) / 255.0


def test_checkpoint_bytes_match_oracle(tmp_path):  # io/checkpoint.cpp:17-35
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    om, gm = pair(random_scene(4, 500, cam, O.pose()))
    om.raise_sh_degree(2); gm.raise_sh_degree(2)
    O.save_checkpoint(str(tmp_path / "o.gsmap"), om)
    gm.save_checkpoint(str(tmp_path / "g.gsmap"))
    assert (tmp_path / "o.gsmap").read_bytes() == (tmp_path / "g.gsmap").read_bytes()


def test_checkpoint_load_and_round_trip(tmp_path):  # test_io.cpp:190-207 on the device
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    g = random_scene(4, 300, cam, O.pose())
    om = O.OracleMap(g)  # fp64 parameters: the device load rounds them to its fp32 store
    O.save_checkpoint(str(tmp_path / "o.gsmap"), om)
    gm = G().GaussianMap.load_checkpoint(str(tmp_path / "o.gsmap"))
    assert len(gm) == 300
    np.testing.assert_array_equal(gm.gaussians["p"], round32(g)["p"])
    np.testing.assert_array_equal(gm.gaussians["degree"], g["degree"])
    m, v, steps = gm.adam_state()
    assert np.all(m == 0) and np.all(v == 0) and np.all(steps == 0)
    assert gm.scene_extent == pytest.approx(O.OracleMap(round32(g)).scene_extent, rel=1e-12)
    # device save -> device load renders bit-exactly (the reference's round-trip property)
    gm.save_checkpoint(str(tmp_path / "g.gsmap"))
    gl = G().load_checkpoint(str(tmp_path / "g.gsmap"), gm.ctx)
    np.testing.assert_array_equal(gl.gaussians["p"], gm.gaussians["p"])
    a = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    b = G().render(gl, gpu_pose(O.pose()), gpu_cam(cam))
    np.testing.assert_array_equal(a.color, b.color)
    np.testing.assert_array_equal(a.depth, b.depth)


def test_checkpoint_errors(tmp_path):  # test_io.cpp:204-206 + the header checks
    with pytest.raises(RuntimeError, match="cannot open"):
        G().load_checkpoint(str(tmp_path / "missing.gsmap"))
    (tmp_path / "junk.gsmap").write_text("not a checkpoint\n")
    with pytest.raises(RuntimeError, match="not a checkpoint file"):
        G().load_checkpoint(str(tmp_path / "junk.gsmap"))
    (tmp_path / "v2.gsmap").write_text("gsmap-checkpoint 2\ncount 0\nend_header\n")
    with pytest.raises(RuntimeError, match="unsupported version"):
        G().load_checkpoint(str(tmp_path / "v2.gsmap"))
    (tmp_path / "short.gsmap").write_bytes(b"gsmap-checkpoint 1\ncount 3\nsh_degree 0\nend_header\n" + bytes(476 * 2))
    with pytest.raises(RuntimeError, match="truncated"):
        G().load_checkpoint(str(tmp_path / "short.gsmap"))
    (tmp_path / "empty.gsmap").write_text("gsmap-checkpoint 1\ncount 0\nsh_degree 0\nend_header\n")
    assert len(G().load_checkpoint(str(tmp_path / "empty.gsmap"))) == 0
    with pytest.raises(RuntimeError, match="cannot open"):
        G().GaussianMap().save_checkpoint(str(tmp_path / "no_dir" / "x.gsmap"))


def test_evaluate_gt_map_scores_sentinel():  # test_pipeline.cpp:128-146
    cam = O.camera(55, 55, 31.5, 23.5, 64, 48)
    om, gm = pair(random_scene(5, 60, cam, O.pose()))
    out = O.render(om, O.pose(), cam)
    stored = q8(out.color)
    r = G().evaluate_view(gm, gpu_pose(O.pose()), gpu_cam(cam), stored, out.depth)
    # a quantization level can flip where the fp64 colour sits within the fp32 render's error
    # of a k + 0.5 boundary; one flip in 9216 values still scores ~88 dB
    assert r["psnr"] == 100.0 or r["psnr"] > 80.0
    assert r["ssim"] == pytest.approx(1.0, abs=1e-5)
    assert r["depth_rmse"] == pytest.approx(0.0, abs=1e-5)
    assert np.isnan(G().evaluate_view(gm, gpu_pose(O.pose()), gpu_cam(cam), stored)["depth_rmse"])


@pytest.mark.parametrize("seed", [1, 2])
def test_evaluate_matches_oracle(seed):  # pipeline.cpp:46-60 per frame
    cam = O.camera(300, 300, 159.5, 119.5, 320, 240)
    pose = O.pose(1, 0.01, -0.02, 0.0, t=(0.02, 0.0, 0.05))
    om, gm = pair(random_scene(seed, 2000, cam, pose))
    gt_map = O.random_scene(O.Rng(seed + 10), 2000, cam, pose)
    gt = O.render(gt_map, pose, cam)
    gc = q8(gt.color)
    gen = np.random.default_rng(seed)
    gd = np.where(gen.uniform(size=(240, 320)) < 0.2, gt.depth, 0.0)
    ro = O.evaluate_view(om, pose, cam, gc, gd)
    rg = G().evaluate_view(gm, gpu_pose(pose), gpu_cam(cam), gc, gd)
    assert rg["psnr"] == pytest.approx(ro["psnr"], rel=1e-5)
    assert rg["ssim"] == pytest.approx(ro["ssim"], abs=2e-5)
    assert rg["depth_rmse"] == pytest.approx(ro["depth_rmse"], rel=1e-4)


def test_evaluate_sequence_records():  # pipeline.cpp:41-64: records per frame, cloud fallback
    cam = O.camera(55, 55, 31.5, 23.5, 64, 48)
    _, gm = pair(random_scene(7, 60, cam, O.pose()))
    gen = np.random.default_rng(3)
    cloud = np.zeros((200, 3))
    cloud[:, 2] = gen.uniform(2, 5, 200)
    cloud[:, :2] = gen.uniform(-0.4, 0.4, (200, 2)) * cloud[:, 2:3]
    frames = [(gpu_pose(O.pose()), np.full((48, 64, 3), 0.5), None, cloud),
              (gpu_pose(O.pose()), np.full((48, 64, 3), 0.5), np.full((48, 64), 2.0), None)]
    recs = G().evaluate_sequence(gm, frames, gpu_cam(cam))
    assert [r["frame"] for r in recs] == [0, 1]
    sparse = G().project_sparse_depth(cloud, gpu_pose(O.pose()), gpu_cam(cam))
    r0 = G().evaluate_view(gm, gpu_pose(O.pose()), gpu_cam(cam), np.full((48, 64, 3), 0.5), sparse)
    # fp64 block sums meet in atomics: equal to the last few ulps, not bit for bit
    assert recs[0]["depth_rmse"] == pytest.approx(r0["depth_rmse"], rel=1e-12)
    assert recs[0]["psnr"] == pytest.approx(r0["psnr"], rel=1e-12)
    assert recs[1]["iteration"] == gm.global_step and recs[1]["wall_time_s"] >= recs[0]["wall_time_s"]


def test_training_state_resume_is_exact(tmp_path):  # checkpoint + optimizer state = a true resume
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    gt = O.random_scene(O.Rng(21), 40, cam, O.pose(), 1.0, 2.0)
    color = np.asarray(O.render(gt, O.pose(), cam).color, np.float32).astype(np.float64)
    g = gt.gaussians
    g["p"][:, 10] = np.log(0.1 / 0.9)
    _, a = pair(g)
    cfg = G().TrainConfig.make(0.2, 0.5, 0)
    mk = lambda: G().Keyframe(gpu_pose(O.pose()), color, np.zeros((48, 64)), 100, 0)
    ka = mk()
    for _ in range(3):
        G().train_keyframe_step(a, ka, cfg, gpu_cam(cam))
    a.save_checkpoint(str(tmp_path / "m.gsmap"))
    a.save_training_state(str(tmp_path / "m.adam"))
    b = G().load_checkpoint(str(tmp_path / "m.gsmap"), a.ctx)
    b.load_training_state(str(tmp_path / "m.adam"))
    assert b.global_step == a.global_step == 3 and b.scene_extent == a.scene_extent
    for x, y in zip(a.adam_state(), b.adam_state()):
        np.testing.assert_array_equal(x, y)
    kb = mk()
    for _ in range(2):
        ra = G().train_keyframe_step(a, ka, cfg, gpu_cam(cam))
        rb = G().train_keyframe_step(b, kb, cfg, gpu_cam(cam))
        assert ra["loss"] == pytest.approx(rb["loss"], rel=1e-12)
    np.testing.assert_array_equal(a.gaussians["p"], b.gaussians["p"])
    with pytest.raises(ValueError, match="count"):
        G().GaussianMap(a.ctx).load_training_state(str(tmp_path / "m.adam"))
