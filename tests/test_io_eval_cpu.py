"""Checkpoint format v1 (io/checkpoint.cpp) and per-frame evaluation (pipeline.cpp:34-64) on the
CPU oracle: ports of test_io.cpp:190-207 and test_pipeline.cpp:128-146."""
import numpy as np
import pytest

from oracle import pyoracle as O


def q8(img):
    """quantize_8bit (pipeline.cpp:34-39): lround(clamp(x, 0, 1) * 255) / 255 (x >= 0: floor(+0.5))."""
    return np.floor(np.clip(img, 0.0, 1.0) * 255.0 + 0.5) / 255.0


def test_checkpoint_round_trip_renders_bit_exactly(tmp_path):  # test_io.cpp:190-207
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    m = O.random_scene(O.Rng(4), 50, cam, O.pose())
    m.raise_sh_degree(2)
    path = str(tmp_path / "m.gsmap")
    O.save_checkpoint(path, m)
    loaded = O.load_checkpoint(path)
    assert len(loaded) == len(m)
    np.testing.assert_array_equal(loaded.gaussians["p"], m.gaussians["p"])
    np.testing.assert_array_equal(loaded.gaussians["degree"], m.gaussians["degree"])
    a, b = O.render(m, O.pose(), cam), O.render(loaded, O.pose(), cam)
    np.testing.assert_array_equal(a.color, b.color)
    np.testing.assert_array_equal(a.depth, b.depth)
    header = f"gsmap-checkpoint 1\ncount 50\nsh_degree {m.gaussians['degree'].max()}\nend_header\n".encode()
    with open(path, "rb") as f:
        assert f.read(len(header)) == header
    assert (tmp_path / "m.gsmap").stat().st_size == len(header) + 50 * 476
    with pytest.raises(O.OracleError, match="cannot open"):
        O.load_checkpoint(str(tmp_path / "missing.gsmap"))
    (tmp_path / "junk.gsmap").write_text("not a checkpoint\n")
    with pytest.raises(O.OracleError, match="not a checkpoint"):
        O.load_checkpoint(str(tmp_path / "junk.gsmap"))


def test_evaluate_gt_map_scores_sentinel():  # test_pipeline.cpp:128-146
    cam = O.camera(55, 55, 31.5, 23.5, 64, 48)
    m = O.random_scene(O.Rng(5), 60, cam, O.pose())
    out = O.render(m, O.pose(), cam)
    r = O.evaluate_view(m, O.pose(), cam, q8(out.color), out.depth)
    assert r["psnr"] == 100.0
    assert r["ssim"] == pytest.approx(1.0)
    assert r["depth_rmse"] == pytest.approx(0.0)
    assert np.isnan(O.evaluate_view(m, O.pose(), cam, q8(out.color))["depth_rmse"])


def test_evaluate_matches_metric_definitions():  # psnr / ssim / depth_rmse of the quantized render
    cam = O.camera(55, 55, 31.5, 23.5, 64, 48)
    m = O.random_scene(O.Rng(6), 60, cam, O.pose())
    out = O.render(m, O.pose(), cam)
    gen = np.random.default_rng(0)
    gt = gen.uniform(0, 1, (48, 64, 3))
    gd = np.where(gen.uniform(size=(48, 64)) < 0.3, gen.uniform(1, 4, (48, 64)), 0.0)
    r = O.evaluate_view(m, O.pose(), cam, gt, gd)
    assert r["psnr"] == pytest.approx(O.psnr(q8(out.color), gt), rel=1e-12)
    assert r["ssim"] == pytest.approx(O.ssim(q8(out.color), gt), rel=1e-12)
    assert r["depth_rmse"] == pytest.approx(O.depth_rmse(out.depth, gd)[0], rel=1e-12)
