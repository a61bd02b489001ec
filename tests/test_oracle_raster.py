"""Ports of proj/tests/test_rasterizer.cpp onto the CPU oracle (render / render_backward), plus
the gradient-check harness (proj/src/pipeline/gradcheck.cpp) at the reference test's settings."""
import math

import numpy as np
import pytest

from oracle import pyoracle as O


def small_cam():  # test_rasterizer.cpp:29
    return O.camera(100, 100, 32, 32, 64, 64)


def max_abs_diff(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) if np.size(a) else 0.0


def test_empty_map_background():  # test_rasterizer.cpp:41-48
    out = O.render(O.OracleMap(), O.pose(), small_cam())
    assert not out.color.any() and not out.depth.any() and not out.visibility.any()
    off, _, _ = out.csr()
    assert off[10 * 64 + 10 + 1] == off[10 * 64 + 10]


def test_single_on_axis_gaussian():  # test_rasterizer.cpp:50-60
    m = O.OracleMap(O.make_blob([0, 0, 2], 0.7, [1, 0, 0]))
    out = O.render(m, O.pose(), small_cam())
    assert out.color[32, 32, 0] == pytest.approx(0.7, rel=1e-12)
    assert out.color[32, 32, 1] == pytest.approx(0.0, abs=1e-12)
    assert out.depth[32, 32] == pytest.approx(1.4, rel=1e-12)
    assert out.visibility[32, 32] == pytest.approx(0.7, rel=1e-12)


def test_two_stacked_front_to_back():  # test_rasterizer.cpp:62-74
    g = np.concatenate([O.make_blob([0, 0, 3], 0.5, [0, 1, 0]), O.make_blob([0, 0, 2], 0.5, [1, 0, 0])])
    out = O.render(O.OracleMap(g), O.pose(), small_cam())
    assert out.color[32, 32, 0] == pytest.approx(0.5, rel=1e-12)
    assert out.color[32, 32, 1] == pytest.approx(0.25, rel=1e-12)
    assert out.visibility[32, 32] == pytest.approx(0.75, rel=1e-12)
    off, gi, _ = out.csr()
    p = 32 * 64 + 32
    lst = gi[off[p]:off[p + 1]]
    assert list(lst) == [1, 0]


def random_pose(rng: np.random.Generator):
    q = rng.normal(size=4)
    return O.pose(*q, t=tuple(rng.uniform(-1, 1, 3) * 0.3))


def test_tile_renderer_matches_brute_force():  # test_rasterizer.cpp:76-88
    rng = O.Rng(99)
    gen = np.random.default_rng(99)
    cam = small_cam()
    for _ in range(12):
        pose = random_pose(gen)
        m = O.random_scene(rng, 200, cam, pose)
        tiled = O.render(m, pose, cam)
        bc, bd, bv = O.brute_force(m, pose, cam)
        assert max_abs_diff(tiled.color, bc) <= 1e-5
        assert max_abs_diff(tiled.depth, bd) <= 1e-5
        assert max_abs_diff(tiled.visibility, bv) <= 1e-5


def test_insertion_order_invariance():  # test_rasterizer.cpp:90-104
    rng = O.Rng(7)
    cam = small_cam()
    m = O.random_scene(rng, 60, cam, O.pose())
    g = m.gaussians
    perm = np.random.default_rng(7).permutation(len(g))
    m2 = O.OracleMap(g[perm])
    a = O.render(m, O.pose(), cam)
    b = O.render(m2, O.pose(), cam)
    assert max_abs_diff(a.color, b.color) == 0.0
    assert max_abs_diff(a.depth, b.depth) == 0.0
    assert max_abs_diff(a.visibility, b.visibility) == 0.0


def test_visibility_complements_transmittance():  # test_rasterizer.cpp:106-120
    rng = O.Rng(11)
    cam = small_cam()
    m = O.random_scene(rng, 150, cam, O.pose())
    out = O.render(m, O.pose(), cam)
    off, _, alpha = out.csr()
    logs = np.log1p(-alpha)
    cums = np.concatenate([[0.0], np.cumsum(logs)])
    t = np.exp(cums[off[1:]] - cums[off[:-1]]).reshape(64, 64)
    assert np.max(np.abs(out.visibility + t - 1.0)) < 1e-6
    assert out.color.max() <= 1.0 + 1e-6


def test_raising_opacity_never_lowers_visibility():  # test_rasterizer.cpp:122-135
    rng = O.Rng(31)
    cam = small_cam()
    gen = np.random.default_rng(31)
    for _ in range(10):
        m = O.random_scene(rng, 40, cam, O.pose(), -2.0, 0.5)
        before = O.render(m, O.pose(), cam)
        g = m.gaussians
        g["p"][gen.integers(len(g)), 10] += 0.8
        m.gaussians = g
        after = O.render(m, O.pose(), cam)
        assert np.all(after.visibility >= before.visibility - 1e-12)


def test_thread_counts_agree_and_deterministic():  # test_rasterizer.cpp:137-176
    rng = O.Rng(23)
    cam = O.camera(120, 120, 63.5, 47.5, 128, 96)
    m = O.random_scene(rng, 250, cam, O.pose())
    serial = O.render(m, O.pose(), cam, threads=1)
    p3 = O.render(m, O.pose(), cam, threads=3)
    p3b = O.render(m, O.pose(), cam, threads=3)
    p7 = O.render(m, O.pose(), cam, threads=7)
    assert max_abs_diff(p3.color, p3b.color) == 0.0
    assert max_abs_diff(serial.color, p3.color) < 1e-12
    assert max_abs_diff(serial.color, p7.color) < 1e-12
    gen = np.random.default_rng(23)
    dc = gen.uniform(-1, 1, (96, 128, 3)); dd = gen.uniform(-1, 1, (96, 128))
    gs = O.render_backward(m, O.pose(), cam, serial, dc, dd, threads=1)
    g3 = O.render_backward(m, O.pose(), cam, p3, dc, dd, threads=3)
    g3b = O.render_backward(m, O.pose(), cam, p3b, dc, dd, threads=3)
    g7 = O.render_backward(m, O.pose(), cam, p7, dc, dd, threads=7)
    assert max_abs_diff(g3[:, :3], g3b[:, :3]) == 0.0
    assert max_abs_diff(gs[:, :3], g7[:, :3]) < 1e-6


def test_zero_cotangent_zero_grads():  # test_rasterizer.cpp:178-193
    rng = O.Rng(5)
    cam = small_cam()
    m = O.random_scene(rng, 30, cam, O.pose())
    out = O.render(m, O.pose(), cam)
    g = O.render_backward(m, O.pose(), cam, out, np.zeros((64, 64, 3)), np.zeros((64, 64)))
    assert np.all(g[:, :11] == 0.0)


def test_non_contributing_zero_grads():  # test_rasterizer.cpp:195-208
    g = np.concatenate([O.make_blob([0, 0, 2], 0.7, [1, 0, 0]), O.make_blob([100, 100, 2], 0.7, [0, 1, 0])])
    m = O.OracleMap(g)
    cam = small_cam()
    out = O.render(m, O.pose(), cam)
    gr = O.render_backward(m, O.pose(), cam, out, np.ones((64, 64, 3)), np.full((64, 64), 0.5))
    assert np.linalg.norm(gr[0, 0:3]) > 0.0
    assert np.linalg.norm(gr[1, 0:3]) == 0.0
    assert np.linalg.norm(gr[1, 3:7]) == 0.0
    assert gr[1, 10] == 0.0


def test_opacity_gradient_closed_form_and_fd():  # test_rasterizer.cpp:210-237
    op = 0.7
    m = O.OracleMap(O.make_blob([0, 0, 2], op, [1, 0, 0]))
    cam = small_cam()
    out = O.render(m, O.pose(), cam)
    dc = np.zeros((64, 64, 3)); dc[32, 32, 0] = 1.0
    g = O.render_backward(m, O.pose(), cam, out, dc, np.zeros((64, 64)))
    assert g[0, 10] == pytest.approx(op * (1 - op), rel=1e-9)
    h = 1e-4

    def loss_at(lv):
        b = O.make_blob([0, 0, 2], op, [1, 0, 0]); b["p"][0, 10] = lv
        return O.render(O.OracleMap(b), O.pose(), cam).color[32, 32, 0]
    lg = math.log(op / (1 - op))
    fd = (loss_at(lg + h) - loss_at(lg - h)) / (2 * h)
    assert g[0, 10] == pytest.approx(fd, rel=1e-5)


def test_backward_rejects_mismatched_cotangent():  # test_rasterizer.cpp:239-248
    m = O.OracleMap(O.make_blob([0, 0, 2], 0.5, [1, 0, 0]))
    cam = small_cam()
    out = O.render(m, O.pose(), cam)
    with pytest.raises(O.InvalidArgument):
        O.render_backward(m, O.pose(), cam, out, np.zeros((10, 10, 3)), np.zeros((64, 64)))


def test_gradcheck_full_render():  # test_rasterizer.cpp:250-261
    r = O.run_gradcheck(seed=3, configs=60, core_configs=120, n_gaussians=25)
    assert r["max_rel_err_core"] < 1e-4
    assert r["max_rel_err_render"] < 1e-3
    assert r["configs_run"] == 60
