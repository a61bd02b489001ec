"""GPU forward parity against the CPU fp64 oracle, through the C-ABI.

Bar (BASELINE.json north_star): projected order, tile keys and tile ranges BIT-EXACT; colour,
depth and visibility within 1e-4 absolute on pixels whose contributor count matches, with the
count of mismatching pixels reported and bounded.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from tests._common import gpu_cam, gpu_pose, pair, random_pose, random_scene, rect_of

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north_star: rendered colour and depth within 1e-4 absolute


def G():
    from paper_2411_02703_b200 import gsmap
    return gsmap


def small_cam():
    return O.camera(100, 100, 32, 32, 64, 64)


def check_keys(om, gm, pose, cam):
    """Projected set, depth order, fp64 means/depths, pixel rects and per-tile lists: exact."""
    oo = O.render(om, pose, cam)
    go = G().render(gm, gpu_pose(pose), gpu_cam(cam))
    op = oo.projected()
    gp = go.projected()
    assert len(op["index"]) == len(gp["index"])
    np.testing.assert_array_equal(gp["index"], op["index"])          # (depth, index) order
    np.testing.assert_array_equal(gp["mean"], op["mean"])            # fp64 mean, bit-exact
    np.testing.assert_array_equal(gp["depth"], op["depth"])          # fp64 depth, bit-exact
    np.testing.assert_array_equal(gp["rect"], rect_of(op["mean"], op["radius"], cam.width, cam.height))
    ooff, oent = oo.bins()
    goff, gent = go.tiles()
    np.testing.assert_array_equal(goff, ooff)                        # tile ranges
    np.testing.assert_array_equal(gent, op["index"][oent])           # tile lists (map index)
    return oo, go


def check_images(oo, go, tol=TOL, max_mismatch_frac=1e-4):
    onc = oo.n_contrib()
    gnc, _ = go.pixel_state()
    same = onc == gnc
    mism = int((~same).sum())
    assert mism <= max(1, max_mismatch_frac * same.size), f"{mism} pixels with a different contributor count"
    for a, b in ((go.color, oo.color), (go.depth, oo.depth), (go.visibility, oo.visibility)):
        err = np.abs(a - b)
        if err.ndim == 3:
            err = err.max(axis=2)
        assert err[same].max(initial=0.0) <= tol
    return mism


def test_empty_map_background():  # test_rasterizer.cpp:41-48
    gm = G().GaussianMap()
    out = G().render(gm, G().Pose(1, 0, 0, 0, 0, 0, 0), gpu_cam(small_cam()))
    assert not out.color.any() and not out.depth.any() and not out.visibility.any()
    assert out.contributors(10, 10) == []


def test_single_on_axis_gaussian():  # test_rasterizer.cpp:50-60
    om, gm = pair(O.make_blob([0, 0, 2], 0.7, [1, 0, 0]))
    out = G().render(gm, gpu_pose(O.pose()), gpu_cam(small_cam()))
    assert out.color[32, 32, 0] == pytest.approx(0.7, abs=1e-6)
    assert out.color[32, 32, 1] == pytest.approx(0.0, abs=1e-7)
    assert out.depth[32, 32] == pytest.approx(1.4, abs=1e-6)
    assert out.visibility[32, 32] == pytest.approx(0.7, abs=1e-6)


def test_two_stacked_front_to_back():  # test_rasterizer.cpp:62-74
    g = np.concatenate([O.make_blob([0, 0, 3], 0.5, [0, 1, 0]), O.make_blob([0, 0, 2], 0.5, [1, 0, 0])])
    om, gm = pair(g)
    out = G().render(gm, gpu_pose(O.pose()), gpu_cam(small_cam()))
    assert out.color[32, 32, 0] == pytest.approx(0.5, abs=1e-6)
    assert out.color[32, 32, 1] == pytest.approx(0.25, abs=1e-6)
    assert out.visibility[32, 32] == pytest.approx(0.75, abs=1e-6)
    assert [gid for gid, _ in out.contributors(32, 32)] == [1, 0]


def test_clamped_stack_does_not_terminate_early():
    """(1 - 0.99)^2 = 1.0000000000000018e-4 in fp64 does NOT cross kTransmittanceMin, but the fp32
    product would; the GPU keeps T in fp64 (SURVEY §7 hard part 2). Three opaque splats on
    the centre pixel: all three must contribute, as in the reference."""
    g = np.concatenate([O.make_blob([0, 0, z], 0.999999, [1, 0, 0]) for z in (2.0, 3.0, 4.0)])
    om, gm = pair(g)
    oo = O.render(om, O.pose(), small_cam())
    go = G().render(gm, gpu_pose(O.pose()), gpu_cam(small_cam()))
    assert len(go.contributors(32, 32)) == oo.n_contrib()[32, 32] == 3
    check_images(oo, go)


@pytest.mark.parametrize("seed", range(12))
def test_keys_and_images_random_scenes(seed):  # test_rasterizer.cpp:76-88 scenes, vs oracle
    gen = np.random.default_rng(99 + seed)
    cam = small_cam()
    pose = random_pose(gen)
    om, gm = pair(random_scene(99 + seed, 200, cam, pose), )
    oo, go = check_keys(om, gm, pose, cam)
    assert check_images(oo, go) == 0


def test_contributor_lists_match_csr():
    gen = np.random.default_rng(4)
    cam = O.camera(120, 120, 63.5, 47.5, 128, 96)
    pose = random_pose(gen)
    om, gm = pair(random_scene(4, 300, cam, pose))
    oo = O.render(om, pose, cam)
    go = G().render(gm, gpu_pose(pose), gpu_cam(cam))
    ooff, og, oa = oo.csr()
    goff, gg, ga = go.csr()
    np.testing.assert_array_equal(goff, ooff)
    np.testing.assert_array_equal(gg, og)
    assert np.abs(ga - oa).max() < 1e-6


def test_insertion_order_invariance():  # test_rasterizer.cpp:90-104
    cam = small_cam()
    g = random_scene(7, 60, cam, O.pose())
    perm = np.random.default_rng(7).permutation(len(g))
    _, gm = pair(g)
    _, gm2 = pair(g[perm])
    a = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    b = G().render(gm2, gpu_pose(O.pose()), gpu_cam(cam))
    assert np.array_equal(a.color, b.color)
    assert np.array_equal(a.depth, b.depth)
    assert np.array_equal(a.visibility, b.visibility)


def test_visibility_complements_transmittance():  # test_rasterizer.cpp:106-120
    cam = small_cam()
    _, gm = pair(random_scene(11, 150, cam, O.pose()))
    out = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    _, t = out.pixel_state()
    assert np.abs(out.visibility + t - 1.0).max() < 1e-5
    assert out.color.max() <= 1.0 + 1e-5


def test_deterministic_repeat():  # test_rasterizer.cpp:137-176 (fixed configuration -> bitwise)
    cam = O.camera(120, 120, 63.5, 47.5, 128, 96)
    _, gm = pair(random_scene(23, 250, cam, O.pose()))
    a = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    b = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    assert np.array_equal(a.color, b.color) and np.array_equal(a.depth, b.depth)


def test_behind_camera_and_offscreen_culled():
    g = np.concatenate([O.make_blob([0, 0, -1], 0.7, [1, 0, 0]), O.make_blob([0, 0, 0.005], 0.7, [1, 0, 0]),
                        O.make_blob([100, 100, 2], 0.7, [0, 1, 0]), O.make_blob([0, 0, 2], 0.7, [0, 0, 1])])
    om, gm = pair(g)
    out = G().render(gm, gpu_pose(O.pose()), gpu_cam(small_cam()))
    assert out.stats().n_visible == 1
    check_keys(om, gm, O.pose(), small_cam())


def test_camera_validation_raises():  # core/types.hpp:22-29
    gm = G().GaussianMap()
    with pytest.raises(ValueError):
        G().render(gm, G().Pose(1, 0, 0, 0, 0, 0, 0), G().Camera(0, 1, 0, 0, 4, 4))
    with pytest.raises(ValueError):
        G().render(gm, G().Pose(1, 0, 0, 0, 0, 0, 0), G().Camera(1, 1, 4.0, 0, 4, 4))


def test_non_multiple_of_tile_image():
    """Ragged last tile row/column (cam.width % 16 != 0)."""
    cam = O.camera(90, 95, 36.2, 20.7, 77, 45)
    gen = np.random.default_rng(5)
    pose = random_pose(gen)
    om, gm = pair(random_scene(5, 180, cam, pose))
    oo, go = check_keys(om, gm, pose, cam)
    assert check_images(oo, go) == 0


@pytest.mark.parametrize("sizes", [(1, 2, 3, 5, 16), (17, 40), (2,) * 30])
def test_depth_ties_ordered_exactly(sizes):
    """Runs of equal depth keys (rasterizer.cpp:69-72: ties by map index; fp64 depths that differ
    below the key's resolution) — the register-network runs (<= 16) and the insertion fallback."""
    cam = O.camera(60, 60, 31.5, 31.5, 64, 64)
    pose = O.pose(1.0, 1e-7, 0.0, 0.0)  # a tiny tilt: same 24-bit key, distinct fp64 depths
    g = random_scene(11, sum(sizes), cam, pose)
    gen = np.random.default_rng(len(sizes))
    k = 0
    for j, m in enumerate(sizes):
        z = 1.0 + 0.37 * j
        for a in range(m):
            if a % 3 == 2:
                g["p"][k, :3] = g["p"][k - 1, :3]  # an exact duplicate depth: ordered by index
            else:
                g["p"][k, :2] = gen.uniform(-0.4, 0.4, 2) * z
                g["p"][k, 2] = z
            k += 1
    g = g[gen.permutation(len(g))]
    om, gm = pair(g)
    oo, go = check_keys(om, gm, pose, cam)
    assert check_images(oo, go) == 0
