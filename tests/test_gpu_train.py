"""GPU loss (L1 + SSIM + masked depth), pyramid, Adam and the fused train_keyframe_step against
the CPU fp64 oracle, through the C-ABI."""
import numpy as np
import pytest

from oracle import pyoracle as O
from tests._common import gpu_cam, gpu_pose, pair, random_pose, random_scene, rel_err, round32

pytestmark = pytest.mark.gpu


def G():
    from paper_2411_02703_b200 import gsmap
    return gsmap


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def test_pyramid_matches_oracle():  # mapper.cpp:65-144
    gen = np.random.default_rng(1)
    col = f32(gen.uniform(0, 1, (37, 53, 3)))
    dep = f32(np.where(gen.uniform(size=(37, 53)) < 0.3, gen.uniform(1, 5, (37, 53)), 0.0))
    kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), col, dep, 10, 2)
    oc = O.build_pyramid(col, 2)
    od = O.build_pyramid(dep, 2, depth=True)
    for l in range(3):
        c, d = kf.level(l)
        assert np.abs(c - oc[l]).max() < 1e-6
        assert np.abs(d - od[l]).max() < 1e-5


def test_pyramid_rejects_too_small():
    with pytest.raises(ValueError):
        G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), np.zeros((3, 3, 3)), np.zeros((3, 3)), 1, 2)


@pytest.mark.parametrize("lam,lam_d", [(0.2, 0.5), (0.0, 0.0), (0.0, 0.5), (0.2, 0.0)])
def test_loss_matches_oracle(lam, lam_d):
    """compute_loss on the GPU's own render vs the oracle's compute_loss on the same images."""
    cam = O.camera(120, 120, 63.5, 47.5, 128, 96)
    om, gm = pair(random_scene(8, 300, cam, O.pose(), 0.0, 2.5))
    gen = np.random.default_rng(8)
    gt = f32(gen.uniform(0, 1, (96, 128, 3)))
    gd = f32(np.where(gen.uniform(size=(96, 128)) < 0.5, gen.uniform(1, 8, (96, 128)), 0.0))
    kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), gt, gd, 10, 0)
    go = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    cfg = G().TrainConfig.make(lam, lam_d, 0)
    r = G().compute_loss(go, kf, 0, cfg)
    ref = O.compute_loss(go.color, go.depth, go.visibility, gt, gd, O.make_cfg(lam, lam_d, 0))
    for k in ("total", "l1", "ssim", "color_loss", "depth_loss"):
        assert r[k] == pytest.approx(ref[k], rel=1e-5, abs=1e-7), k
    assert r["psnr"] == pytest.approx(O.psnr(go.color, gt), rel=1e-6)
    scale = np.abs(ref["dl_dcolor"]).max()
    assert np.abs(r["dl_dcolor"] - ref["dl_dcolor"]).max() <= 1e-4 * scale + 1e-12
    dscale = max(np.abs(ref["dl_ddepth"]).max(), 1e-30)
    assert np.abs(r["dl_ddepth"] - ref["dl_ddepth"]).max() <= 1e-5 * dscale


def test_loss_rejects_wrong_level_resolution():
    cam = O.camera(100, 100, 32, 32, 64, 64)
    _, gm = pair(O.make_blob([0, 0, 2], 0.5, [1, 0, 0]))
    kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), np.zeros((64, 64, 3)), np.zeros((64, 64)), 10, 1)
    go = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    with pytest.raises(ValueError):
        G().compute_loss(go, kf, 1, G().TrainConfig.make())
    with pytest.raises(ValueError):
        G().compute_loss(go, kf, 5, G().TrainConfig.make())


def test_adam_matches_oracle():  # gaussian_map.cpp:37-54
    gen = np.random.default_rng(3)
    g0 = O.empty_gaussians(300)
    g0["p"][:] = gen.normal(size=(300, 59)); g0["degree"] = gen.integers(0, 4, 300)
    om, gm = pair(g0)
    assert gm.scene_extent == om.scene_extent
    for t in range(3):
        grads = round32_arr(gen.normal(size=(300, 59)) * 10.0 ** gen.uniform(-6, 1, (300, 59)))
        for i, d in enumerate(g0["degree"]):  # inactive SH coefficients carry no gradient
            grads[i, 11 + 3 * (d + 1) ** 2:] = 0.0
        om.apply_gradients(grads)
        gg = G().RenderGradients(gm.ctx)
        gg.write(grads)
        gm.apply_gradients(gg)
        a, b = gm.gaussians["p"], om.gaussians["p"]
        lr = np.array([1.6e-4 * om.scene_extent] * 3 + [1e-3] * 4 + [5e-3] * 3 + [5e-2] + [2.5e-3] * 48)
        # Adam's step is ~lr*sign; fp32 parameter storage rounds at ~6e-8 relative
        assert np.all(np.abs(a - b) <= 1e-4 * lr + 4e-7 * np.abs(b)), t
    _, _, steps = gm.adam_state()
    assert np.all(steps == 3) and gm.global_step == 3


def round32_arr(a):
    return np.asarray(a, np.float32).astype(np.float64)


def test_apply_gradients_rejects_mismatch():  # test_mapper.cpp:337-344
    _, gm = pair(O.make_blob([0, 0, 2], 0.5, [1, 0, 0]))
    gg = G().RenderGradients(gm.ctx)
    gg.write(np.zeros((3, 59)))
    with pytest.raises(ValueError):
        gm.apply_gradients(gg)


def test_level_schedule_and_budget():  # test_mapper.cpp:206-239
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    _, gm = pair(random_scene(9, 30, cam, O.pose()))
    kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), np.full((48, 64, 3), 0.3), np.zeros((48, 64)), 30, 2)
    cfg = G().TrainConfig.make(levels=2, ipl=10)
    levels = [G().train_keyframe_step(gm, kf, cfg, gpu_cam(cam))["level"] for _ in range(30)]
    assert levels == [2] * 10 + [1] * 10 + [0] * 10
    assert G().train_keyframe_step(gm, kf, cfg, gpu_cam(cam)) is None
    assert gm.global_step == 30


def test_train_steps_track_oracle():
    """A few full train_keyframe_step iterations (render -> loss -> backward -> Adam) on both;
    losses agree and parameters stay within a few Adam steps' worth of each other."""
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    gt_map = O.random_scene(O.Rng(21), 40, cam, O.pose(), 1.0, 2.0)
    gt = O.render(gt_map, O.pose(), cam)
    g = gt_map.gaussians
    g["p"][:, 10] = np.log(0.1 / 0.9)
    g["p"][:, 7:10] += 0.4
    om, gm = pair(g)
    color = f32(gt.color)
    sparse = f32(np.where(np.random.default_rng(1).uniform(size=(48, 64)) < 0.2, gt.depth, 0.0))
    okf = O.Keyframe(O.pose(), color, sparse, 6, 1)
    gkf = G().Keyframe(gpu_pose(O.pose()), color, sparse, 6, 1)
    ocfg = O.make_cfg(0.2, 0.5, 1)
    gcfg = G().TrainConfig.make(0.2, 0.5, 1)
    for it in range(6):
        ro = O.train_keyframe_step(om, okf, ocfg, cam)
        rg = G().train_keyframe_step(gm, gkf, gcfg, gpu_cam(cam))
        assert rg["level"] == ro["level"]
        assert rg["loss"] == pytest.approx(ro["loss"], rel=2e-3)
        assert rg["psnr"] == pytest.approx(ro["psnr"], rel=1e-3)
    lr = np.array([1.6e-4 * om.scene_extent] * 3 + [1e-3] * 4 + [5e-3] * 3 + [5e-2] + [2.5e-3] * 48)
    d = np.abs(gm.gaussians["p"] - om.gaussians["p"])
    assert np.all(d <= 6 * 2 * lr + 1e-6)
    assert np.mean(d <= 0.05 * lr + 1e-6) > 0.95


def test_train_steps_bitwise_reproducible():
    """Two identical runs (fresh context, map and keyframes) report bitwise-equal losses and
    psnr and end with bitwise-equal parameters and Adam state: every reduction on the path (the
    sorts, the partial rows, the loss / psnr sums) is fixed-order, with no atomics on values
    (the reference is deterministic for a fixed thread count, test_rasterizer.cpp:137-176)."""
    from fixtures import pyfixture as F
    scene = F.Scene(n_gaussians=20_000, width=320, height=256, n_frames=2, seed=1)
    train = round32(scene.training_map(seed=2, noise=0.06))
    fx, fy, cx, cy, W, H = scene.camera
    cam = G().Camera(fx, fy, cx, cy, W, H)
    pose = G().Pose(*scene.poses[0])
    gt_ctx = G().Context(0)
    gt = G().render(G().GaussianMap(gt_ctx, scene.gaussians), pose, cam).color
    sparse = scene.sparse_depth(0)

    def run():
        ctx = G().Context(0)
        m = G().GaussianMap(ctx, train)
        kf = G().Keyframe(pose, gt, sparse, 9, 2, ctx=ctx)
        reps = [G().train_keyframe_step(m, kf, G().TrainConfig.make(0.2, 0.5, 2), cam) for _ in range(9)]
        return reps, m.gaussians["p"], m.adam_state()

    a, b = run(), run()
    assert [r["level"] for r in a[0]] == [2, 2, 2, 1, 1, 1, 0, 0, 0]
    assert a[0] == b[0]  # loss and psnr, bit for bit
    assert np.array_equal(a[1], b[1])
    for x, y in zip(a[2], b[2]):
        assert np.array_equal(x, y)


def test_train_step_requires_pyramid_semantics():
    _, gm = pair(O.make_blob([0, 0, 2], 0.5, [1, 0, 0]))
    kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), np.zeros((64, 64, 3)), np.zeros((64, 64)), 0, 0)
    assert G().train_keyframe_step(gm, kf, G().TrainConfig.make(), G().Camera(100, 100, 32, 32, 64, 64)) is None


def test_pair_capacity_overflow_reruns_step():
    """The step is enqueued without reading the (tile, gaussian) pair count back; the pair
    buffers use a capacity remembered per resolution. A render that outgrows it must leave the
    map untouched (no Adam update, no step count) and be re-run at exact size."""
    cam = O.camera(400, 400, 319.5, 239.5, 640, 480)
    g = random_scene(31, 6000, cam, O.pose(), 0.0, 2.0)
    small, big = g.copy(), g.copy()
    small["p"][:, 7:10] = np.log(0.002)  # ~1 tile each: a small remembered capacity
    big["p"][:, 7:10] = np.log(0.2)      # tens of tiles each: far beyond it
    gen = np.random.default_rng(2)
    color = f32(gen.uniform(0, 1, (480, 640, 3)))
    sparse = f32(np.where(gen.uniform(size=(480, 640)) < 0.1, gen.uniform(1, 8, (480, 640)), 0.0))
    cfg = G().TrainConfig.make(0.2, 0.5, 0)

    def step(ctx, gmap):
        kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), color, sparse, 5, 0, ctx=ctx)
        return G().train_keyframe_step(gmap, kf, cfg, gpu_cam(cam))

    ctx1 = G().Context(0)
    step(ctx1, G().GaussianMap(ctx1, round32(small)))
    mb1 = G().GaussianMap(ctx1, round32(big))
    r1 = step(ctx1, mb1)
    ctx2 = G().Context(0)
    mb2 = G().GaussianMap(ctx2, round32(big))
    r2 = step(ctx2, mb2)
    assert r1["loss"] == pytest.approx(r2["loss"], rel=1e-9)
    assert mb1.global_step == mb2.global_step == 1
    assert np.all(mb1.adam_state()[2] == 1)
    d = np.abs(mb1.gaussians["p"] - mb2.gaussians["p"])
    assert np.mean(d <= 1e-6) > 0.999 and d.max() < 0.2

    # the public render re-renders too: same frame object, small then big
    fr = G().RenderOutput(ctx1)
    G().render(G().GaussianMap(ctx1, round32(small)), gpu_pose(O.pose()), gpu_cam(cam), fr)
    G().render(G().GaussianMap(ctx1, round32(big)), gpu_pose(O.pose()), gpu_cam(cam), fr)
    fresh = G().render(G().GaussianMap(ctx2, round32(big)), gpu_pose(O.pose()), gpu_cam(cam))
    assert fr.stats().n_pairs == fresh.stats().n_pairs > 100_000
    np.testing.assert_array_equal(fr.color, fresh.color)


def test_upload_level_is_seen_by_next_reader():
    """gs_keyframe_upload_level runs on the copy stream; the loss / read-back that follows must
    see the new level (same loss as a keyframe built from that image)."""
    cam = O.camera(120, 120, 63.5, 47.5, 128, 96)
    om, gm = pair(random_scene(8, 300, cam, O.pose(), 0.0, 2.5))
    gen = np.random.default_rng(5)
    c0 = f32(gen.uniform(0, 1, (96, 128, 3))); d0 = np.zeros((96, 128))
    c1 = f32(gen.uniform(0, 1, (96, 128, 3)))
    d1 = f32(np.where(gen.uniform(size=(96, 128)) < 0.3, gen.uniform(1, 8, (96, 128)), 0.0))
    ka = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), c0, d0, 10, 1)
    kb = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), c1, d1, 10, 1)
    go = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    cfg = G().TrainConfig.make(0.2, 0.5, 1)
    before = G().compute_loss(go, ka, 0, cfg)["total"]
    for _ in range(3):  # repeated uploads, each read right after
        ka.upload_level(0, c1, d1)
        c, d = ka.level(0)
        np.testing.assert_array_equal(c, c1)
        np.testing.assert_array_equal(d, d1)
        assert G().compute_loss(go, ka, 0, cfg)["total"] == pytest.approx(
            G().compute_loss(go, kb, 0, cfg)["total"], rel=1e-12)
        ka.upload_level(0, c0, d0)
        assert G().compute_loss(go, ka, 0, cfg)["total"] == pytest.approx(before, rel=1e-12)


def test_visible_capacity_overflow_reruns_step():
    """Same as above for the visible-count capacity (depth sort / rank-indexed kernels): a view
    that sees far more Gaussians than the remembered capacity is flagged and re-run exactly."""
    cam = O.camera(400, 400, 319.5, 239.5, 640, 480)
    g = random_scene(32, 20000, cam, O.pose(), 0.0, 2.0)
    g["p"][:, 7:10] = np.log(0.003)
    few = g.copy()
    few["p"][1000:, 2] = -5.0  # behind the camera: 1000 visible
    gen = np.random.default_rng(3)
    color = f32(gen.uniform(0, 1, (480, 640, 3)))
    sparse = np.zeros((480, 640))
    cfg = G().TrainConfig.make(0.2, 0.5, 0)

    def step(ctx, gmap):
        kf = G().Keyframe(G().Pose(1, 0, 0, 0, 0, 0, 0), color, sparse, 5, 0, ctx=ctx)
        return G().train_keyframe_step(gmap, kf, cfg, gpu_cam(cam))

    ctx1 = G().Context(0)
    step(ctx1, G().GaussianMap(ctx1, round32(few)))
    m1 = G().GaussianMap(ctx1, round32(g))
    r1 = step(ctx1, m1)
    ctx2 = G().Context(0)
    m2 = G().GaussianMap(ctx2, round32(g))
    r2 = step(ctx2, m2)
    assert r1["loss"] == pytest.approx(r2["loss"], rel=1e-9)
    assert np.all(m1.adam_state()[2] == 1)
    d = np.abs(m1.gaussians["p"] - m2.gaussians["p"])
    assert np.mean(d <= 1e-6) > 0.999
    fr = G().RenderOutput(ctx1)
    G().render(G().GaussianMap(ctx1, round32(few)), gpu_pose(O.pose()), gpu_cam(cam), fr)
    G().render(G().GaussianMap(ctx1, round32(g)), gpu_pose(O.pose()), gpu_cam(cam), fr)
    fresh = G().render(G().GaussianMap(ctx2, round32(g)), gpu_pose(O.pose()), gpu_cam(cam))
    assert fr.stats().n_visible == fresh.stats().n_visible > 15000
    np.testing.assert_array_equal(fr.color, fresh.color)


def test_prune_keeps_state_aligned():  # test_mapper.cpp:298-311
    from oracle import pyoracle as O
    g = O.empty_gaussians(10)
    g["p"][:, 0] = np.arange(10.0)
    g["p"][:, 2] = 3.0
    g["p"][:, 3] = 1.0
    g["p"][:, 7:10] = np.log(0.3)
    g["p"][:, 10] = 0.0  # logit(0.5)
    m = G().GaussianMap(None, g)
    assert m.prune(0.005) == 0
    g["p"][4, 10] = np.log(0.001 / 0.999)
    m = G().GaussianMap(None, round32(g))
    assert m.prune(0.005) == 1
    assert len(m) == 9
    p = m.gaussians["p"]
    assert p[4, 0] == 5.0  # compacted over the hole
    mm, vv, steps = m.adam_state()
    assert mm.shape[0] == vv.shape[0] == steps.shape[0] == 9
    with pytest.raises(ValueError):
        m.prune(0.0)
    with pytest.raises(ValueError):
        m.prune(1.0)


def test_prune_matches_oracle_after_training():
    """Train a few steps (non-trivial Adam state), prune a third of the map on both, then the
    parameters, optimizer state and a render agree; training continues in lockstep."""
    from oracle import pyoracle as O
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    g = random_scene(31, 60, cam, O.pose(), 1.0, 2.0)
    g["p"][::3, 10] = np.log(0.001 / 0.999)  # a third below the threshold
    om, gm = pair(g)
    gt = O.render(O.OracleMap(round32(random_scene(5, 40, cam, O.pose()))), O.pose(), cam)
    color = f32(gt.color)
    okf = O.Keyframe(O.pose(), color, np.zeros((48, 64)), 20, 0)
    gkf = G().Keyframe(gpu_pose(O.pose()), color, np.zeros((48, 64)), 20, 0)
    ocfg = O.make_cfg(0.2, 0.0, 0)
    gcfg = G().TrainConfig.make(0.2, 0.0, 0)
    for _ in range(3):
        O.train_keyframe_step(om, okf, ocfg, cam)
        G().train_keyframe_step(gm, gkf, gcfg, gpu_cam(cam))
    ro, rg = om.prune(0.005), gm.prune(0.005)
    assert ro == rg == 20
    assert len(om) == len(gm) == 40
    lr = np.array([1.6e-4 * om.scene_extent] * 3 + [1e-3] * 4 + [5e-3] * 3 + [5e-2] + [2.5e-3] * 48)
    assert np.all(np.abs(gm.gaussians["p"] - om.gaussians["p"]) <= 3 * 2 * lr + 1e-6)
    om_m, om_v, om_s = om.adam_state()
    gm_m, gm_v, gm_s = gm.adam_state()
    np.testing.assert_array_equal(om_s, gm_s)
    o_out = O.render(om, O.pose(), cam)
    g_out = G().render(gm, gpu_pose(O.pose()), gpu_cam(cam))
    assert np.abs(g_out.color - o_out.color).max() < 2e-2  # params differ by a few Adam steps
    r_o = O.train_keyframe_step(om, okf, ocfg, cam)
    r_g = G().train_keyframe_step(gm, gkf, gcfg, gpu_cam(cam))
    assert r_g["loss"] == pytest.approx(r_o["loss"], rel=5e-3)


def test_project_sparse_depth_kats_and_oracle():  # test_io.cpp:106-147
    from oracle import pyoracle as O
    cam = O.camera(100, 100, 32, 32, 64, 64)
    p = np.array([[0.0, 0.0, 2.0, 0.5, 0.5, 0.5]])
    d1 = G().project_sparse_depth(p, gpu_pose(O.pose()), gpu_cam(cam))
    assert d1[32, 32] == 2.0 and (d1 > 0).sum() == 1
    far = p.copy(); far[0, 2] = 3.0
    d2 = G().project_sparse_depth(np.concatenate([far, p]), gpu_pose(O.pose()), gpu_cam(cam))
    assert d2[32, 32] == 2.0  # min depth wins
    gen = np.random.default_rng(8)
    cloud = np.zeros((500, 6))
    cloud[:, :3] = gen.uniform(-1.5, 1.5, (500, 3)); cloud[:, 2] += 2.0
    pose = random_pose(gen, 0.3)
    dg = G().project_sparse_depth(cloud, gpu_pose(pose), gpu_cam(cam))
    do = O.project_sparse_depth(cloud, pose, cam)
    np.testing.assert_array_equal(dg, do)  # bit-exact (fp64 transform in the oracle's order)
    assert (dg > 0).sum() <= len(cloud)
    gen.shuffle(cloud)
    np.testing.assert_array_equal(G().project_sparse_depth(cloud, gpu_pose(pose), gpu_cam(cam)), dg)


def test_project_sparse_depth_matches_oracle_on_scene_clouds():
    from fixtures import pyfixture as F
    from oracle import pyoracle as O
    scene = F.Scene(n_gaussians=20000, width=320, height=256, n_frames=3, seed=1)
    cam = O.camera(*scene.camera)
    for f in range(3):
        q = scene.poses[f]
        pose = O.pose(q[0], q[1], q[2], q[3], t=q[4:7])
        cloud = scene.cloud(f)
        dg = G().project_sparse_depth(cloud, gpu_pose(pose), gpu_cam(cam))
        np.testing.assert_array_equal(dg, O.project_sparse_depth(cloud, pose, cam))
        np.testing.assert_array_equal(dg, scene.sparse_depth(f))


def _init_close(gp, op):
    """fp32 parameters equal; the log-scale may differ by 1 fp32 ulp in rare cases (the reference
    sums its 3 distances in heap order, the device in ascending order: <= 1 fp64 ulp apart)."""
    a, b = gp.astype(np.float32), op.astype(np.float32)
    other = np.r_[0:7, 10:59]
    np.testing.assert_array_equal(a[:, other], b[:, other])
    ulp = np.abs(a[:, 7:10].view(np.int32).astype(np.int64) - b[:, 7:10].view(np.int32).astype(np.int64))
    assert ulp.max() <= 1 and (ulp == 0).mean() >= 0.999


@pytest.mark.parametrize("n,spread", [(1, 1.0), (2, 1.0), (7, 0.01), (3000, 3.0)])
def test_init_from_points_matches_oracle(n, spread):  # mapper.cpp:19-61, test_mapper.cpp init KATs
    from oracle import pyoracle as O
    gen = np.random.default_rng(n)
    pts = np.zeros((n, 6))
    pts[:, :3] = gen.uniform(-spread, spread, (n, 3)) + np.array([0.0, 0.0, 4.0])
    pts[:, 3:] = gen.uniform(0, 1, (n, 3))
    if n >= 7:
        pts[1, :3] = pts[0, :3]  # a duplicate point: distance 0 -> floored scale
    om = O.OracleMap()
    assert om.init_from_points(pts) == n
    gm = G().GaussianMap(None)
    assert gm.init_from_points(pts) == n
    assert len(gm) == n
    _init_close(gm.gaussians["p"], om.gaussians["p"])
    assert np.all(gm.gaussians["degree"] == 0)
    # the device keeps fp32 positions: its extent is the oracle's on the fp32-rounded map
    assert gm.scene_extent == pytest.approx(O.OracleMap(round32(om.gaussians)).scene_extent, rel=1e-12)
    m, v, steps = gm.adam_state()
    assert np.all(m == 0) and np.all(v == 0) and np.all(steps == 0)


def test_init_from_points_appends_and_matches_fixture_grid():
    """On a scene's LiDAR cloud: the fixture's CPU grid 3-NN (same ascending sum) agrees exactly,
    and appending to a non-empty map keeps the existing Gaussians and optimizer state."""
    from fixtures import pyfixture as F
    scene = F.Scene(n_gaussians=20000, width=320, height=256, n_frames=2, seed=1)
    cloud = scene.cloud(0)
    ref = F.init_from_points(cloud, threads=1)
    gm = G().GaussianMap(None, round32(ref[:10]))
    before = gm.gaussians["p"].copy()
    assert gm.init_from_points(cloud) == len(cloud)
    p = gm.gaussians["p"]
    np.testing.assert_array_equal(p[:10], before)
    np.testing.assert_array_equal(p[10:].astype(np.float32), ref["p"].astype(np.float32))


def test_sh_schedule():  # test_mapper.cpp:278-296 on the device map
    m = G().GaussianMap(None)
    m.init_from_points(np.array([[0, 0, 2, 0.5, 0.5, 0.5]], dtype=float))
    m.global_step = 99
    assert m.maybe_upgrade_sh(100) == 0
    m.global_step = 100
    assert m.maybe_upgrade_sh(100) == 1
    m.global_step = 300
    assert m.maybe_upgrade_sh(100) == 3
    assert m.gaussians["degree"][0] == 3
    m.global_step = 1000
    assert m.maybe_upgrade_sh(100) == 3
    assert m.maybe_upgrade_sh(0) == 3  # disabled: the current maximum


def _kf_cam():
    return O.camera(100, 100, 31.5, 23.5, 64, 48)


def _opaque(pos, opacity):  # test_keyframe.cpp:22-30
    return O.make_blob(pos, opacity, (0.8, 0.2, 0.2), log_scale=np.log(0.5))


def test_filter_points_by_visibility_kats():  # test_keyframe.cpp:98-136 on the device
    cam, pose = _kf_cam(), O.pose()
    gen = np.random.default_rng(1)
    pts = np.zeros((20, 6))
    pts[:, :3] = gen.uniform(-1, 1, (20, 3)) + [0, 0, 3.0]
    empty = G().GaussianMap(None)
    np.testing.assert_array_equal(G().filter_points_by_visibility(pts, empty, gpu_pose(pose), gpu_cam(cam), 0.5), pts)
    wall = np.concatenate([_opaque((x, y, 4.0), 0.95) for x in np.arange(-2.0, 2.0 + 1e-9, 0.25)
                           for y in np.arange(-1.5, 1.5 + 1e-9, 0.25)])
    _, gm = pair(wall)
    pts = np.array([[0, 0, 3.0, 0, 0, 0], [50, 0, 3.0, 0.1, 0.2, 0.3], [0, 0, -3.0, 0, 0, 0]])
    kept = G().filter_points_by_visibility(pts, gm, gpu_pose(pose), gpu_cam(cam), 0.5)
    np.testing.assert_array_equal(kept, pts[1:])
    for tau in (-0.1, 1.5):
        with pytest.raises(ValueError, match="tau_alpha"):
            G().filter_points_by_visibility(pts, gm, gpu_pose(pose), gpu_cam(cam), tau)


def _filter_case(seed, n_pts):
    cam = O.camera(300, 300, 159.5, 119.5, 320, 240)
    pose = O.pose(1, 0.02, -0.03, 0.01, t=(0.05, -0.02, 0.1))
    g = random_scene(seed, 3000, cam, pose)
    om, gm = pair(g)
    gen = np.random.default_rng(seed)
    pts = np.zeros((n_pts, 6))
    pts[:, 2] = gen.uniform(-1.0, 9.0, n_pts)
    pts[:, 0] = gen.uniform(-0.7, 0.7, n_pts) * np.abs(pts[:, 2])
    pts[:, 1] = gen.uniform(-0.6, 0.6, n_pts) * np.abs(pts[:, 2])
    pts[:, 3:] = gen.uniform(0, 1, (n_pts, 3))
    return cam, pose, om, gm, pts


@pytest.mark.parametrize("tau", [0.0, 0.3, 0.5, 0.9, 1.0])
def test_filter_points_by_visibility_matches_oracle(tau):  # keyframe.cpp:49-74
    """Kept sets equal; a point may differ only where the oracle's fp64 visibility at its pixel
    is within the render tolerance (1e-5) of tau (the device's visibility is fp32)."""
    cam, pose, om, gm, pts = _filter_case(7, 20000)
    ref = O.filter_points_by_visibility(pts, om, pose, cam, tau)
    kept = G().filter_points_by_visibility(pts, gm, gpu_pose(pose), gpu_cam(cam), tau)
    ok = np.zeros(len(pts), bool); ok[ref] = True
    row = {r.tobytes(): i for i, r in enumerate(pts)}
    dev = np.zeros(len(pts), bool)
    order = [row[r.tobytes()] for r in kept]
    assert order == sorted(order)  # stable: the input order
    dev[order] = True
    diff = np.nonzero(dev != ok)[0]
    if len(diff):
        vis = O.render(om, pose, cam).visibility
        w, x, y, z = pose.qw, pose.qx, pose.qy, pose.qz
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        for i in diff:
            pc = R @ pts[i, :3] + [pose.tx, pose.ty, pose.tz]
            px = int(np.floor(cam.fx * pc[0] / pc[2] + cam.cx + 0.5))
            py = int(np.floor(cam.fy * pc[1] / pc[2] + cam.cy + 0.5))
            assert abs(vis[py, px] - tau) < 1e-5, (i, vis[py, px])
    assert (dev != ok).sum() <= 3
    assert 0 < ok.sum() <= len(pts)


def test_integrate_points_matches_filter_then_init():  # pipeline.cpp:151-155
    cam, pose, om, gm, pts = _filter_case(11, 5000)
    ref = O.filter_points_by_visibility(pts, om, pose, cam, 0.5)
    n0 = len(gm)
    before = gm.gaussians["p"].copy()
    assert gm.integrate_points(pts, gpu_pose(pose), gpu_cam(cam), 0.5) == len(ref)
    assert len(gm) == n0 + len(ref)
    p = gm.gaussians["p"]
    np.testing.assert_array_equal(p[:n0], before)
    fresh = O.OracleMap()
    fresh.init_from_points(pts[ref])
    _init_close(p[n0:], fresh.gaussians["p"])
    m, v, steps = gm.adam_state()
    assert np.all(m[n0:] == 0) and np.all(v[n0:] == 0)


def test_batch_trainer_matches_summed_oracle_views():  # sum of per-view grads, one Adam step
    """BatchTrainer at world size 1 (the collective is skipped): the accumulated gradient planes
    equal the oracle's per-view RenderGradients summed (GaussianGrad::add), and the replica
    after the single Adam step tracks the oracle's apply_gradients of that sum."""
    from paper_2411_02703_b200.batch import BatchTrainer
    import torch
    from tests._common import grad_errors
    cam = O.camera(120, 120, 47.5, 39.5, 96, 80)
    gt_map = O.random_scene(O.Rng(31), 60, cam, O.pose(), 1.0, 2.0)
    g = gt_map.gaussians
    g["p"][:, 10] = np.log(0.3 / 0.7)
    g["p"][:, 7:10] += 0.3
    om, gm = pair(g)
    gen = np.random.default_rng(5)
    poses = [O.pose(1.0, *(gen.normal(size=3) * 0.02), t=tuple(gen.normal(size=3) * 0.05)) for _ in range(4)]
    ocfg = O.make_cfg(0.2, 0.5, 0)
    gcfg = G().TrainConfig.make(0.2, 0.5, 0)
    kfs, acc = [], np.zeros((len(g), 59))
    for p in poses:
        gt = O.render(gt_map, p, cam)
        color = f32(gt.color)
        sparse = f32(np.where(gen.uniform(size=(80, 96)) < 0.2, gt.depth, 0.0))
        kfs.append(G().Keyframe(gpu_pose(p), color, sparse, 6, 0))
        out = O.render(om, p, cam)
        loss = O.compute_loss(out.color, out.depth, out.visibility, color, sparse, ocfg)
        acc += O.render_backward(om, p, cam, out, loss["dl_dcolor"], loss["dl_ddepth"])
    tr = BatchTrainer(gm, gm.ctx, torch.device("cuda:0"))
    assert tr.step(kfs, range(4), gcfg, gpu_cam(cam)) == 4
    torch.cuda.synchronize()
    gg = tr.buf.view(59, tr.cap)[:, : len(g)].T.double().cpu().numpy()
    e, ge = grad_errors(gg, acc, round32(g))
    assert ge.max() < 1e-3 and np.mean(e < 1e-3) >= 0.995
    om.apply_gradients(acc)
    lr = np.array([1.6e-4 * om.scene_extent] * 3 + [1e-3] * 4 + [5e-3] * 3 + [5e-2] + [2.5e-3] * 48)
    d = np.abs(gm.gaussians["p"] - om.gaussians["p"])
    assert np.all(d <= 2 * lr + 1e-6)
    assert np.mean(d <= 0.05 * lr + 1e-6) > 0.95
    assert gm.global_step == 1


def test_train_step_prefetch_matches_upload_then_step():  # gs_train_step_prefetch
    """Uploading step s+1's level behind step s (copy stream) gives the same training as
    uploading each level right before its step; the prefetched data is what step s+1 reads."""
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    gt = O.random_scene(O.Rng(21), 40, cam, O.pose(), 1.0, 2.0)
    g = gt.gaussians
    g["p"][:, 10] = np.log(0.1 / 0.9)
    color_x = f32(O.render(gt, O.pose(), cam).color)
    gen = np.random.default_rng(4)
    color_y = f32(np.clip(color_x + gen.normal(0, 0.05, color_x.shape), 0, 1))
    sparse = np.zeros((48, 64))
    ky = G().Keyframe(gpu_pose(O.pose()), color_y, sparse, 100, 2)
    host = [tuple(np.ascontiguousarray(a, np.float64) for a in ky.level(l)) for l in range(3)]
    cfg = G().TrainConfig.make(0.2, 0.5, 2, 1)
    lv = lambda s: 2 - (s % 3)
    _, m1 = pair(g)
    _, m2 = pair(g)
    k1 = G().Keyframe(gpu_pose(O.pose()), color_x, sparse, 100, 2)
    k2 = G().Keyframe(gpu_pose(O.pose()), color_x, sparse, 100, 2)
    r1, r2 = [], []
    for s in range(6):
        k1.consumed_iters = 2 - lv(s)
        k1.upload_level(lv(s), *host[lv(s)])
        r1.append(G().train_keyframe_step(m1, k1, cfg, gpu_cam(cam)))
    k2.upload_level(lv(0), *host[lv(0)])
    for s in range(6):
        k2.consumed_iters = 2 - lv(s)
        pf = (k2, lv(s + 1), *host[lv(s + 1)]) if s < 5 else None
        r2.append(G().train_keyframe_step(m2, k2, cfg, gpu_cam(cam), prefetch=pf))
    for a, b in zip(r1, r2):
        assert a["level"] == b["level"] and a["loss"] == pytest.approx(b["loss"], rel=1e-12)
    np.testing.assert_array_equal(m1.gaussians["p"], m2.gaussians["p"])
    # images are checked against the level's shape (the C side reads exactly that many doubles);
    # other dtypes / layouts are converted first
    with pytest.raises(ValueError, match="needs colour"):
        G().train_keyframe_step(m2, k2, cfg, gpu_cam(cam), prefetch=(k2, 0, host[1][0], host[1][1]))
    with pytest.raises(ValueError, match="needs colour"):
        k2.upload_level(0, host[0][0][:, :-1], host[0][1])
    k2.upload_level(0, host[0][0].astype(np.float32), np.asfortranarray(host[0][1]))
    c, d = k2.level(0)
    np.testing.assert_array_equal(c, host[0][0].astype(np.float32))
    np.testing.assert_array_equal(d, host[0][1])


def test_speculative_next_render_changes_nothing():  # gs_train_step_prefetch with a (keyframe, level) hint
    """Naming the next step lets the library enqueue its render during this step's read-back.
    Training with correct hints, wrong hints, and a host edit of the map between steps gives
    exactly the training without hints."""
    cam = O.camera(100, 100, 31.5, 23.5, 64, 48)
    gt = O.random_scene(O.Rng(23), 60, cam, O.pose(), 1.0, 2.0)
    g = gt.gaussians
    g["p"][:, 10] = np.log(0.2 / 0.8)
    poses = [O.pose(), O.pose(1, 0.0, 0.02, 0.0, t=(0.05, 0.0, 0.0))]
    colors = [f32(O.render(gt, p, cam).color) for p in poses]
    cfg = G().TrainConfig.make(0.2, 0.5, 2, 1)
    sched = [(k, 2 - s % 3) for k in (0, 1, 0, 1) for s in range(3)]

    def run(mode):
        _, m = pair(g)
        kfs = [G().Keyframe(gpu_pose(poses[k]), colors[k], np.zeros((48, 64)), 3, 2) for k in (0, 1)]
        reps = []
        for i, (k, lvl) in enumerate(sched):
            if kfs[k].consumed_iters >= 3:
                kfs[k].consumed_iters = 0
            hint = None
            if i + 1 < len(sched):
                nk, nl = sched[i + 1]
                if mode == "hint":
                    hint = (kfs[nk], nl)
                elif mode == "wrong":
                    hint = (kfs[1 - nk], (nl + 1) % 3)
                elif mode == "edit":
                    hint = (kfs[nk], nl)
            rep = G().train_keyframe_step(m, kfs[k], cfg, gpu_cam(cam), prefetch=hint)
            assert rep["level"] == lvl
            reps.append(rep["loss"])
            if mode == "edit" and i == 4:  # host edit between steps: the speculation is stale
                gg = m.gaussians
                gg["p"][:, 10] -= 0.01
                m.gaussians = gg
        return reps, m.gaussians["p"]

    import ctypes
    ctx = G().default_context()
    cnt = np.zeros(2, np.int64)
    spec = lambda: (G().lib().gs_debug_speculation(ctypes.c_void_p(ctx.h), cnt.ctypes.data_as(ctypes.c_void_p)),
                    cnt.copy())[1]
    base_l, base_p = run(None)
    for mode in ("hint", "wrong"):
        before = spec()
        l, p = run(mode)
        after = spec()
        if mode == "hint":
            assert after[1] - before[1] >= 4  # speculative renders were actually used
        else:
            assert after[1] == before[1]      # mispredicted: enqueued, never used
        np.testing.assert_allclose(l, base_l, rtol=1e-12)
        np.testing.assert_array_equal(p, base_p)
    # the edited run differs from the base but must equal an edited run without hints
    l_e, p_e = run("edit")
    _, m2 = pair(g)
    # replay "edit" without hints
    kfs = [G().Keyframe(gpu_pose(poses[k]), colors[k], np.zeros((48, 64)), 3, 2) for k in (0, 1)]
    ref = []
    for i, (k, lvl) in enumerate(sched):
        if kfs[k].consumed_iters >= 3:
            kfs[k].consumed_iters = 0
        ref.append(G().train_keyframe_step(m2, kfs[k], cfg, gpu_cam(cam))["loss"])
        if i == 4:
            gg = m2.gaussians
            gg["p"][:, 10] -= 0.01
            m2.gaussians = gg
    np.testing.assert_allclose(l_e, ref, rtol=1e-12)
    np.testing.assert_array_equal(p_e, m2.gaussians["p"])


def test_speculation_survives_capacity_overflow():
    """A speculative next-step render that outgrows its frame's remembered pair capacity is
    caught by the step that uses it (overflow flag) and re-run at exact size: training with
    hints across a capacity jump equals plain training."""
    import ctypes
    cam = O.camera(400, 400, 319.5, 239.5, 640, 480)
    g = random_scene(31, 6000, cam, O.pose(), 0.0, 2.0)
    small, big = g.copy(), g.copy()
    small["p"][:, 7:10] = np.log(0.002)
    big["p"][:, 7:10] = np.log(0.2)
    gen = np.random.default_rng(2)
    color = f32(gen.uniform(0, 1, (480, 640, 3)))
    sparse = f32(np.where(gen.uniform(size=(480, 640)) < 0.1, gen.uniform(1, 8, (480, 640)), 0.0))
    cfg = G().TrainConfig.make(0.2, 0.5, 0)
    pose = G().Pose(1, 0, 0, 0, 0, 0, 0)

    ctx1 = G().Context(0)
    ms = G().GaussianMap(ctx1, round32(small))
    ks = G().Keyframe(pose, color, sparse, 10, 0, ctx=ctx1)
    for _ in range(4):  # both train frames learn the small capacity
        G().train_keyframe_step(ms, ks, cfg, gpu_cam(cam), prefetch=(ks, 0))
    mb1 = G().GaussianMap(ctx1, round32(big))
    kb1 = G().Keyframe(pose, color, sparse, 10, 0, ctx=ctx1)
    r1 = [G().train_keyframe_step(mb1, kb1, cfg, gpu_cam(cam), prefetch=(kb1, 0) if i < 3 else None)["loss"]
          for i in range(4)]
    cnt = np.zeros(2, np.int64)
    G().lib().gs_debug_speculation(ctypes.c_void_p(ctx1.h), cnt.ctypes.data_as(ctypes.c_void_p))
    assert cnt[1] >= 2  # speculative renders were used, overflowing ones included

    ctx2 = G().Context(0)
    mb2 = G().GaussianMap(ctx2, round32(big))
    kb2 = G().Keyframe(pose, color, sparse, 10, 0, ctx=ctx2)
    r2 = [G().train_keyframe_step(mb2, kb2, cfg, gpu_cam(cam))["loss"] for _ in range(4)]
    np.testing.assert_allclose(r1, r2, rtol=1e-9)
    assert mb1.global_step == mb2.global_step == 4
    d = np.abs(mb1.gaussians["p"] - mb2.gaussians["p"])
    assert np.mean(d <= 1e-6) > 0.999 and d.max() < 0.2
