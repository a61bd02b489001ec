"""The oracle restatement (oracle/_build/liborc.so) is pinned to the REFERENCE ITSELF
(oracle/_ref/libgsref.so: /root/reference/proj/src compiled unchanged against the Eigen 3.4
subset restatement oracle/ref_eigen, driven through the same orc_* C-ABI by oracle/pyref.py).

Every comparison below is bitwise (np.array_equal / ==): projected means, depths, 2D
covariances, radii and order; images and the CSR contributor table; gradients; the loss and its
cotangents; SSIM / PSNR; Adam; training steps; pyramids; map growth; sparse depth; the
visibility filter; checkpoints byte for byte; the reference's own synthetic generator against
the fixture restatement; and the reference's own finite-difference gradcheck harness. C1
(100k Gaussians, 640x512) runs render + backward at full size.

The reference build needs /root/reference (this container) or a prebuilt oracle/_ref; without
either the module is skipped.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref

pytestmark = pytest.mark.skipif(not pyref.available(), reason="reference build (oracle/_ref) unavailable")


@pytest.fixture(scope="module")
def R():
    return pyref.load()


def _cam(M, W=128, H=96):
    return M.camera(120.0, 120.0, (W - 1) / 2, (H - 1) / 2, W, H)


def _pose(M, k=0):
    qs = [(0.98, 0.05, -0.1, 0.02, (0.05, -0.02, 0.1)), (0.9, -0.2, 0.3, 0.1, (-0.3, 0.1, 0.4)),
          (1.0, 0.0, 0.0, 0.0, (0.0, 0.0, 0.0))]
    w, x, y, z, t = qs[k]
    return M.pose(w, x, y, z, t=t)


def _scene(M, seed, n, cam, pose, lo=-2.5, hi=1.5):
    return M.random_scene(M.Rng(seed), n, cam, pose, lo, hi).gaussians


def _eq(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, what
    bad = np.flatnonzero(~((a == b) | (np.isnan(a) & np.isnan(b))).ravel())
    assert bad.size == 0, f"{what}: {bad.size} of {a.size} differ, first {bad[:5]}"


def test_build_kind(R):
    import ctypes
    f = R.lib().orc_build_kind
    f.restype = ctypes.c_char_p
    assert f().decode().startswith("reference")
    assert not hasattr(O.lib(), "orc_build_kind")


@pytest.mark.parametrize("k", [0, 1, 2])
def test_pose_and_camera(R, k):
    po, pr = _pose(O, k), _pose(R, k)
    for f in ("qw", "qx", "qy", "qz", "tx", "ty", "tz"):
        assert getattr(po, f) == getattr(pr, f), f
    _eq(O.camera_center(po), R.camera_center(pr), "camera_center")
    for lvl in range(4):
        a = O.camera_scaled(_cam(O, 1283, 1021), lvl)
        b = R.camera_scaled(_cam(R, 1283, 1021), lvl)
        assert a.tuple() == b.tuple()


def test_core_primitives(R):
    gen = np.random.default_rng(3)
    for _ in range(300):
        q = gen.uniform(-1, 1, 4)
        ls = gen.uniform(-4, 1, 3)
        _eq(O.build_covariance(q, ls), R.build_covariance(q, ls), "build_covariance")
        coeffs = gen.uniform(-1, 1, 48)
        d = gen.normal(size=3)
        d /= np.linalg.norm(d)
        for deg in range(4):
            _eq(O.eval_sh(coeffs, deg, d), R.eval_sh(coeffs, deg, d), "eval_sh")
        mean, x = gen.uniform(-3, 3, 2), gen.uniform(-3, 3, 2)
        a = gen.normal(size=(2, 2))
        cov = a @ a.T + 0.3 * np.eye(2)
        assert O.eval_gaussian_2d(mean, cov, x) == R.eval_gaussian_2d(mean, cov, x)
    cam_o, cam_r = _cam(O), _cam(R)
    g = _scene(O, 5, 400, cam_o, _pose(O))
    for i in range(len(g)):
        a = O.project_gaussian(g[i:i + 1], _pose(O, 1), cam_o)
        b = R.project_gaussian(g[i:i + 1], _pose(R, 1), cam_r)
        assert (a is None) == (b is None)
        if a is not None:
            for k in a:
                _eq(a[k], b[k], f"project_gaussian.{k}")


@pytest.mark.parametrize("seed,n,k", [(7, 300, 0), (11, 2000, 1), (13, 800, 2)])
def test_render_and_backward_bitwise(R, seed, n, k):
    cam_o, cam_r = _cam(O), _cam(R)
    assert np.array_equal(_scene(O, seed, n, cam_o, _pose(O, k)), _scene(R, seed, n, cam_r, _pose(R, k)))
    g = _scene(O, seed, n, cam_o, _pose(O, k))
    om, rm = O.OracleMap(g), R.OracleMap(g)
    oo, ro = O.render(om, _pose(O, k), cam_o, threads=4), R.render(rm, _pose(R, k), cam_r, threads=4)
    po, pr = oo.projected(), ro.projected()
    for key in po:
        _eq(po[key], pr[key], f"projected.{key}")
    for a, b, what in ((oo.color, ro.color, "color"), (oo.depth, ro.depth, "depth"),
                       (oo.visibility, ro.visibility, "visibility")):
        _eq(a, b, what)
    for a, b, what in zip(oo.csr(), ro.csr(), ("offsets", "gaussian", "alpha")):
        _eq(a, b, f"csr.{what}")
    gen = np.random.default_rng(seed)
    dc = gen.uniform(-1, 1, (cam_o.height, cam_o.width, 3))
    dd = gen.uniform(-1, 1, (cam_o.height, cam_o.width))
    _eq(O.render_backward(om, _pose(O, k), cam_o, oo, dc, dd, threads=4),
        R.render_backward(rm, _pose(R, k), cam_r, ro, dc, dd, threads=4), "gradients")
    # the tile-free brute-force oracle of the reference tests (tests/support/brute_force.hpp)
    for a, b in zip(O.brute_force(om, _pose(O, k), cam_o), R.brute_force(rm, _pose(R, k), cam_r)):
        _eq(a, b, "brute_force")


@pytest.mark.parametrize("lam,lam_d", [(0.0, 0.0), (0.2, 0.5), (1.0, 0.0), (0.0, 1.0)])
def test_loss_ssim_psnr(R, lam, lam_d):
    gen = np.random.default_rng(int(lam * 10 + lam_d * 100))
    H, W = 37, 53
    color, gt = gen.uniform(0, 1, (H, W, 3)), gen.uniform(0, 1, (H, W, 3))
    depth, vis = gen.uniform(0.5, 5, (H, W)), gen.uniform(0.9, 1.0, (H, W))
    gtd = np.where(gen.uniform(size=(H, W)) < 0.4, gen.uniform(0.5, 5, (H, W)), 0.0)
    a = O.compute_loss(color, depth * vis, vis, gt, gtd, O.make_cfg(lam, lam_d, 0))
    b = R.compute_loss(color, depth * vis, vis, gt, gtd, R.make_cfg(lam, lam_d, 0))
    for key in a:
        _eq(a[key], b[key], f"compute_loss.{key}")
    sa, ga = O.ssim(color, gt, with_grad=True)
    sb, gb = R.ssim(color, gt, with_grad=True)
    assert sa == sb
    _eq(ga, gb, "ssim gradient")
    assert O.psnr(color, gt) == R.psnr(color, gt)
    assert O.depth_rmse(depth, gtd) == R.depth_rmse(depth, gtd)


def test_pyramids(R):
    gen = np.random.default_rng(1)
    img = gen.uniform(0, 1, (77, 101, 3))
    dep = np.where(gen.uniform(size=(77, 101)) < 0.3, gen.uniform(1, 9, (77, 101)), 0.0)
    for a, b in zip(O.build_pyramid(img, 3), R.build_pyramid(img, 3)):
        _eq(a, b, "pyramid")
    for a, b in zip(O.build_pyramid(dep, 3, depth=True), R.build_pyramid(dep, 3, depth=True)):
        _eq(a, b, "depth pyramid")


def test_adam_and_training_steps(R):
    cam_o, cam_r = _cam(O), _cam(R)
    g = _scene(O, 21, 600, cam_o, _pose(O))
    gt = O.render(O.OracleMap(_scene(O, 22, 600, cam_o, _pose(O))), _pose(O), cam_o)
    sparse = np.where(np.random.default_rng(0).uniform(size=gt.depth.shape) < 0.3, gt.depth, 0.0)
    om, rm = O.OracleMap(g), R.OracleMap(g)
    # one Adam step from explicit gradients
    grads = np.random.default_rng(1).normal(size=(len(g), 59)) * 1e-2
    om.apply_gradients(grads)
    rm.apply_gradients(grads)
    _eq(om.gaussians["p"], rm.gaussians["p"], "adam params")
    ma, va, sa = om.adam_state()
    mb, vb, sb = rm.adam_state()
    _eq(ma, mb, "adam m"); _eq(va, vb, "adam v"); _eq(sa, sb, "adam step")
    assert om.scene_extent == rm.scene_extent and om.global_step == rm.global_step
    # a pyramid of training steps (L1 + SSIM + depth), two keyframes, with the SH schedule
    kfo = [O.Keyframe(_pose(O), gt.color, sparse, 6, 2), O.Keyframe(_pose(O, 1), gt.color, sparse, 3, 1)]
    kfr = [R.Keyframe(_pose(R), gt.color, sparse, 6, 2), R.Keyframe(_pose(R, 1), gt.color, sparse, 3, 1)]
    po, pr = O.ThreadPool(4), R.ThreadPool(4)
    for it in range(9):
        a = O.train_keyframe_step(om, kfo[it % 2], O.make_cfg(0.2, 0.5, 2), cam_o, po)
        b = R.train_keyframe_step(rm, kfr[it % 2], R.make_cfg(0.2, 0.5, 2), cam_r, pr)
        assert a == b, (it, a, b)
        assert om.maybe_upgrade_sh(3) == rm.maybe_upgrade_sh(3)
    _eq(om.gaussians["p"], rm.gaussians["p"], "trained params")
    _eq(om.gaussians["degree"], rm.gaussians["degree"], "degrees")
    for x, y in zip(om.adam_state(), rm.adam_state()):
        _eq(x, y, "trained adam state")
    # housekeeping
    assert om.prune(0.3) == rm.prune(0.3)
    _eq(om.gaussians["p"], rm.gaussians["p"], "pruned params")
    om.raise_sh_degree(2); rm.raise_sh_degree(2)
    assert om.max_active_degree() == rm.max_active_degree()


def test_map_growth_sparse_depth_filter_checkpoint(R):
    cam_o, cam_r = _cam(O, 96, 80), _cam(R, 96, 80)
    gen = np.random.default_rng(4)
    pts = np.concatenate([gen.uniform(-2, 2, (700, 2)), gen.uniform(2, 6, (700, 1)), gen.uniform(0, 1, (700, 3))], 1)
    om, rm = O.OracleMap(), R.OracleMap()
    assert om.init_from_points(pts) == rm.init_from_points(pts) == len(pts)
    _eq(om.gaussians["p"], rm.gaussians["p"], "init_from_points")
    assert om.scene_extent == rm.scene_extent
    for k in range(2):
        _eq(O.project_sparse_depth(pts, _pose(O, k), cam_o), R.project_sparse_depth(pts, _pose(R, k), cam_r),
            "project_sparse_depth")
        for tau in (0.2, 0.5, 0.9):
            _eq(O.filter_points_by_visibility(pts, om, _pose(O, k), cam_o, tau),
                R.filter_points_by_visibility(pts, rm, _pose(R, k), cam_r, tau), "filter_points_by_visibility")
    with tempfile.TemporaryDirectory() as d:
        a, b = os.path.join(d, "o.gsmap"), os.path.join(d, "r.gsmap")
        O.save_checkpoint(a, om)
        R.save_checkpoint(b, rm)
        assert open(a, "rb").read() == open(b, "rb").read()
        _eq(O.load_checkpoint(b).gaussians["p"], R.load_checkpoint(a).gaussians["p"], "checkpoint load")


def test_reference_gradcheck_harness(R):
    """gradcheck.cpp (the reference's own FD harness) and its restatement agree exactly."""
    assert O.run_gradcheck(seed=3, configs=12, core_configs=24) == R.run_gradcheck(seed=3, configs=12, core_configs=24)


def test_synthetic_fixture_matches_reference_generator(R):
    """fixtures/synthetic.cpp (the bench's scene) restates io/synthetic.cpp: GT Gaussians, camera,
    poses and LiDAR clouds equal the reference generator's at the same spec."""
    import ctypes as C

    from fixtures import pyfixture as F
    L = R.lib()
    L.orc_synthetic_scene.restype = C.c_void_p
    L.orc_synthetic_scene.argtypes = [C.c_int, C.c_double, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_double,
                                      C.c_double, C.c_int, C.POINTER(C.c_int)]
    L.orc_synthetic_map.restype = C.c_void_p
    L.orc_synthetic_map.argtypes = [C.c_void_p]
    L.orc_synthetic_free.argtypes = [C.c_void_p]
    for traj, n, W, H in (("line", 600, 160, 120), ("orbit", 400, 96, 64)):
        st = C.c_int(0)
        h = L.orc_synthetic_scene(n, 18.0, 4, 1, W, H, 0.8125 * W, 0.06, int(traj == "orbit"), C.byref(st))
        assert st.value == 0, R.lib().orc_last_error()
        ref_map = R.OracleMap(handle=L.orc_synthetic_map(h))
        ref_g = ref_map.gaussians
        ref_map.h = None  # owned by the scene
        try:
            fx = F.Scene(n_gaussians=n, width=W, height=H, n_frames=4, seed=1, trajectory=traj)
            _eq(fx.gaussians["p"], ref_g["p"], "synthetic gaussians")
            _eq(fx.gaussians["degree"], ref_g["degree"], "synthetic degrees")
            cam = R.Camera()
            L.orc_synthetic_camera(C.c_void_p(h), C.byref(cam))
            assert cam.tuple() == tuple(fx.camera)
            for f in range(4):
                pose, npts = R.Pose(), C.c_int64()
                L.orc_synthetic_frame(C.c_void_p(h), f, C.byref(pose), C.byref(npts))
                assert (pose.qw, pose.qx, pose.qy, pose.qz, pose.tx, pose.ty, pose.tz) == tuple(fx.poses[f])
                pts = np.zeros((npts.value, 6))
                L.orc_synthetic_cloud(C.c_void_p(h), f, pts.ctypes.data_as(C.c_void_p))
                _eq(fx.cloud(f), pts, "synthetic cloud")
        finally:
            L.orc_synthetic_free(C.c_void_p(h))


def test_c1_full_size_bitwise(R):
    """C1 (BASELINE configs[0]): 100k Gaussians of the bench scene's colourised-LiDAR training
    map at 640x512 — render and backward equal the reference's bit for bit."""
    from fixtures import pyfixture as F
    scene = F.Scene(n_gaussians=100_000, width=640, height=512, n_frames=2, seed=1)
    g = scene.training_map(seed=2, noise=0.06)
    g["p"] = g["p"].astype(np.float32).astype(np.float64)
    cam_o, cam_r = O.camera(*scene.camera), R.camera(*scene.camera)
    po, pr = O.pose(*scene.poses[0][:4], t=scene.poses[0][4:]), R.pose(*scene.poses[0][:4], t=scene.poses[0][4:])
    om, rm = O.OracleMap(g), R.OracleMap(g)
    oo, ro = O.render(om, po, cam_o, threads=8), R.render(rm, pr, cam_r, threads=8)
    a, b = oo.projected(), ro.projected()
    for key in a:
        _eq(a[key], b[key], f"C1 projected.{key}")
    _eq(oo.color, ro.color, "C1 color")
    _eq(oo.n_contrib(), ro.n_contrib(), "C1 contributor counts")
    dc = np.sign(oo.color - 0.5) / oo.color.size
    dd = np.zeros(oo.depth.shape)
    _eq(O.render_backward(om, po, cam_o, oo, dc, dd, threads=8), R.render_backward(rm, pr, cam_r, ro, dc, dd, threads=8),
        "C1 gradients")
