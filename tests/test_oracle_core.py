"""Pins the CPU oracle's core math against the reference's own known-answer and property tests
(proj/tests/test_core.cpp). The reference cannot be compiled here (no Eigen), so these ports are
what makes the restatement trustworthy before any GPU result is compared to it."""
import math

import numpy as np
import pytest

from oracle import pyoracle as O

RNG = np.random.default_rng(12345)


def random_quat():
    while True:
        q = RNG.uniform(-1, 1, 4)
        if np.linalg.norm(q) >= 0.3:
            return q


def quat_matrix(q):
    """Independent route: textbook unit-quaternion rotation (test_core.cpp:77-81 uses Eigen)."""
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def test_covariance_identity_rotation_squared_scales():  # test_core.cpp:61-65
    s = O.build_covariance([1, 0, 0, 0], [0.0, math.log(2.0), math.log(3.0)])
    assert np.linalg.norm(s - np.diag([1, 4, 9])) < 1e-12


def test_covariance_90deg_z_swaps_axes():  # test_core.cpp:67-72
    c = math.cos(math.pi / 4)
    s = O.build_covariance([c, 0, 0, math.sin(math.pi / 4)], [0.0, math.log(2.0), 0.0])
    assert np.linalg.norm(s - np.diag([4, 1, 1])) < 1e-12


def test_covariance_matches_dense_composition():  # test_core.cpp:74-86
    for _ in range(500):
        q = random_quat()
        s = RNG.uniform(-3, 1, 3)
        r = quat_matrix(q)
        sm = np.diag(np.exp(s))
        expect = r @ sm @ sm.T @ r.T
        assert np.linalg.norm(O.build_covariance(q, s) - expect) < 1e-12


def test_covariance_symmetric_psd():  # test_core.cpp:88-104 (1e4 draws instead of 1e6)
    min_eig, max_asym = 1e300, 0.0
    for _ in range(10000):
        s = O.build_covariance(random_quat(), RNG.uniform(-4, 2, 3))
        max_asym = max(max_asym, np.linalg.norm(s - s.T))
        ev = np.linalg.eigvalsh(s)
        min_eig = min(min_eig, ev.min() / max(1.0, ev.max()))
    assert max_asym == 0.0
    assert min_eig >= -1e-12


def test_covariance_rotation_equivariance():  # test_core.cpp:106-119
    def qmul(a, b):
        w1, x1, y1, z1 = a; w2, x2, y2, z2 = b
        return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                         w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])
    for _ in range(200):
        q1 = random_quat(); q1 /= np.linalg.norm(q1)
        q2 = random_quat(); q2 /= np.linalg.norm(q2)
        s = RNG.uniform(-2, 1, 3)
        lhs = O.build_covariance(qmul(q1, q2), s)
        r1 = quat_matrix(q1)
        assert np.linalg.norm(lhs - r1 @ O.build_covariance(q2, s) @ r1.T) < 1e-10


def test_project_on_axis_principal_point():  # test_core.cpp:121-131
    g = O.empty_gaussians(1); g["p"][0, 0:3] = [0, 0, 1]
    cam = O.camera(100, 100, 50, 50, 101, 101)
    p = O.project_gaussian(g, O.pose(), cam)
    assert p is not None
    assert p["mean"][0] == pytest.approx(50.0, rel=1e-12)
    assert p["mean"][1] == pytest.approx(50.0, rel=1e-12)
    assert p["depth"] == pytest.approx(1.0)
    assert p["radius"] >= 1


def test_project_behind_camera_culled():  # test_core.cpp:133-138
    g = O.empty_gaussians(1); g["p"][0, 0:3] = [0, 0, -1]
    assert O.project_gaussian(g, O.pose(), O.camera(100, 100, 50, 50, 101, 101)) is None


def test_project_mean_equals_pinhole_random_poses():  # test_core.cpp:140-154
    cam = O.camera(80, 90, 31.5, 23.5, 64, 48)
    for _ in range(1000):
        q = RNG.normal(size=4)
        pose = O.pose(*q, t=tuple(RNG.uniform(-1, 1, 3)))
        p_cam = np.array([RNG.uniform(-2, 2), RNG.uniform(-2, 2), RNG.uniform(0.05, 10)])
        r = quat_matrix(np.array([pose.qw, pose.qx, pose.qy, pose.qz]))
        g = O.empty_gaussians(1)
        g["p"][0, 0:3] = r.T @ (p_cam - np.array([pose.tx, pose.ty, pose.tz]))
        g["p"][0, 3:7] = random_quat()
        g["p"][0, 7:10] = RNG.uniform(-3, 0, 3)
        p = O.project_gaussian(g, pose, cam)
        assert p is not None
        assert abs(p["mean"][0] - (cam.fx * p_cam[0] / p_cam[2] + cam.cx)) < 1e-10
        assert abs(p["mean"][1] - (cam.fy * p_cam[1] / p_cam[2] + cam.cy)) < 1e-10


def test_projected_covariance_monte_carlo():  # test_core.cpp:156-184
    sigma, z, fx = 0.1, 2.0, 100.0
    g = O.empty_gaussians(1); g["p"][0, 0:3] = [0, 0, z]; g["p"][0, 7:10] = math.log(sigma)
    p = O.project_gaussian(g, O.pose(), O.camera(fx, fx, 50, 50, 101, 101))
    gen = np.random.default_rng(7)
    q = gen.normal(0.0, sigma, (200000, 3)); q[:, 2] += z
    uv = np.stack([fx * q[:, 0] / q[:, 2] + 50, fx * q[:, 1] / q[:, 2] + 50], 1)
    emp = np.cov(uv.T, bias=True)
    for i in range(2):
        assert abs(p["cov2d"][i, i] - 25.0) < 0.05 * 25.0
    assert np.linalg.norm(emp - (p["cov2d"] - 0.3 * np.eye(2))) < 0.05 * 25.0


def test_eval2d_unit_at_mean_and_offset():  # test_core.cpp:186-193
    m = [3.5, -2.0]
    assert O.eval_gaussian_2d(m, np.eye(2), m) == pytest.approx(1.0, rel=1e-15)
    assert O.eval_gaussian_2d(m, np.eye(2), [4.5, -2.0]) == pytest.approx(math.exp(-0.5), rel=1e-12)


def test_eval2d_matches_solve_oracle():  # test_core.cpp:195-208
    for _ in range(1000):
        a = RNG.uniform(-2, 2, (2, 2))
        cov = a @ a.T + 0.3 * np.eye(2)
        mean = RNG.uniform(-10, 10, 2); x = RNG.uniform(-12, 12, 2)
        d = x - mean
        expect = math.exp(-0.5 * d @ np.linalg.solve(cov, d))
        assert O.eval_gaussian_2d(mean, cov, x) == pytest.approx(expect, rel=1e-12, abs=1e-300)


def test_eval2d_in_unit_interval():  # test_core.cpp:210-224
    for _ in range(300):
        a = RNG.uniform(-2, 2, (2, 2))
        cov = a @ a.T + 0.3 * np.eye(2)
        mean = RNG.uniform(-5, 5, 2); x = RNG.uniform(-8, 8, 2)
        v = O.eval_gaussian_2d(mean, cov, x)
        assert 0.0 < v <= 1.0
        assert v <= O.eval_gaussian_2d(mean, cov, mean)


def sh_reference(i, d):  # test_core.cpp:35-57
    x, y, z = d
    pi = math.pi
    return [0.5 * math.sqrt(1 / pi), math.sqrt(3 / (4 * pi)) * y, math.sqrt(3 / (4 * pi)) * z,
            math.sqrt(3 / (4 * pi)) * x, 0.5 * math.sqrt(15 / pi) * x * y, 0.5 * math.sqrt(15 / pi) * y * z,
            0.25 * math.sqrt(5 / pi) * (3 * z * z - 1), 0.5 * math.sqrt(15 / pi) * x * z,
            0.25 * math.sqrt(15 / pi) * (x * x - y * y), 0.25 * math.sqrt(35 / (2 * pi)) * y * (3 * x * x - y * y),
            0.5 * math.sqrt(105 / pi) * x * y * z, 0.25 * math.sqrt(21 / (2 * pi)) * y * (5 * z * z - 1),
            0.25 * math.sqrt(7 / pi) * (5 * z ** 3 - 3 * z), 0.25 * math.sqrt(21 / (2 * pi)) * x * (5 * z * z - 1),
            0.25 * math.sqrt(105 / pi) * z * (x * x - y * y),
            0.25 * math.sqrt(35 / (2 * pi)) * x * (x * x - 3 * y * y)][i]


def test_sh_degree0_offset():  # test_core.cpp:225-233
    c = np.zeros((16, 3)); c[0] = [0.5 / 0.28209479177387814, 0, 0]
    out = O.eval_sh(c, 0, [0, 0, 1])
    assert out == pytest.approx([1.0, 0.5, 0.5], rel=1e-12)


def test_sh_degree0_view_independent():  # test_core.cpp:235-241
    c = RNG.uniform(-1, 1, (16, 3))
    assert np.linalg.norm(O.eval_sh(c, 0, [1, 0, 0]) - O.eval_sh(c, 0, [0, 0.6, 0.8])) == 0.0


def test_sh_matches_textbook():  # test_core.cpp:243-254
    for _ in range(500):
        c = RNG.uniform(-1, 1, (16, 3))
        d = RNG.uniform(-1, 1, 3)
        while np.linalg.norm(d) < 0.1:
            d = RNG.uniform(-1, 1, 3)
        d /= np.linalg.norm(d)
        expect = 0.5 + sum(sh_reference(i, d) * c[i] for i in range(16))
        assert np.linalg.norm(O.eval_sh(c, 3, d) - expect) < 1e-10


def test_camera_scaling_lattice():  # test_core.cpp:256-265
    cam = O.camera(130, 130, 79.5, 59.5, 160, 120)
    half = O.camera_scaled(cam, 1)
    assert (half.width, half.height) == (80, 60)
    z, u_half = 3.0, 17.0
    x = (2.0 * u_half + 0.5 - cam.cx) * z / cam.fx
    assert half.fx * x / z + half.cx == pytest.approx(u_half, rel=1e-12)


def test_camera_validate_rejects():  # core/types.hpp:22-29
    for bad in (O.camera(0, 1, 0, 0, 4, 4), O.camera(1, 1, 0, 0, 0, 4), O.camera(1, 1, 4.0, 0, 4, 4)):
        with pytest.raises(O.InvalidArgument):
            O.validate_camera(bad)
    O.validate_camera(O.camera(1, 1, 3.9, 0, 4, 4))
