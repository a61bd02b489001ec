"""Shared helpers for the parity tests: build the SAME inputs for the oracle and the GPU.

The GPU map stores fp32 parameters, so "same inputs" means the fp64 reference map holds the
fp32-representable values the device holds (round32). Poses/cameras are passed bit-for-bit.
"""
import numpy as np

from oracle import pyoracle as O


def round32(g: np.ndarray) -> np.ndarray:
    g = g.copy()
    g["p"] = g["p"].astype(np.float32).astype(np.float64)
    return g


def gpu_pose(p):
    from paper_2411_02703_b200 import gsmap as G
    return G.Pose(p.qw, p.qx, p.qy, p.qz, p.tx, p.ty, p.tz)


def gpu_cam(c):
    from paper_2411_02703_b200 import gsmap as G
    return G.Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height)


def pair(gaussians: np.ndarray, ctx=None):
    """(OracleMap, GaussianMap) holding identical (fp32-representable) parameters."""
    from paper_2411_02703_b200 import gsmap as G
    g = round32(gaussians)
    om = O.OracleMap(g)
    gm = G.GaussianMap(ctx, g)
    return om, gm


def rel_err(a, b, floor=1e-6):
    """gradcheck.cpp:21-24 — |a-b| / max(|a|, |b|, 1e-6)."""
    a = np.asarray(a); b = np.asarray(b)
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)


def rect_of(mean, radius, W, H):
    """rasterizer.cpp:81-84 integer pixel rect of the oracle's projected Gaussian."""
    x0 = np.maximum(0, np.ceil(mean[:, 0] - radius)).astype(np.int64)
    x1 = np.minimum(W - 1, np.floor(mean[:, 0] + radius)).astype(np.int64)
    y0 = np.maximum(0, np.ceil(mean[:, 1] - radius)).astype(np.int64)
    y1 = np.minimum(H - 1, np.floor(mean[:, 1] + radius)).astype(np.int64)
    return np.stack([x0, y0, x1, y1], 1)


def random_scene(seed, n, cam, pose, lo=-2.5, hi=1.5):
    rng = O.Rng(seed)
    return O.random_scene(rng, n, cam, pose, lo, hi).gaussians


def random_pose(gen: np.random.Generator, tscale=0.3):
    q = gen.normal(size=4)
    return O.pose(*q, t=tuple(gen.uniform(-1, 1, 3) * tscale))
