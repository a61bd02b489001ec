"""The forward's execution variants render the same image, through the C-ABI on the device.

The blend's per-pixel arithmetic does not depend on how the pixels of a tile are spread over
threads (2 or 4 per thread), on the order the tiles are launched in (longest list first), or on
which warp-uniform entry variant (rect covers the live box / opacity below 0.99f) evaluates an
entry: those must agree bitwise. The transmittance modes (fp32 + error band, df32) and the
segmented forward take every termination decision exactly (rasterizer.cpp:143-151), so they must
agree on every pixel's contributor count, with colours equal to fp32 rounding.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from tests._common import gpu_cam, gpu_pose, pair, random_pose, random_scene

pytestmark = pytest.mark.gpu


def G():
    from paper_2411_02703_b200 import gsmap
    return gsmap


def scene(seed=5, n=40000):
    gen = np.random.default_rng(seed)
    cam = O.camera(330, 330, 159.5, 127.5, 320, 256)
    pose = random_pose(gen, 0.1)
    _, gm = pair(random_scene(seed, n, cam, pose, -1.0, 1.5))
    return gm, pose, cam


def state(gm, pose, cam):
    out = G().render(gm, gpu_pose(pose), gpu_cam(cam))
    nc, t = out.pixel_state()
    return dict(color=out.color.copy(), depth=out.depth.copy(), vis=out.visibility.copy(), nc=nc, t=t,
                pairs=out.stats().n_pairs)


def test_forward_pixels_per_thread_bitwise():
    gm, pose, cam = scene()
    L = G().lib()
    a = state(gm, pose, cam)
    assert a["pairs"] / ((cam.width // 16) * (cam.height // 16)) > 200  # lists long enough to terminate
    try:
        assert L.gs_debug_set_blend_ppt(4, 0) == 0
        b = state(gm, pose, cam)
    finally:
        L.gs_debug_set_blend_ppt(0, 0)
    for k in ("color", "depth", "vis", "nc", "t"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_forward_transmittance_modes_agree():
    """fp32 + band everywhere vs df32 everywhere: the same stopping contributor for every pixel."""
    gm, pose, cam = scene(seed=9)
    L = G().lib()
    res = {}
    try:
        for name, df_list in (("band", 1 << 30), ("df32", 0)):
            assert L.gs_debug_set_blend_df_list(df_list) == 0
            res[name] = state(gm, pose, cam)
    finally:
        L.gs_debug_set_blend_df_list(-1)
    a, b = res["band"], res["df32"]
    np.testing.assert_array_equal(a["nc"], b["nc"])
    assert (a["nc"] > 0).mean() > 0.5
    for k in ("color", "depth", "vis"):
        np.testing.assert_allclose(a[k], b[k], rtol=0, atol=2e-6, err_msg=k)
    # T_final: band carries fp32 T, df32 the (Th + Tl) sum; both within fp32 rounding of the product
    np.testing.assert_allclose(a["t"], b["t"], rtol=1e-5, atol=1e-12)


def test_segmented_forward_agrees_with_sequential():
    """The segmented forward (local walks, per-pixel chain, exact finish) against the sequential
    walk on the same view and list segments."""
    gm, pose, cam = scene(seed=13)
    L = G().lib()
    res = {}
    try:
        assert L.gs_debug_set_blend_segments(4) == 0
        for name, max_tiles in (("sequential", 0), ("segmented", 1 << 20)):
            assert L.gs_debug_set_seg_forward(max_tiles) == 0
            res[name] = state(gm, pose, cam)
    finally:
        L.gs_debug_set_seg_forward(-1)
        L.gs_debug_set_blend_segments(0)
    a, b = res["sequential"], res["segmented"]
    np.testing.assert_array_equal(a["nc"], b["nc"])
    for k in ("color", "depth", "vis"):
        np.testing.assert_allclose(a[k], b[k], rtol=0, atol=1e-5, err_msg=k)
