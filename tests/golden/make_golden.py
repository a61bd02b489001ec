"""Freezes the REFERENCE's outputs as this repo's golden fixtures (the reference
stores no golden vectors). They are produced by the reference itself — its own sources under
/root/reference/proj/src compiled unchanged into oracle/_ref/libgsref.so (oracle/ref/Makefile,
against the Eigen 3.4 subset restatement oracle/ref_eigen) — through oracle/pyref.py. The
tests then require the oracle restatement (tests/test_golden_cpu.py) and the device
(tests/test_gpu_golden.py) to reproduce them.

    python tests/golden/make_golden.py        # rewrites tests/golden/lvigs_crop.npz (needs
                                              # /root/reference: run in the build container)

generate(O) with O = oracle.pyoracle runs the same workload on the restatement.

Workload: a crop of the bench's synthetic scene (the reference's generate_synthetic_scene
restated in fixtures/: walls + speckle, line trajectory, LiDAR clouds) at 4000 Gaussians and
160x128, with the colourised-LiDAR training map (3-NN init). Everything below is fp64 on
fp32-representable parameters (the device's storage):
  - frame 0 render: colour / depth / visibility, contributor counts, depth order and the tile
    lists (bin_tiles order as map indices; bin_tiles is internal to rasterizer.cpp, so the lists
    are derived from the reference's projected means and radii by tile_lists() below, which
    restates rasterizer.cpp:76-91);
  - the C1 loss (L1 only) against the GT render, its dL/dC and the backward's gradients;
  - 3 C1 training steps (level 0, L1 only) and 6 pyramid steps (3 levels, L1 + SSIM + depth).
Image-valued outputs are stored as float32 (the comparison bars are >= 1e-5); integer outputs
and trained parameters exactly.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from fixtures import pyfixture as F  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lvigs_crop.npz")
N, W, H = 4000, 160, 128


def round32(g):
    g = g.copy()
    g["p"] = g["p"].astype(np.float32).astype(np.float64)
    return g


def f32(a):
    return np.asarray(a, np.float32)


def tile_lists(pr, width, height, tile=16):
    """bin_tiles (rasterizer.cpp:76-91) from the projected list: (tile offsets, ranks)."""
    tx_n, ty_n = (width + tile - 1) // tile, (height + tile - 1) // tile
    bins = [[] for _ in range(tx_n * ty_n)]
    for r, ((mx, my), rad) in enumerate(zip(pr["mean"], pr["radius"])):
        x0 = max(0, int(np.ceil(mx - rad))); x1 = min(width - 1, int(np.floor(mx + rad)))
        y0 = max(0, int(np.ceil(my - rad))); y1 = min(height - 1, int(np.floor(my + rad)))
        if x0 > x1 or y0 > y1:
            continue
        for ty in range(y0 // tile, y1 // tile + 1):
            for tx in range(x0 // tile, x1 // tile + 1):
                bins[ty * tx_n + tx].append(r)
    off = np.zeros(len(bins) + 1, np.int64)
    off[1:] = np.cumsum([len(b) for b in bins])
    ent = np.array([r for b in bins for r in b], np.int64)
    return off, ent


def generate(O=None):
    """The golden workload on O (default: the reference through oracle/pyref.py)."""
    if O is None:
        from oracle import pyref
        O = pyref.load()
    scene = F.Scene(n_gaussians=N, width=W, height=H, n_frames=2, seed=1)
    cam = O.camera(*scene.camera)
    poses = [O.pose(p[0], p[1], p[2], p[3], t=p[4:7]) for p in scene.poses]
    train = round32(scene.training_map(seed=2, noise=0.06, threads=1))
    gt = O.render(O.OracleMap(round32(scene.gaussians)), poses[0], cam)
    gt_color = f32(gt.color).astype(np.float64)
    sparse = f32(scene.sparse_depth(0)).astype(np.float64)

    m = O.OracleMap(train)
    out = O.render(m, poses[0], cam)
    pr = out.projected()
    off, ent = tile_lists(pr, W, H)
    tile_gid = pr["index"][ent].astype(np.int32)

    c1 = O.make_cfg(0.0, 0.0, 0)
    loss = O.compute_loss(out.color, out.depth, out.visibility, gt_color, sparse, c1)
    dc = f32(loss["dl_dcolor"]).astype(np.float64)
    dd = np.zeros((H, W))
    grads = O.render_backward(m, poses[0], cam, out, dc, dd)

    c1_losses, c1_psnr = [], []
    mt = O.OracleMap(train)
    kf = O.Keyframe(poses[0], gt_color, sparse, 3, 0)
    for _ in range(3):
        r = O.train_keyframe_step(mt, kf, c1, cam)
        c1_losses.append(r["loss"]); c1_psnr.append(r["psnr"])
    c1_params = mt.gaussians["p"].copy()

    c3 = O.make_cfg(0.2, 0.5, 2, 2)
    mp = O.OracleMap(train)
    kp = O.Keyframe(poses[0], gt_color, sparse, 6, 2)
    c3_losses, c3_levels = [], []
    for _ in range(6):
        r = O.train_keyframe_step(mp, kp, c3, cam)
        c3_losses.append(r["loss"]); c3_levels.append(r["level"])
    c3_params = mp.gaussians["p"].copy()

    return dict(
        camera=np.array(scene.camera, np.float64), pose0=np.array(scene.poses[0], np.float64),
        train_p=train["p"], train_degree=train["degree"].astype(np.int8),
        gt_color=f32(gt_color), sparse_depth=f32(sparse),
        color=f32(out.color), depth=f32(out.depth), visibility=f32(out.visibility),
        n_contrib=out.n_contrib().astype(np.int32), order=pr["index"].astype(np.int32),
        depth_sorted=pr["depth"], tile_off=off.astype(np.int64), tile_gid=tile_gid,
        c1_loss=np.array([loss["total"], loss["l1"]]), c1_dl_dcolor=f32(dc), c1_grads=grads,
        c1_step_losses=np.array(c1_losses), c1_step_psnr=np.array(c1_psnr), c1_params=c1_params,
        c3_step_losses=np.array(c3_losses), c3_step_levels=np.array(c3_levels, np.int32), c3_params=c3_params,
    )


if __name__ == "__main__":
    d = generate()
    np.savez_compressed(OUT, **d)
    print(OUT, os.path.getsize(OUT), "bytes;", {k: v.shape for k, v in d.items()})
