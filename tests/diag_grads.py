"""Diagnostic (not a test): where do GPU and oracle gradients differ?"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle as O  # noqa: E402
from tests._common import pair, random_pose, random_scene, rel_err  # noqa: E402
from tests.test_gpu_backward import active_columns, both_grads  # noqa: E402

names = ["px", "py", "pz", "qw", "qx", "qy", "qz", "s0", "s1", "s2", "op"] + [f"sh{k}{c}" for k in range(16) for c in "rgb"]
GROUPS = [(0, 3), (3, 7), (7, 10), (10, 11)] + [(11 + 3 * k, 14 + 3 * k) for k in range(16)]


def group_err(a, b):
    out = np.zeros((a.shape[0], len(GROUPS)))
    for gi, (s, e) in enumerate(GROUPS):
        d = np.linalg.norm(a[:, s:e] - b[:, s:e], axis=1)
        n = np.maximum(np.maximum(np.linalg.norm(a[:, s:e], axis=1), np.linalg.norm(b[:, s:e], axis=1)), 1e-6)
        out[:, gi] = d / n
    return out


for seed in range(6):
    gen = np.random.default_rng(100 + seed)
    cam = O.camera(120, 120, 63.5, 47.5, 128, 96)
    pose = random_pose(gen)
    om, gm = pair(random_scene(100 + seed, 250, cam, pose))
    dc = gen.uniform(-1, 1, (96, 128, 3)); dd = gen.uniform(-1, 1, (96, 128))
    og, gg = both_grads(om, gm, pose, cam, dc, dd)
    mask = active_columns(om.gaussians)
    e = rel_err(gg, og); e[~mask] = 0
    ge = group_err(gg, og)
    bad = np.argwhere(e > 1e-3)
    print(f"seed {seed}: scalars>1e-3 {len(bad)} / {mask.sum()}  gauss-bad {len(set(bad[:,0]))}  worst-group {ge.max():.2e}")
    for i, j in bad[:6]:
        print("   g %d %s oracle %.6e gpu %.6e rowmax %.3e err %.2e" % (i, names[j], og[i, j], gg[i, j], np.abs(og[i]).max(), e[i, j]))
