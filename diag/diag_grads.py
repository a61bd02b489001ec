"""Diagnostic (not a test): where do GPU and oracle gradients differ on smooth configs?"""
import sys

import numpy as np

sys.path.insert(0, ".")
from tests.test_gpu_backward import active_columns, both_grads, grad_errors, gradcheck_configs  # noqa: E402

names = ["px", "py", "pz", "qw", "qx", "qy", "qz", "s0", "s1", "s2", "op"] + [f"sh{k}{c}" for k in range(16) for c in "rgb"]
rows = []
for ci, (om, gm, pose, cam, wc, wd) in enumerate(gradcheck_configs(3, 40)):
    og, gg = both_grads(om, gm, pose, cam, wc, wd)
    mask = active_columns(om.gaussians)
    rowmax = np.abs(og).max(axis=1, keepdims=True)
    floor = np.maximum(1e-6, 1e-3 * rowmax)
    e2 = np.abs(gg - og) / np.maximum(np.maximum(np.abs(gg), np.abs(og)), floor)
    e2[~mask] = 0
    for i, j in np.argwhere(e2 > 3e-4):
        rows.append((e2[i, j], ci, i, names[j], og[i, j], gg[i, j], rowmax[i, 0]))
rows.sort(reverse=True)
for r in rows[:15]:
    print("e2 %.2e cfg %d g %d %s oracle %.6e gpu %.6e rowmax %.3e" % r)
