"""Diagnostic (not a test): tie runs of the 24-bit depth sort key on the bench workload."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2411_02703_b200 import gsmap as G  # noqa: E402

scene, train, _ = bench.build_fixture(1_000_000)
ctx = G.Context(0)
fx, fy, cx, cy, W, H = scene.camera
cam = G.Camera(fx, fy, cx, cy, W, H)
m = G.GaussianMap(ctx, train)
for f in (0, 3):
    for lvl in (2, 0):
        fr = G.render(m, G.Pose(*scene.poses[f]), G.camera_scaled(cam, lvl))
        pr = fr.projected()
        d = pr["depth"].astype(np.float32)
        base = np.float32(0.01).view(np.uint32)
        k24 = np.minimum((d.view(np.uint32) - base) >> 4, 0xffffff)
        k32 = d.view(np.uint32)
        for name, k in (("k24", k24), ("k32", k32)):
            _, counts = np.unique(k, return_counts=True)
            runs = counts[counts > 1]
            print(f"frame {f} L{lvl} {name}: n={len(k)} tie runs={len(runs)} elems={runs.sum()} max={counts.max()} "
                  f"sum L^2={int((runs.astype(np.int64) ** 2).sum())}", flush=True)
