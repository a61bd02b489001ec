"""compute-sanitizer target: a C1-shaped run of the hot path — the bench
fixture's colourised-LiDAR map, a 3-level pyramid keyframe, train_keyframe_step at every level
with the next step named (speculative render), a public render + backward + Adam, a loss read.

    compute-sanitizer --tool memcheck  python profiles/sanitize_step.py 100000 640 512
    compute-sanitizer --tool racecheck python profiles/sanitize_step.py 20000 320 256

Logs from the B200 runs: profiles/r2_sanitizer_*.log."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from fixtures import pyfixture as F  # noqa: E402
from paper_2411_02703_b200 import gsmap as G  # noqa: E402

n, W, H = (int(a) for a in sys.argv[1:4])
scene = F.Scene(n_gaussians=n, width=W, height=H, n_frames=2, seed=1)
train = scene.training_map(seed=2, noise=0.06)
fx, fy, cx, cy, _, _ = scene.camera
cam = G.Camera(fx, fy, cx, cy, W, H)
poses = [G.Pose(*p) for p in scene.poses]
ctx = G.Context(0)
gt = G.render(G.GaussianMap(ctx, scene.gaussians), poses[0], cam).color
kfs = [G.Keyframe(p, gt, scene.sparse_depth(f), 3, 2, ctx=ctx) for f, p in enumerate(poses)]
m = G.GaussianMap(ctx, train)
cfg = G.TrainConfig.make(0.2, 0.5, 2, 1)
for s in range(6):
    kf, nk = kfs[(s // 3) % 2], kfs[((s + 1) // 3) % 2]
    rep = G.train_keyframe_step(m, kf, cfg, cam, prefetch=(nk, 2 - (s + 1) % 3))
    print("step", s, rep)
out = G.render(m, poses[1], cam)
dc = np.sign(out.color - gt) / out.color.size
grads = G.render_backward(m, poses[1], cam, out, dc, np.zeros(out.depth.shape))
m.apply_gradients(grads)
ctx.synchronize()
print("sanitize target done", len(m))
