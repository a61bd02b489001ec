"""Diagnostic (not a test): host enqueue time vs device time per profiling scope of the train
step (bench workload)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2411_02703_b200 import gsmap as G  # noqa: E402

scene, train, _ = bench.build_fixture(1_000_000)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = G.Context(0, s.cuda_stream)
fx, fy, cx, cy, W, H = scene.camera
cam = G.Camera(fx, fy, cx, cy, W, H)
poses = [G.Pose(*p) for p in scene.poses]
gt_map = G.GaussianMap(ctx, scene.gaussians)
fr = G.RenderOutput(ctx)
kfs = []
for f in range(8):
    G.render(gt_map, poses[f], cam, fr)
    kfs.append(G.Keyframe(poses[f], fr.color.copy(), scene.sparse_depth(f), 3, 2, ctx=ctx))
del gt_map
m = G.GaussianMap(ctx, train)
cfg = G.TrainConfig.make(0.2, 0.5, 2, 1)
L = G.lib()
for st in range(6):
    G.train_keyframe_step(m, kfs[(st // 3) % 8], cfg, cam)
ctx.profile(True)
for st in range(24):
    kf = kfs[(st // 3) % 8]
    if kf.consumed_iters >= 3:
        kf.consumed_iters = 0
    G.train_keyframe_step(m, kf, cfg, cam)
dev = ctx.profile_read()
names = C.create_string_buffer(4096); ms = np.zeros(64); n = C.c_int32()
G._check(L.gs_debug_profile_host(C.c_void_p(ctx.h), names, 4096, ms.ctypes.data_as(C.c_void_p), 64, C.byref(n)))
ctx.profile(False)
for i, k in enumerate(names.value.decode().split("\n")[: n.value]):
    print(f"{k:28s} host {ms[i] / 24 * 1e3:8.1f} us/step   device {dev[k][0] / 24 * 1e3:8.1f} us/step")
