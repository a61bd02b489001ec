"""Diagnostic (not a test): is the train step host-launch-bound? Times the bench workload with
the per-step loss read-back (normal) and with it deferred (the host enqueues ahead)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2411_02703_b200 import gsmap as G  # noqa: E402

scene, train, _ = bench.build_fixture(1_000_000)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = G.Context(0, stream.cuda_stream)
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


def run(steps, defer):
    L.gs_debug_defer_step_sync(C.c_void_p(ctx.h), int(defer))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    t0.record(stream)
    for s in range(steps):
        kf = kfs[(s // 3) % 8]
        if kf.consumed_iters >= 3:
            kf.consumed_iters = 0
        G.train_keyframe_step(m, kf, cfg, cam)
    h1 = time.perf_counter()
    t1.record(stream)
    torch.cuda.synchronize()
    L.gs_debug_defer_step_sync(C.c_void_p(ctx.h), 0)
    return t0.elapsed_time(t1) / steps, (h1 - h0) * 1e3 / steps


for defer in (False, True, False, True):
    run(6, defer)
    gpu, host = run(48, defer)
    print(f"defer={defer}: {gpu:.3f} ms/step on the device clock, host enqueue {host:.3f} ms/step", flush=True)

# sanity: do deferred steps do the same work? same 6 steps from the same state, both modes
import numpy as np  # noqa: E402
state = m.gaussians, m.adam_state(), m.global_step
outs = []
for defer in (False, True):
    m.gaussians = state[0]; m.set_adam_state(*state[1]); m.global_step = state[2]
    for kf in kfs:
        kf.consumed_iters = 0
    L.gs_debug_defer_step_sync(C.c_void_p(ctx.h), int(defer))
    for s in range(6):
        G.train_keyframe_step(m, kfs[(s // 3) % 8], cfg, cam)
    L.gs_debug_defer_step_sync(C.c_void_p(ctx.h), 0)
    torch.cuda.synchronize()
    outs.append((m.gaussians["p"].copy(), m.adam_state()[2].copy()))
print("max |dp|", np.abs(outs[0][0] - outs[1][0]).max(), "steps", outs[0][1].max(), outs[1][1].max())
