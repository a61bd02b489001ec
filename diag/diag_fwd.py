"""Diagnostic (not a test): per-level blend kernel times for each pixels-per-thread variant and
forward slow-path counts as training proceeds."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2411_02703_b200 import gsmap as G  # noqa: E402

scene, train, _ = bench.build_fixture(1_000_000)
ctx = G.Context(0)
fx, fy, cx, cy, W, H = scene.camera
cam = G.Camera(fx, fy, cx, cy, W, H)
poses = [G.Pose(*p) for p in scene.poses]
gt_map = G.GaussianMap(ctx, scene.gaussians)
fr = G.RenderOutput(ctx)
kfs = []
for f in range(2):
    G.render(gt_map, poses[f], cam, fr)
    kfs.append(G.Keyframe(poses[f], fr.color.copy(), scene.sparse_depth(f), 3, 2, ctx=ctx))
del gt_map
m = G.GaussianMap(ctx, train)
cfg = G.TrainConfig.make(0.2, 0.5, 2, 1)
cnt = np.zeros(2, np.int64)
L = G.lib()
if os.environ.get("DIAG_SEGFWD"):
    L.gs_debug_set_seg_forward(int(os.environ["DIAG_SEGFWD"]))
if os.environ.get("DIAG_SEG"):
    L.gs_debug_set_blend_segments(int(os.environ["DIAG_SEG"]))
if os.environ.get("DIAG_DF"):
    L.gs_debug_set_blend_df_list(int(os.environ["DIAG_DF"]))
PPTS = tuple(int(x) for x in os.environ.get("DIAG_PPTS", "1,2,4,8").split(","))
for stage in range(int(os.environ.get("DIAG_STAGES", "3"))):
    for lvl in (2, 1, 0):
        line = []
        for ppt in PPTS:
            L.gs_debug_set_blend_ppt(ppt, ppt)
            kf = kfs[0]
            kf.consumed_iters = 2 - lvl
            mstate = m.gaussians, m.adam_state(), m.global_step
            ctx.profile(True)
            L.gs_debug_counters(C.c_void_p(ctx.h), cnt.ctypes.data_as(C.c_void_p), 1)
            G.train_keyframe_step(m, kf, cfg, cam)
            prof = {}
            for key, (ms_, n_) in ctx.profile_read().items():  # keys "name@L<l>"
                a = prof.setdefault(key.partition("@")[0], [0.0, 0])
                a[0] += ms_; a[1] += n_
            L.gs_debug_counters(C.c_void_p(ctx.h), cnt.ctypes.data_as(C.c_void_p), 1)
            ctx.profile(False)
            m.gaussians = mstate[0]
            m.set_adam_state(*mstate[1])
            m.global_step = mstate[2]
            line.append(f"ppt{ppt}: fwd {prof['blend_fwd'][0]:.3f} bwd {prof['blend_bwd'][0]:.3f}")
        L.gs_debug_set_blend_ppt(0, 0)
        G.render(m, poses[0], G.camera_scaled(cam, lvl), fr)
        st = fr.stats()
        print(f"stage {stage} L{lvl} [{st.n_contrib/1e6:.0f}M contribs, near {cnt[0]} replay {cnt[1]}]: " + " | ".join(line),
              flush=True)
    for s in range(24):  # train between stages
        kf = kfs[1]
        if kf.consumed_iters >= 3:
            kf.consumed_iters = 0
        G.train_keyframe_step(m, kf, cfg, cam)
