"""Keyframe-batch training sharded over ranks.

The reference trains one view per step (train_keyframe_step, mapper.cpp:214-238) and has no
batching. The batch step here is defined on the reference's own primitives:

  1. every rank renders its share of the views and sums their RenderGradients into one
     gradient plane buffer (GaussianGrad::add, gaussian.hpp:51-57, done on the device by
     gs_train_accumulate);
  2. one collective sums the buffers over ranks: only the S_p = 11 + 3(d+1)^2 planes the map's
     highest SH degree d makes active (the others are zero on every rank and Adam leaves their
     parameters untouched), i.e. 56 MB instead of 236 MB per step at 1M Gaussians and d = 0;
  3. every rank applies the same Adam step to its replica (apply_gradients,
     gaussian_map.cpp:37-54), so the replicas stay bit-identical.

The gradient buffer is a torch tensor laid out [59][cap] (the library's plane layout,
include/gsmap_b200.h gs_grads_create_external), so the collective is one NCCL all-reduce on
a contiguous prefix, on torch's current stream (the library shares it through the context).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

N_PARAMS = 59


def active_planes(max_degree: int) -> int:
    """Trainable scalars per Gaussian at SH degree d (gaussian.hpp:16-26): 14 at d=0, 59 at d=3."""
    if not 0 <= max_degree <= 3:
        raise ValueError("active_planes: degree must be in [0, 3]")
    return 11 + 3 * (max_degree + 1) ** 2


def rank_views(n_views: int, rank: int, world: int) -> range:
    """The contiguous share of an n_views batch that `rank` renders (views must divide evenly,
    so every rank does the same work and the step time is not set by a straggler)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank_views: bad rank/world")
    if n_views % world:
        raise ValueError(f"rank_views: {n_views} views do not shard over {world} ranks")
    per = n_views // world
    return range(rank * per, (rank + 1) * per)


def reduce_gradient_planes(buf: torch.Tensor, n_planes: int, cap: int, group=None, device_sync=None) -> None:
    """Sum the first n_planes planes of a flat [59][cap] gradient buffer over the ranks, in place:
    NCCL on the device buffer; with a host backend (gloo: one GPU shared by several ranks in
    tests, or CPU-only ranks) the planes go through host memory."""
    if buf.numel() < N_PARAMS * cap or not 0 < n_planes <= N_PARAMS:
        raise ValueError("reduce_gradient_planes: buffer/plane count mismatch")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        part = buf[: n_planes * cap]
        if part.is_cuda and dist.get_backend(group) != "nccl":
            if device_sync is not None:
                device_sync()  # the gradients were written on the library's stream
            host = part.cpu()
            dist.all_reduce(host, group=group)
            part.copy_(host)
            torch.cuda.current_stream(part.device).synchronize()  # before Adam reads it
        else:
            dist.all_reduce(part, group=group)


class BatchTrainer:
    """One keyframe batch per step(): local views -> gradient all-reduce -> one Adam step."""

    def __init__(self, m, ctx, device: torch.device, slack: int = 1024, group=None):
        from . import gsmap as G
        self.G, self.m, self.ctx, self.device, self.slack, self.group = G, m, ctx, device, slack, group
        self.frame = G.RenderOutput(ctx)
        self.cap = 0
        self._alloc()

    def _alloc(self):
        self.cap = len(self.m) + self.slack
        self.buf = torch.zeros(N_PARAMS * self.cap, dtype=torch.float32, device=self.device)
        self.grads = self.G.RenderGradients(self.ctx, external_ptr=self.buf.data_ptr(), capacity=self.cap)

    def step(self, keyframes, views, cfg, cam, lr=None, after_accumulate=None) -> int:
        """Accumulate `views` (indices into keyframes, already at their scheduled level), reduce,
        apply Adam; returns the number of local views rendered. `after_accumulate()` runs once the
        views' work is enqueued, before the collective (e.g. the next batch's input uploads on
        the copy stream, overlapping this batch's compute)."""
        if len(self.m) > self.cap:  # the map grew since the buffer was sized
            self._alloc()
        self.grads.zero(self.m)
        for k in views:
            self.G.train_accumulate(self.m, keyframes[k], cfg, cam, self.grads, self.frame, sync=False)
        if after_accumulate is not None:
            after_accumulate()
        reduce_gradient_planes(self.buf, active_planes(self.m.max_active_degree()), self.cap, self.group,
                               device_sync=self.ctx.synchronize)
        self.m.apply_gradients(self.grads, lr if lr is not None else cfg.lr)
        return len(views)
