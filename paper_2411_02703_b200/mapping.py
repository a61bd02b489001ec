"""The reference's single-thread mapping loop around the hot path, driving the device map.

This mirrors PipelineState's optimizer role (pipeline.cpp:130-180, single_thread mode
:196-203). It is not a pipeline: keyframe admission, the voxel store, sequence IO and threads
stay out of scope. Each keyframe arrives with its pose, colour image and LiDAR
cloud (the reference drains the voxel store instead: `kf->points`, pipeline.cpp:116):

  integrate_keyframe (pipeline.cpp:148-160), one device call (gs_integrate_keyframe):
      filter_points_by_visibility -> init_gaussians_from_points, project_sparse_depth +
      build_keyframe_pyramid; then one train_keyframe_step + housekeeping
  optimize_once (pipeline.cpp:163-173): a uniformly sampled keyframe with budget left
      (KeyframeQueue::sample_for_optimization, keyframe.cpp:122-138) -> train step + housekeeping
  housekeeping (pipeline.cpp:133-145): maybe_upgrade_sh; prune every prune_interval steps

Every call runs on the device; the loop itself is host bookkeeping.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import gsmap as G


@dataclass
class MappingConfig:
    """The PipelineConfig / KeyframeConfig / TrainConfig fields the loop reads (defaults:
    keyframe.hpp:41-43, config.hpp:27, mapper.hpp:17-24)."""
    iter_budget: int = 60
    tau_alpha: float = 0.5
    prune_interval: int = 50
    prune_threshold: float = 0.005
    sh_interval: int = 300
    seed: int = 1
    train: G.TrainConfig = field(default_factory=G.TrainConfig.make)


class _Entry:
    __slots__ = ("kf", "remaining", "index")

    def __init__(self, kf, remaining, index):
        self.kf, self.remaining, self.index = kf, remaining, index


class MappingLoop:
    def __init__(self, m: G.GaussianMap, cam: G.Camera, cfg: MappingConfig | None = None, timed: bool = False):
        self.m, self.cam, self.cfg = m, cam, cfg or MappingConfig()
        self.active: list[_Entry] = []
        self.rng = np.random.default_rng(self.cfg.seed)
        self.reports: list[tuple[int, dict]] = []  # (keyframe index, StepReport)
        self.timed = timed
        self.times: dict[str, float] = {}
        self.calls: dict[str, int] = {}
        self.added: list[int] = []
        self.pruned = 0
        self.n_keyframes = 0
        self._pending: _Entry | None = None  # the next sampled step (drawn one ahead)

    def _clock(self, name, fn, *a):
        # host wall time per call, without device synchronisation (a sync here would also wait
        # for the next step's speculative render and leave the device idle through the host's
        # bookkeeping): a train step returns after its own loss read-back, the housekeeping
        # calls after enqueuing their work
        if not self.timed:
            return fn(*a)
        t = time.perf_counter()
        r = fn(*a)
        self.times[name] = self.times.get(name, 0.0) + time.perf_counter() - t
        self.calls[name] = self.calls.get(name, 0) + 1
        return r

    def _level_after(self, e: _Entry, extra: int) -> int:
        """schedule_level (mapper.cpp:221-224) of e's keyframe after `extra` more steps on it."""
        t = self.cfg.train
        n = t.pyramid_levels
        ipl = t.iters_per_level if t.iters_per_level > 0 else max(1, self.cfg.iter_budget // (n + 1))
        return n - min(n, (e.kf.consumed_iters + extra) // ipl)

    def _step(self, e: _Entry, nxt: _Entry | None = None):
        # naming the next step lets its render overlap this step's read-back (bitwise-equal results)
        hint = (nxt.kf, self._level_after(nxt, 1 if nxt is e else 0)) if nxt is not None else None
        rep = self._clock("train_step", G.train_keyframe_step, self.m, e.kf, self.cfg.train, self.cam, None, hint)
        if rep is not None:
            self.reports.append((e.index, rep))
            self.housekeeping()
        return rep

    def housekeeping(self):
        self._clock("maybe_upgrade_sh", self.m.maybe_upgrade_sh, self.cfg.sh_interval)
        step = self._clock("global_step", lambda: self.m.global_step)
        if self.cfg.prune_interval > 0 and step > 0 and step % self.cfg.prune_interval == 0:
            self.pruned += self._clock("prune", self.m.prune, self.cfg.prune_threshold)

    def integrate_keyframe(self, pose: G.Pose, color: np.ndarray, cloud6: np.ndarray) -> G.Keyframe:
        cfg = self.cfg
        # filter -> init, sparse depth and pyramid in one device call (the cloud crosses once)
        kf, added = self._clock("integrate_keyframe", self.m.integrate_keyframe, pose, self.cam, color, cloud6,
                                cfg.tau_alpha, cfg.iter_budget, cfg.train.pyramid_levels)
        self.added.append(added)
        e = _Entry(kf, cfg.iter_budget, self.n_keyframes)
        self.n_keyframes += 1
        if e.remaining > 0:
            e.remaining -= 1
            self._step(e)
        if e.remaining > 0:
            self.active.append(e)
        return kf

    def _draw(self) -> _Entry | None:
        """KeyframeQueue::sample_for_optimization (keyframe.cpp:122-138): a uniform pick among the
        keyframes with budget left; its budget is taken and a spent keyframe retires."""
        eligible = [i for i, e in enumerate(self.active) if e.remaining > 0]
        if not eligible:
            return None
        i = eligible[int(self.rng.integers(len(eligible)))]
        e = self.active[i]
        e.remaining -= 1
        if e.remaining == 0:
            del self.active[i]
        return e

    def optimize_once(self) -> bool:
        # the sampler runs one step ahead (same draws, same eligible sets: nothing between two
        # steps changes eligibility), so each step can name its successor
        e = self._pending if self._pending is not None else self._draw()
        if e is None:
            return False
        self._pending = self._draw()
        self._step(e, self._pending)
        if e.remaining == 0 and e is not self._pending:  # retired (keyframe.cpp:133-136)
            self._clock("retire_keyframe", e.kf.close)
        return True

    def run(self, frames) -> int:
        """frames: iterable of (pose, colour HWC, cloud [n][6]); integrates every frame, then
        optimizes until every budget is spent. Returns the number of train steps."""
        n0 = len(self.reports)
        for pose, color, cloud in frames:
            self.integrate_keyframe(pose, color, cloud)
        while self.optimize_once():
            pass
        return len(self.reports) - n0
