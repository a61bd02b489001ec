#!/usr/bin/env python
"""Benchmark of the LVI-GS mapping hot path on B200 (BASELINE.json metric).

Metric: training iterations/s (render -> L1+SSIM+depth loss -> backward -> Adam, one keyframe
view per iteration at its scheduled pyramid level) and Mpix/s, 1M Gaussians at 1280x1024,
3-level pyramid (levels 2,1,0 = 320x256 / 640x512 / 1280x1024), lambda=0.2, lambda_d=0.5.

  python bench.py [--steps K] [--warmup W] [--impl ours|reference] [--sh-degree 0|3]
  torchrun --nproc-per-node N bench.py --gpus N      (C4: 8-view batch sharded over N GPUs,
                                                      NCCL all-reduce of the gradient SoA)
  python bench.py --workload c5                       (C5: the mapping loop growing a map from
                                                      8 LiDAR keyframes at 1920x1080; §8f rows)

Workload: synthetic scene = proj/src/io/synthetic.cpp restated (fixtures/),
focal 0.8125*W, extent 18, line trajectory, 8 frames, seed 1, LiDAR noise 0.06 m; the
training map is the colourised-LiDAR initialisation (all 1M GT centres displaced along the
frame-0 beam, 3-NN isotropic scale, opacity 0.1, SH degree 0). GT colour = the GT map
rendered at level 0; LiDAR depth = project_sparse_depth of each frame's cloud. Eight
keyframes, each consumes its pyramid coarse-to-fine (iters_per_level = 1) and is then
recycled, so every 3 consecutive iterations cover levels 2, 1, 0 once (K multiple of 3).
Inputs (1M-Gaussian params + Adam state ~ 240 MB at d=0) exceed the 126 MB L2: no flush.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training iters/sec (fwd+bwd+Adam) and Mpix/s at 1M Gaussians 1280×1024, 1/2/4/8 B200"
N_GAUSS, W0, H0, N_FRAMES, LEVELS = 1_000_000, 1280, 1024, 8, 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=240)
    ap.add_argument("--warmup", type=int, default=24)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sh-degree", type=int, default=0)
    ap.add_argument("--n-gaussians", type=int, default=N_GAUSS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no baselines)")
    ap.add_argument("--batch", action="store_true", help="C4 batch path even at world size 1 (testing)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c5"],
                    help="c5: the single-thread mapping loop (integrate -> train -> housekeeping) at 1920x1080")
    ap.add_argument("--c5-gaussians", type=int, default=2_000_000, help="C5 GT scene size")
    ap.add_argument("--c5-budget", type=int, default=60, help="C5 iter_budget per keyframe (keyframe.hpp:43)")
    ap.add_argument("--c5-phases", action="store_true", help="C5: per-phase event table of the integration calls")
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload
def build_fixture(n_gauss):
    from fixtures import pyfixture as F
    t = time.time()
    scene = F.Scene(n_gaussians=n_gauss, width=W0, height=H0, n_frames=N_FRAMES, seed=1)
    train = scene.training_map(seed=2, noise=0.06)
    return scene, train, time.time() - t


def level_shapes():
    out, h, w = [], H0, W0
    for _ in range(LEVELS + 1):
        out.append((h, w)); h, w = (h + 1) // 2, (w + 1) // 2
    return out


def schedule(step):
    """(keyframe index, level) of iteration `step` (3 iterations per keyframe, coarse first)."""
    return (step // 3) % N_FRAMES, LEVELS - (step % 3)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~2 ms on a background thread while
    the timed region runs (nvidia-smi's own start-up takes longer than a 20-step region). One
    sample is taken on entry and one on exit, so even the shortest region has readings."""
    NAMES = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
             ("hw_power_brake_slowdown", 0x80), ("sw_power_cap", 0x4))

    def __init__(self, device_index=0, period=0.002):
        self.dev = device_index
        self.period = float(os.environ.get("GS_CLOCK_PERIOD", period))
        self.h = None
        self.samples = []
        self.mx = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the NVML device of this CUDA device (CUDA_VISIBLE_DEVICES may renumber)
            import torch
            p = torch.cuda.get_device_properties(self.dev)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def _sample(self):
        import pynvml
        try:
            sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((sm, r))
        except Exception:
            pass

    def _run(self):
        while not self.stop.wait(self.period):
            self._sample()

    def __enter__(self):
        import threading
        try:
            import pynvml
            self.h = self._handle()
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None
            return self
        self.stop = threading.Event()
        self._sample()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        if self.h is None:
            return
        self._sample()
        self.stop.set()
        self.th.join()

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.NAMES if r & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.mx,
                "reasons": reasons, "samples": len(sm), "source": "NVML, ~2 ms period during the timed region"}


# ----------------------------------------------------------------------------- roofline model
def algorithmic(stats_by_level, n, sp):
    """Algorithmic bytes / flops / ex2 per launch of each kernel family, averaged over the
    three levels. stats_by_level[l] = (n_vis, pairs, pixels, contribs, tiles)."""
    out = {}
    for l, (nv, K, P, SC, T) in stats_by_level.items():
        per = {
            "preprocess_fwd": (4 * sp * n + 64 * nv, 300 * n, 0),
            "depth_sort_pack_scan": (24 * nv + 136 * nv, 0, 0),
            "tile_keys_sort_ranges": (36 * K, 0, 0),
            "blend_fwd": (64 * K + 28 * P, 22 * SC, SC),
            "loss_l1_ssim_depth": (52 * P, 650 * P, 0),
            "blend_bwd": (64 * K + 24 * P + 40 * K, 70 * SC, SC),
            "preprocess_bwd": (40 * K + 40 * nv + 8 * sp * nv, 600 * nv, 0),
            "adam": ((28 * sp + 8) * n, 10 * sp * n, 0),
        }
        for k, v in per.items():
            acc = out.setdefault(k, [0.0, 0.0, 0.0])
            for i in range(3):
                acc[i] += v[i] / len(stats_by_level)
    return out


# ----------------------------------------------------------------------------- our arm
def local_device() -> int:
    """This rank's GPU: LOCAL_RANK (modulo the visible devices)."""
    import torch
    return int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())


def coll_device(dev: int) -> str:
    """Where a collective's tensor lives: the GPU under NCCL, the host under gloo."""
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else f"cuda:{dev}"


def run_ours(args, rank, world):
    import torch
    from paper_2411_02703_b200 import gsmap as G

    dev = local_device()
    torch.cuda.set_device(dev)
    # one explicit stream for everything: the C-ABI context launches on it and the timing
    # events are recorded on it (torch's default stream handle is 0, for which the context
    # would create a stream of its own)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = G.Context(dev, stream.cuda_stream)
    scene, train, t_fix = build_fixture(args.n_gaussians)
    fx, fy, cx, cy, W, H = scene.camera
    cam = G.Camera(fx, fy, cx, cy, W, H)
    poses = [G.Pose(*p) for p in scene.poses]

    # GT colour = the GT map rendered at level 0 by the same renderer (setup, untimed)
    gt_map = G.GaussianMap(ctx, scene.gaussians)
    gt_frame = G.RenderOutput(ctx)
    kfs, host_levels = [], []
    for f in range(N_FRAMES):
        G.render(gt_map, poses[f], cam, gt_frame)
        color = gt_frame.color.copy()
        sparse = scene.sparse_depth(f)
        kfs.append(G.Keyframe(poses[f], color, sparse, initial_iters=3, levels=LEVELS, ctx=ctx))
        lv = []
        for l in range(LEVELS + 1):  # pinned fp64 HWC copies of the pyramid for the e2e leg
            c, d = kfs[-1].level(l)
            pc = torch.empty(c.shape, dtype=torch.float64, pin_memory=True).numpy(); pc[...] = c
            pd = torch.empty(d.shape, dtype=torch.float64, pin_memory=True).numpy(); pd[...] = d
            lv.append((pc, pd))
        host_levels.append(lv)
    del gt_map, gt_frame
    m = G.GaussianMap(ctx, train)
    if args.sh_degree:
        m.raise_sh_degree(args.sh_degree)
    cfg = G.TrainConfig.make(0.2, 0.5, LEVELS, 1)
    lvl_cams = [G.camera_scaled(cam, l) for l in range(LEVELS + 1)]
    shapes = level_shapes()

    batch = world > 1 or args.batch
    views_per_rank = 1
    if batch:  # C4: 8-view batch sharded over ranks, NCCL all-reduce of the active gradient planes
        from paper_2411_02703_b200.batch import BatchTrainer, rank_views
        trainer = BatchTrainer(m, ctx, torch.device(f"cuda:{dev}"))
        my_views = rank_views(N_FRAMES, rank, world)
        views_per_rank = len(my_views)

    def step(s, e2e=False, prefetch=None, hint=None):
        if not batch:
            k, lvl = schedule(s)
            kf = kfs[k]
            if kf.consumed_iters >= 3:
                kf.consumed_iters = 0
            if e2e:
                kf.upload_level(lvl, *host_levels[k][lvl])
            pf = None
            if prefetch is not None:  # step `prefetch`'s input, uploaded behind this step's work
                nk, nl = schedule(prefetch)
                pf = (kfs[nk], nl, *host_levels[nk][nl])
            elif hint is not None:  # the next step (its render is enqueued during this read-back)
                nk, nl = schedule(hint)
                pf = (kfs[nk], nl)
            rep = G.train_keyframe_step(m, kf, cfg, cam, prefetch=pf)
            assert rep is not None and rep["level"] == lvl
            return 1, shapes[lvl][0] * shapes[lvl][1]
        lvl = LEVELS - (s % 3)
        px = 0
        for k in my_views:
            kf = kfs[k]
            kf.consumed_iters = (LEVELS - lvl)
            if e2e:
                kf.upload_level(lvl, *host_levels[k][lvl])
            px += shapes[lvl][0] * shapes[lvl][1]
        after = None
        if prefetch is not None:  # batch `prefetch`'s inputs, uploaded behind this batch's views
            nl = LEVELS - (prefetch % 3)
            after = lambda: [kfs[k].upload_level(nl, *host_levels[k][nl]) for k in my_views]
        trainer.step(kfs, my_views, cfg, cam, after_accumulate=after)
        torch.cuda.current_stream().synchronize()
        return views_per_rank, px

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    for s in range(args.warmup):  # (no hint past the warm-up: the timed region renders all its steps)
        step(s, hint=s + 1 if s + 1 < args.warmup else None)
    barrier()
    # GS_PROFILE_RANGE=1: restrict an `ncu --profile-from-start off` capture to the timed steps
    prof_range = os.environ.get("GS_PROFILE_RANGE") == "1"
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    launches0 = ctx.launches
    cap0 = ctx.capacity_stats()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.freeze()  # setup objects leave the collector's generations: no multi-ms gen-2 pauses in the timed loop
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(dev) as clk:
        e0.record(stream)
        views = pix = 0
        for s in range(args.steps):
            v, p = step(args.warmup + s, hint=args.warmup + s + 1 if s + 1 < args.steps else None)
            views += v; pix += p
            step_ev[s].record(stream)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    # per-level step times (per-level rates)
    lvl_ms = {}
    intervals = []
    for s in range(args.steps):
        d = step_ev[s - 1].elapsed_time(step_ev[s]) if s else e0.elapsed_time(step_ev[0])
        intervals.append(round(d, 4))
        lvl = (LEVELS - ((args.warmup + s) % 3)) if batch else schedule(args.warmup + s)[1]
        lvl_ms.setdefault(lvl, []).append(d)
    per_level = {f"L{l}": {"ms_per_step": round(float(np.mean(v)), 4), "steps": len(v),
                           "mpix_per_s": round(shapes[l][0] * shapes[l][1] * views_per_rank * world / (np.mean(v) / 1e3) / 1e6, 2)}
                 for l, v in sorted(lvl_ms.items())}
    launches = ctx.launches - launches0
    cap1 = ctx.capacity_stats()
    capacity = {k: cap1[k] - cap0[k] for k in cap1}
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    ms_max = ms
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=coll_device(dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    total_views = views * world
    total_pix = pix * world
    value = total_views / (ms_max / 1e3)

    result = {"metric": METRIC, "value": round(value, 3), "unit": "iters/s", "n_gpus": world,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
              "higher_is_better": True, "scaling": "strong" if batch else "weak", "vs_baseline": None,
              "iteration": ("one keyframe view's render + loss + backward; value counts views of the 8-view batch "
                            "(one all-reduce + Adam per batch)" if batch else
                            "one keyframe view: render + loss + backward + Adam at its scheduled level"),
              "dtype": "f32 (fp64 geometry, fp64 transmittance)",
              "data": "synthetic (reference synthetic.cpp scene, colourised-LiDAR-initialised map)",
              "mpix_per_s": round(total_pix / (ms_max / 1e3) / 1e6, 3), "per_level": per_level,
              "per_level_note": "intervals between consecutive step reports; each step names the next, whose render "
                                "is enqueued during this step's read-back and so falls in this step's interval",
              "config": {"workload": ("C4: 8-keyframe batch sharded over ranks, NCCL all-reduce" if batch else
                                      "C3: 1M Gaussians 1280x1024, 3-level pyramid (L2,L1,L0 in turn), L1+SSIM+depth loss"),
                         "n_gaussians": len(m), "width": W0, "height": H0, "pyramid_levels": LEVELS + 1,
                         "sh_degree": args.sh_degree, "lambda": 0.2, "lambda_d": 0.5, "keyframes": N_FRAMES,
                         "l2": "inputs larger than L2 (params+Adam+grads > 126 MB)",
                         "parallelism": f"dp{world}" if batch else "single-view"},
              "gpu_launches": launches, "clocks": clk.summary(), "fixture_s": round(t_fix, 2),
              "timed_region_capacity_events": capacity,
              # device time between consecutive step reports (per-step view of the timed region)
              "step_intervals_ms": intervals if args.steps <= 300 else None}

    # ---------------- per-kernel profile pass (separate from the headline timing)
    ctx.profile(True)
    for s in range(args.steps):
        step(args.warmup + args.steps + s)
    prof_lv = ctx.profile_read()
    ctx.profile(False)
    # scopes of a train step carry its level ("name@L<l>"): per-level table + the aggregate
    prof, per_level_kernels = {}, {}
    for key, (tot_ms, cnt) in prof_lv.items():
        name, _, lv = key.partition("@")
        acc = prof.setdefault(name, [0.0, 0])
        acc[0] += tot_ms; acc[1] += cnt
        if lv:
            per_level_kernels.setdefault(lv, {})[name] = round(tot_ms / max(cnt, 1), 4)
    # per-level workload counters for the algorithmic model
    stats = {}
    fr = G.RenderOutput(ctx)
    for l in range(LEVELS + 1):
        G.render(m, poses[0], lvl_cams[l], fr)
        st = fr.stats()
        stats[l] = (st.n_visible, st.n_pairs, st.width * st.height, st.n_contrib, st.tiles_x * st.tiles_y)
    sp = 11 + 3 * (args.sh_degree + 1) ** 2
    alg = algorithmic(stats, len(m), sp)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    import ctypes as C
    fp32 = C.c_double(); ex2 = C.c_double()
    G._check(G.lib().gs_microbench(dev, 0, C.byref(fp32)))
    G._check(G.lib().gs_microbench(dev, 1, C.byref(ex2)))
    kernels = {}
    for k, (tot_ms, cnt) in prof.items():
        avg = tot_ms / max(cnt, 1) * 1e-3
        b, fl, x = alg.get(k, (0, 0, 0))
        kernels[k] = {"share": round(tot_ms / sum(v[0] for v in prof.values()), 4), "avg_ms": round(avg * 1e3, 4),
                      "launches": cnt, "gbs": round(b / avg / 1e9, 1) if b else None,
                      "tflops": round(fl / avg / 1e12, 3) if fl else None}
    dom = max(prof, key=lambda k: prof[k][0])
    avg = prof[dom][0] / prof[dom][1] * 1e-3
    b, fl, x = alg.get(dom, (0, 0, 0))
    t_hbm, t_fp, t_ex = b / (hbm * 1e9), fl / fp32.value, x / ex2.value
    if t_hbm >= max(t_fp, t_ex):
        roof = {"bound": "hbm", "achieved": round(b / avg / 1e9, 1), "peak": hbm, "unit": "GB/s"}
    else:
        roof = {"bound": "fp32" if t_fp >= t_ex else "mufu.ex2",
                "achieved": round((fl / avg if t_fp >= t_ex else x / avg) / 1e12, 3),
                "peak": round((fp32.value if t_fp >= t_ex else ex2.value) / 1e12, 3),
                "unit": "TFLOP/s" if t_fp >= t_ex else "Tex2/s"}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    roof["kernel"] = dom
    # measured DRAM bytes per launch of the same kernel (ncu dram__bytes_read + _write, one
    # capture per pyramid level, averaged like `achieved`), committed under profiles/
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r2_traffic.json")
    if not os.path.exists(tpath):
        tpath = os.path.join(ROOT, "profiles", "r1_traffic.json")
    if os.path.exists(tpath):
        tk = json.load(open(tpath)).get("kernels", {}).get(dom)
        traffic = tk.get("dram_bytes_per_launch") if tk else None
    roof["traffic"] = traffic
    roof["algorithmic_bytes_per_launch"] = int(b)
    # the same kernel seen against HBM (it is not bandwidth-bound: this is the minor roof)
    roof["hbm_view"] = {"achieved": round(b / avg / 1e9, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(b / avg / 1e9 / hbm, 4)}
    roof["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs" if roof["bound"] == "hbm"
                           else "gs_microbench on this device (FP32 FMA / MUFU.EX2 issue rate)")
    roof["model"] = "SURVEY §8d algorithmic bytes/flops per launch, averaged over the 3 pyramid levels"
    result["roofline"] = roof
    # SURVEY §8d step-level figure: sum over the step's kernels of t_roof = max(bytes / HBM,
    # flop / FP32, ex2 / MUFU) against the measured step time
    t_roof = sum(max(b_ / (hbm * 1e9), f_ / fp32.value, x_ / ex2.value) for b_, f_, x_ in alg.values())
    result["step_roofline"] = {"sum_t_roof_ms": round(t_roof * 1e3, 4), "measured_ms": round(ms_max / args.steps, 4),
                               "frac": round(t_roof * 1e3 / (ms_max / args.steps), 4),
                               "model": "SURVEY §8d: per kernel t_roof = max(B / hbm_gbs, F / FP32 FFMA rate, "
                                        "X / MUFU.EX2 rate), workload counters from the device, averaged over levels"}
    # per-level step time = the level's kernel times from the profile pass (device time of that
    # level's render + loss + backward + Adam); the interval between step reports is kept beside
    # it (each interval also holds the next step's speculative render)
    for lv, ks in per_level_kernels.items():
        if lv in per_level:
            kt = sum(ks.values())
            per_level[lv]["interval_ms"] = per_level[lv]["ms_per_step"]
            per_level[lv]["ms_per_step"] = round(kt, 4)
            h_, w_ = shapes[int(lv[1:])]
            per_level[lv]["mpix_per_s"] = round(h_ * w_ / (kt / 1e3) / 1e6, 2)
    result["per_level_note"] = ("ms_per_step: the level's kernel times (profile pass, CUDA events on the context "
                                "stream); interval_ms: time between consecutive step reports in the timed region, "
                                "which also holds the next step's speculative render")
    result["kernels"] = kernels
    result["per_level_kernel_ms"] = per_level_kernels
    result["workload_counters"] = {f"L{l}": dict(zip(["n_visible", "pairs", "pixels", "contribs", "tiles"], v))
                                   for l, v in stats.items()}

    # ---------------- e2e: same metric through the C-ABI with host buffers each step
    if not args.no_e2e:
        # the e2e leg continues the step sequence (keyframe consumption and level schedule stay
        # consistent whatever the warm-up and step counts)
        eb = args.warmup + 2 * args.steps
        for s in range(3):
            step(eb + s, e2e=True)
        eb += 3
        barrier()
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        t0.synchronize()  # every upload below is issued after t0 has fired
        views = 0
        h2d = 0
        if not batch:
            # double buffering: step s + 1's input upload (copy stream) is issued by step s's
            # train call right behind its enqueued work (gs_train_step_prefetch), so the copies
            # and their API calls overlap compute; every step's copy is inside the timed region
            # (step 0's included) and each train step waits for its own level's upload
            k0, l0 = schedule(eb)
            kfs[k0].upload_level(l0, *host_levels[k0][l0])
        else:
            l0 = LEVELS - eb % 3
            for k in my_views:
                kfs[k].upload_level(l0, *host_levels[k][l0])
        for s in range(args.steps):
            v, _ = step(eb + s, e2e=False, prefetch=eb + s + 1 if s + 1 < args.steps else None)
            views += v
            lvl = LEVELS - ((eb + s) % 3)
            h2d += 32 * shapes[lvl][0] * shapes[lvl][1] * (views_per_rank if batch else 1)
        t1.record(stream)
        barrier()
        e_ms = t0.elapsed_time(t1)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e_ms], device=coll_device(dev))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        result["e2e"] = {"value": round(views * world / (e_ms / 1e3), 3), "unit": "iters/s",
                         "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": 24,
                         "path": "gs_train_step_prefetch: each step enqueues its work, then the next step's input "
                                 "upload (host fp64 HWC pyramid level, pinned; copy stream), then reads its report"}
    return result, (scene, train, kfs, host_levels)


# ----------------------------------------------------------------------------- CPU (oracle) arm
def reference_cpu():
    """The reference's own CPU implementation: oracle/_ref/libgsref.so (the reference sources
    compiled unchanged, built here and shipped with the repo) when present, else the oracle
    restatement. Returns (module with the oracle's wrappers, cpu_baseline kind, description)."""
    from oracle import pyref
    if pyref.available():
        return pyref.load(), "reference", ("the reference itself: /root/reference/proj/src compiled unchanged "
                                           "(-O3 -DNDEBUG, oracle/ref/Makefile) into oracle/_ref/libgsref.so")
    from oracle import pyoracle as O
    return O, "port", "oracle restatement (oracle/, fp64, -O3 -ffp-contract=off)"


def cpu_sample(scene, train, gt_levels, threads=0):
    """The reference's train_keyframe_step (fp64, ThreadPool with every host thread) over one
    coarse-to-fine cycle of keyframe 0 (levels 2, 1, 0): 3 iterations."""
    O, kind, what = reference_cpu()
    fx, fy, cx, cy, W, H = scene.camera
    cam = O.camera(fx, fy, cx, cy, W, H)
    p = scene.poses[0]
    pose = O.Pose(*p)
    om = O.OracleMap(train)
    color0, depth0 = gt_levels
    kf = O.Keyframe(pose, color0, depth0, 3, LEVELS)
    cfg = O.make_cfg(0.2, 0.5, LEVELS, 1)
    pool = O.ThreadPool(threads)
    t = time.time()
    px = 0
    level_s = {}
    for it in range(3):
        t0 = time.time()
        r = O.train_keyframe_step(om, kf, cfg, cam, pool)
        level_s[f"L{r['level']}"] = round(time.time() - t0, 3)
        h, w = level_shapes()[r["level"]]
        px += h * w
    dt = time.time() - t
    # a single-thread run beside the pool -- the first (coarsest-level) iteration of
    # the same keyframe on a fresh copy of the map, ThreadPool(1)
    kf1 = O.Keyframe(pose, color0, depth0, 3, LEVELS)
    om1 = O.OracleMap(train)
    t0 = time.time()
    r1 = O.train_keyframe_step(om1, kf1, cfg, cam, O.ThreadPool(1))
    t1 = time.time() - t0
    lv = f"L{r1['level']}"
    return {"value": round(3 / dt, 5), "unit": "iters/s", "cores": pool.threads, "kind": kind,
            "mpix_per_s": round(px / dt / 1e6, 4),
            "sample": f"{what}, train_keyframe_step: one L2->L1->L0 cycle (3 iterations) of keyframe 0 of the "
                      "same 1M-Gaussian workload",
            "seconds": round(dt, 2), "seconds_per_level": level_s,
            "single_thread": {"level": r1["level"], "seconds": round(t1, 3), "threads": 1,
                              "pool_seconds_same_level": level_s.get(lv),
                              "pool_speedup": round(t1 / level_s[lv], 2) if level_s.get(lv) else None}}


# ----------------------------------------------------------------------------- C5 mapping loop
def run_c5(args):
    """the reference's single-thread mapping loop (pipeline.cpp:130-203)
    over the device map, growing it from 8 LiDAR keyframes at 1920x1080 (GT scene of
    --c5-gaussians). Integrate = filter_points_by_visibility + init_gaussians_from_points +
    project_sparse_depth + pyramid + one step; then sampled steps until every keyframe's
    iter_budget is spent; housekeeping = maybe_upgrade_sh (300) + prune every 50 steps. Then
    evaluate_sequence over the 8 frames and a checkpoint save + load of the final map.
    value = train steps / wall time of the whole loop (integration and housekeeping inside)."""
    import torch
    from fixtures import pyfixture as F
    from paper_2411_02703_b200 import gsmap as G
    from paper_2411_02703_b200.mapping import MappingConfig, MappingLoop
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = G.Context(dev, stream.cuda_stream)
    t = time.time()
    scene = F.Scene(n_gaussians=args.c5_gaussians, width=1920, height=1080, n_frames=N_FRAMES, seed=1)
    clouds = [scene.cloud(f) for f in range(N_FRAMES)]
    fx, fy, cx, cy, W, H = scene.camera
    cam = G.Camera(fx, fy, cx, cy, W, H)
    poses = [G.Pose(*p) for p in scene.poses]
    gt_map = G.GaussianMap(ctx, scene.gaussians)
    fr = G.RenderOutput(ctx)
    colors = []
    for f in range(N_FRAMES):
        G.render(gt_map, poses[f], cam, fr)
        colors.append(np.floor(np.clip(fr.color, 0.0, 1.0) * 255.0 + 0.5) / 255.0)  # stored as 8-bit images
    del gt_map, fr

    def pinned(a):  # the sequence loader's frames staged in pinned host memory (as the C3 e2e leg)
        out = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
        out[...] = a
        return out
    clouds = [pinned(c) for c in clouds]
    colors = [pinned(c) for c in colors]
    t_fix = time.time() - t
    mk = lambda budget: MappingConfig(iter_budget=budget, train=G.TrainConfig.make(0.2, 0.5, LEVELS))
    # warm-up: a short loop on a throw-away map (allocations, CUB temp sizes, first launches)
    MappingLoop(G.GaussianMap(ctx), cam, mk(3)).run(list(zip(poses, colors, clouds))[:3])
    torch.cuda.synchronize()
    m = G.GaussianMap(ctx)
    loop = MappingLoop(m, cam, mk(args.c5_budget), timed=True)
    if args.c5_phases:
        ctx.profile(True)  # per-phase CUDA-event table of the integration calls (train steps included)
    launches0 = ctx.launches
    cap0 = ctx.capacity_stats()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.freeze()  # setup objects leave the collector's generations: no multi-ms gen-2 pauses in the timed loop
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        steps = loop.run(zip(poses, colors, clouds))
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    dev_ms = e0.elapsed_time(e1)
    launches = ctx.launches - launches0
    cap1 = ctx.capacity_stats()
    capacity = {k: cap1[k] - cap0[k] for k in cap1}
    phases = None
    if args.c5_phases:
        phases = {k: {"ms": round(v[0], 2), "calls": v[1]} for k, v in ctx.profile_read().items()}
        ctx.profile(False)
    # evaluate_sequence (gt depth = the projected cloud, as without a gt depth file)
    torch.cuda.synchronize()
    t = time.perf_counter()
    recs = G.evaluate_sequence(m, [(poses[f], colors[f], None, clouds[f]) for f in range(N_FRAMES)], cam)
    torch.cuda.synchronize()
    t_eval = time.perf_counter() - t
    path = os.path.join("/tmp", f"gsmap_c5_{os.getpid()}.gsmap")
    t = time.perf_counter()
    m.save_checkpoint(path)
    t_save = time.perf_counter() - t
    t = time.perf_counter()
    m2 = G.load_checkpoint(path, ctx)
    t_load = time.perf_counter() - t
    ck_bytes = os.path.getsize(path)
    os.remove(path)
    assert len(m2) == len(m)
    del m2
    rows = {k: {"calls": loop.calls[k], "ms_total": round(loop.times[k] * 1e3, 2),
                "ms_per_call": round(loop.times[k] * 1e3 / loop.calls[k], 3)} for k in sorted(loop.times)}
    rows["host_bookkeeping"] = {"ms_total": round((wall - sum(loop.times.values())) * 1e3, 2)}
    psnr = [r["psnr"] for r in recs]
    return {"metric": "C5 mapping loop: train iterations/s including keyframe integration and housekeeping",
            "value": round(steps / wall, 3), "unit": "iters/s", "n_gpus": 1, "steps": steps, "warmup": 1,
            "ms_per_step": round(wall / steps * 1e3, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (fp64 geometry, fp64 transmittance)",
            "data": "synthetic (reference synthetic.cpp scene; the map grows from the frames' LiDAR clouds)",
            "config": {"workload": "C5: map expansion stream, 8 keyframes, 1920x1080, 3-level pyramid",
                       "gt_gaussians": args.c5_gaussians, "iter_budget": args.c5_budget, "tau_alpha": 0.5,
                       "prune_interval": 50, "sh_interval": 300, "cloud_points": [len(c) for c in clouds]},
            "device_ms": round(dev_ms, 2), "wall_ms": round(wall * 1e3, 2), "gpu_launches": launches,
            "capacity_events": capacity,
            "map": {"final_gaussians": len(m), "added_per_keyframe": loop.added, "pruned": loop.pruned,
                    "max_sh_degree": m.max_active_degree()},
            "rows": rows, "rows_note": "host wall time per call (no device synchronisation around the calls: a train "
                                       "step returns after its own loss read-back, the housekeeping calls once enqueued)",
            "integrate_phases": phases,
            "evaluate": {"frames": len(recs), "ms_per_frame": round(t_eval * 1e3 / len(recs), 3),
                         "mean_psnr": round(float(np.mean(psnr)), 4),
                         "mean_ssim": round(float(np.mean([r["ssim"] for r in recs])), 5)},
            "checkpoint": {"bytes": ck_bytes, "save_ms": round(t_save * 1e3, 1), "load_ms": round(t_load * 1e3, 1),
                           "save_gbs": round(ck_bytes / t_save / 1e9, 3), "load_gbs": round(ck_bytes / t_load / 1e9, 3)},
            "clocks": clk.summary(), "fixture_s": round(t_fix, 2)}


def run_reference(args, rank):
    """--impl reference: the reference's own CPU path (oracle/_ref: its sources compiled
    unchanged; the oracle restatement only if that build is missing) on this host's cores."""
    if rank != 0:
        return None
    O, kind, what = reference_cpu()
    scene, train, t_fix = build_fixture(args.n_gaussians)
    fx, fy, cx, cy, W, H = scene.camera
    cam = O.camera(fx, fy, cx, cy, W, H)
    pose = O.Pose(*scene.poses[0])
    pool = O.ThreadPool(0)
    gt = O.render(O.OracleMap(scene.gaussians), pose, cam, threads=pool.threads)
    color = gt.color.copy()
    depth = scene.sparse_depth(0)
    del gt
    om = O.OracleMap(train)
    kf = O.Keyframe(pose, color, depth, 3, LEVELS)
    cfg = O.make_cfg(0.2, 0.5, LEVELS, 1)
    warm = min(args.warmup, 1)
    timed = min(args.steps, 3)
    for _ in range(warm):
        O.train_keyframe_step(om, kf, cfg, cam, pool)
    kf.consumed_iters = 0
    t = time.time()
    px = 0
    for _ in range(timed):
        r = O.train_keyframe_step(om, kf, cfg, cam, pool)
        h, w = level_shapes()[r["level"]]
        px += h * w
    dt = time.time() - t
    v = timed / dt
    sample = (f"{what}: train_keyframe_step (fp64, ThreadPool({pool.threads})), {timed} iterations "
              f"(levels 2,1,0) of keyframe 0 after {warm} warm-up; same fixture as --impl ours")
    return {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "iters/s", "n_gpus": 0,
            "steps": timed, "warmup": warm, "ms_per_step": round(dt / timed * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "mpix_per_s": round(px / dt / 1e6, 4),
            "config": {"workload": "C3: 1M Gaussians 1280x1024, 3-level pyramid, L1+SSIM+depth loss",
                       "n_gaussians": len(train), "width": W0, "height": H0},
            "cpu_baseline": {"kind": kind, "cores": pool.threads, "sample": sample, "value": round(v, 5),
                             "unit": "iters/s"},
            "e2e": {"value": round(v, 5), "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.workload == "c5":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "C5 is measured on the device arm only "
                              "(the oracle's O(n^2) 3-NN init at 566k points per keyframe does not finish)"}))
            return
        print(json.dumps(run_c5(args)), flush=True)
        return
    if args.impl == "reference":
        res = run_reference(args, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1 or args.batch:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(local_device())
        # GS_DIST_BACKEND=gloo: host-side collectives, for a functional run of the multi-rank
        # path with several ranks on one GPU (never a measurement)
        dist.init_process_group(os.environ.get("GS_DIST_BACKEND", "nccl"))
    result, ctxdata = run_ours(args, rank, world)
    if world == 1 and not args.batch and args.sh_degree == 0 and not args.profile_only:
        # d = 0 and d = 3 reported separately (same workload, every SH band active)
        import copy
        a3 = copy.copy(args)
        a3.sh_degree, a3.no_e2e = 3, True
        r3, _ = run_ours(a3, rank, world)
        result["sh_degree_3"] = {k: r3[k] for k in ("value", "ms_per_step", "mpix_per_s", "per_level", "kernels",
                                                    "per_level_kernel_ms")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        scene, train, kfs, host_levels = ctxdata
        c0, d0 = host_levels[0][0]
        result["cpu_baseline"] = cpu_sample(scene, train, (np.array(c0), np.array(d0)))
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1 or args.batch:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
