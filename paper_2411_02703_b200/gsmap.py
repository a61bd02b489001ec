"""Python mirror of the reference's hot-path interface over the B200 C-ABI (include/gsmap_b200.h).

Names, argument meaning and error behaviour follow proj/include/gsmap/{render/rasterizer.hpp,
map/gaussian_map.hpp, map/mapper.hpp}: ``render``, ``render_backward``,
``GaussianMap.apply_gradients``, ``compute_loss``, ``train_keyframe_step``; ``ValueError``
stands in for std::invalid_argument and ``LogicError`` for std::logic_error.

There is no CPU fallback: importing this module on a machine where the in-tree
``libgsmap_b200.so`` is missing raises, and every call runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgsmap_b200.so")
# diagnostics only (diag/build_variant.sh): time an experimental build of the same sources
if os.environ.get("GSMAP_B200_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(_HERE), "diag", "_variants", os.environ["GSMAP_B200_VARIANT"],
                            "libgsmap_b200.so")

GAUSS_DTYPE = np.dtype([("p", "<f8", (59,)), ("degree", "<i4"), ("pad", "<i4")])

GS_OK, GS_EINVAL, GS_ELOGIC, GS_ECUDA, GS_ENCCL, GS_ENOMEM, GS_ERUNTIME = range(7)


class Camera(C.Structure):  # gsmap::CameraModel (core/types.hpp:15-45)
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose(C.Structure):  # gsmap::Pose with q already normalised (core/types.hpp:48-64)
    _fields_ = [("qw", C.c_double), ("qx", C.c_double), ("qy", C.c_double), ("qz", C.c_double),
                ("tx", C.c_double), ("ty", C.c_double), ("tz", C.c_double)]


class LearningRates(C.Structure):  # map/gaussian_map.hpp:34-40
    _fields_ = [("position", C.c_double), ("rotation", C.c_double), ("log_scale", C.c_double),
                ("opacity", C.c_double), ("sh", C.c_double)]

    @classmethod
    def default(cls):
        return cls(1.6e-4, 1e-3, 5e-3, 5e-2, 2.5e-3)


class TrainConfig(C.Structure):  # map/mapper.hpp:17-30 (hot-path fields)
    _fields_ = [("lambda_", C.c_double), ("lambda_d", C.c_double), ("pyramid_levels", C.c_int32),
                ("iters_per_level", C.c_int32), ("lr", LearningRates)]

    @classmethod
    def make(cls, lam=0.2, lam_d=0.5, levels=2, ipl=0, lr=None):
        return cls(lam, lam_d, levels, ipl, lr or LearningRates.default())


class LossResult(C.Structure):
    _fields_ = [("total", C.c_double), ("color_loss", C.c_double), ("depth_loss", C.c_double),
                ("l1", C.c_double), ("ssim", C.c_double), ("psnr", C.c_double)]


class StepReport(C.Structure):
    _fields_ = [("ran", C.c_int32), ("level", C.c_int32), ("loss", C.c_double), ("psnr", C.c_double)]


class FrameStats(C.Structure):
    _fields_ = [("n_visible", C.c_int64), ("n_pairs", C.c_int64), ("n_contrib", C.c_int64),
                ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("width", C.c_int32), ("height", C.c_int32)]


class LogicError(RuntimeError):
    """std::logic_error"""


class CudaError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"gsmap_b200: CUDA extension {LIB_PATH} is not built "
                              "(run __graft_entry__.build()); there is no CPU fallback")
        _lib = C.CDLL(LIB_PATH)
        _lib.gs_last_error.restype = C.c_char_p
        _lib.gs_version.restype = C.c_char_p
    return _lib


def _check(st: int):
    if st == GS_OK:
        return
    msg = lib().gs_last_error().decode()
    if st == GS_EINVAL:
        raise ValueError(msg)
    if st == GS_ELOGIC:
        raise LogicError(msg)
    if st == GS_ENOMEM:
        raise MemoryError(msg)
    if st == GS_ERUNTIME:
        raise RuntimeError(msg)
    raise CudaError(msg)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _vp(h):
    return C.c_void_p(h)


def exported_symbols():
    """Names the header declares; used by the CPU symbol test."""
    return [n for n in dir(lib()) if n.startswith("gs_")]


# --------------------------------------------------------------------------- context
class Context:
    """One device + one CUDA stream (defaults to the library's own non-blocking stream)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        _check(lib().gs_context_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h.value
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().gs_context_destroy(_vp(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().gs_context_synchronize(_vp(self.h)))

    def set_stream(self, stream: int):
        _check(lib().gs_context_set_stream(_vp(self.h), C.c_void_p(stream)))

    @property
    def launches(self) -> int:
        n = C.c_int64()
        _check(lib().gs_context_launch_count(_vp(self.h), C.byref(n)))
        return n.value

    def capacity_stats(self) -> dict:
        """Pair-capacity policy counters (gs_debug_capacity): growths after a read-back, train
        steps re-run after an overflow, renders that read their pair count before binning."""
        out = np.zeros(3, np.int64)
        _check(lib().gs_debug_capacity(_vp(self.h), _p(out)))
        return {"cap_growths": int(out[0]), "overflow_reruns": int(out[1]), "count_syncs": int(out[2])}

    def profile(self, enable: bool = True):
        """Per-kernel CUDA-event timing on the context stream (resets the table)."""
        _check(lib().gs_context_profile(_vp(self.h), int(enable)))

    def profile_read(self) -> dict:
        names = C.create_string_buffer(4096)
        ms = np.zeros(64); cnt = np.zeros(64, np.int64); n = C.c_int32()
        _check(lib().gs_context_profile_read(_vp(self.h), names, 4096, _p(ms), _p(cnt), 64, C.byref(n)))
        keys = names.value.decode().split("\n")[: n.value]
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def camera_scaled(cam: Camera, level: int) -> Camera:
    out = Camera()
    _check(lib().gs_camera_scaled(C.byref(cam), level, C.byref(out)))
    return out


def validate_camera(cam: Camera):
    _check(lib().gs_camera_validate(C.byref(cam)))


# --------------------------------------------------------------------------- GaussianMap
class GaussianMap:
    """gsmap::GaussianMap (map/gaussian_map.hpp:44-96) resident on the GPU (fp32 SoA + Adam)."""

    def __init__(self, ctx: Context | None = None, gaussians: np.ndarray | None = None, _handle=None):
        self.ctx = ctx or default_context()
        if _handle is not None:
            self.h = _handle
            return
        h = C.c_void_p()
        _check(lib().gs_map_create(_vp(self.ctx.h), C.byref(h)))
        self.h = h.value
        if gaussians is not None and len(gaussians):
            self.append(gaussians)

    def save_checkpoint(self, path: str):
        """save_checkpoint (io/checkpoint.cpp:17-35), format v1."""
        _check(lib().gs_save_checkpoint(_vp(self.h), os.fsencode(path)))

    def save_training_state(self, path: str):
        """Adam m / v / step and global_step beside a checkpoint (true resume)."""
        _check(lib().gs_save_training_state(_vp(self.h), os.fsencode(path)))

    def load_training_state(self, path: str):
        _check(lib().gs_load_training_state(_vp(self.h), os.fsencode(path)))

    @classmethod
    def load_checkpoint(cls, path: str, ctx: Context | None = None) -> "GaussianMap":
        """load_checkpoint (io/checkpoint.cpp:37-71): a new device map with fresh Adam state."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib().gs_load_checkpoint(_vp(ctx.h), os.fsencode(path), C.byref(h)))
        return cls(ctx, _handle=h.value)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gs_map_destroy(_vp(self.h))
                self.h = None
        except Exception:
            pass

    def __len__(self):
        n = C.c_int64()
        _check(lib().gs_map_size(_vp(self.h), C.byref(n)))
        return n.value

    def append(self, g: np.ndarray):
        g = np.ascontiguousarray(g, dtype=GAUSS_DTYPE)
        _check(lib().gs_map_append(_vp(self.h), _p(g), C.c_int64(len(g))))

    @property
    def gaussians(self) -> np.ndarray:
        n = len(self)
        g = np.zeros(n, dtype=GAUSS_DTYPE)
        _check(lib().gs_map_get_gaussians(_vp(self.h), _p(g), C.c_int64(n)))
        return g

    @gaussians.setter
    def gaussians(self, g: np.ndarray):
        g = np.ascontiguousarray(g, dtype=GAUSS_DTYPE)
        _check(lib().gs_map_set_gaussians(_vp(self.h), _p(g), C.c_int64(len(g))))

    def adam_state(self):
        n = len(self)
        m = np.zeros((n, 59)); v = np.zeros((n, 59)); s = np.zeros(n, np.int64)
        _check(lib().gs_map_get_adam(_vp(self.h), _p(m), _p(v), _p(s), C.c_int64(n)))
        return m, v, s

    def set_adam_state(self, m, v, s):
        m = np.ascontiguousarray(m, np.float64); v = np.ascontiguousarray(v, np.float64)
        s = np.ascontiguousarray(s, np.int64)
        _check(lib().gs_map_set_adam(_vp(self.h), _p(m), _p(v), _p(s), C.c_int64(len(s))))

    @property
    def scene_extent(self) -> float:
        e = C.c_double()
        _check(lib().gs_map_scene_extent(_vp(self.h), C.byref(e)))
        return e.value

    @scene_extent.setter
    def scene_extent(self, e: float):
        _check(lib().gs_map_set_scene_extent(_vp(self.h), C.c_double(e)))

    @property
    def global_step(self) -> int:
        s = C.c_int64()
        _check(lib().gs_map_global_step(_vp(self.h), C.byref(s)))
        return s.value

    @global_step.setter
    def global_step(self, s: int):
        _check(lib().gs_map_set_global_step(_vp(self.h), C.c_int64(s)))

    def raise_sh_degree(self, d: int):
        _check(lib().gs_map_raise_sh_degree(_vp(self.h), d))

    def maybe_upgrade_sh(self, sh_interval: int) -> int:
        """maybe_upgrade_sh (mapper.cpp:240-246): degree = min(3, global_step / sh_interval)."""
        d = C.c_int32()
        _check(lib().gs_maybe_upgrade_sh(_vp(self.h), C.c_int32(sh_interval), C.byref(d)))
        return d.value

    def init_from_points(self, points6: np.ndarray) -> int:
        """init_gaussians_from_points (mapper.cpp:43-61) on the device; returns the number added."""
        pts = np.ascontiguousarray(points6, np.float64)
        if pts.ndim != 2 or pts.shape[1] != 6:
            raise ValueError("init_from_points: points must be [n][6]")
        added = C.c_int64()
        _check(lib().gs_map_init_from_points(_vp(self.h), _p(pts), C.c_int64(len(pts)), C.byref(added)))
        return added.value

    def integrate_points(self, points6: np.ndarray, pose: Pose, cam: Camera, tau_alpha: float) -> int:
        """filter_points_by_visibility + init_gaussians_from_points on the device (pipeline.cpp:151-155)."""
        pts = np.ascontiguousarray(points6, np.float64)
        added = C.c_int64()
        _check(lib().gs_map_integrate_points(_vp(self.h), _p(pts), C.c_int64(len(pts)), C.byref(pose), C.byref(cam),
                                             C.c_double(tau_alpha), C.byref(added)))
        return added.value

    def integrate_keyframe(self, pose: Pose, cam: Camera, color: np.ndarray, points6: np.ndarray, tau_alpha: float,
                           initial_iters: int, levels: int) -> tuple["Keyframe", int]:
        """integrate_keyframe (pipeline.cpp:148-155) in one device call: the cloud is uploaded once,
        filtered by visibility and initialised into the map; the returned Keyframe holds the
        pyramid of `color` and of the cloud's project_sparse_depth. Returns (keyframe, added)."""
        col = np.ascontiguousarray(color, np.float64)
        if col.shape != (cam.height, cam.width, 3):
            raise ValueError("integrate_keyframe: colour shape does not match the camera")
        pts = np.ascontiguousarray(points6, np.float64).reshape(-1, 6)
        h = C.c_void_p()
        added = C.c_int64()
        _check(lib().gs_integrate_keyframe(_vp(self.h), C.byref(pose), C.byref(cam), _p(col), _p(pts),
                                           C.c_int64(len(pts)), C.c_double(tau_alpha), initial_iters, levels,
                                           C.byref(h), C.byref(added)))
        return Keyframe(pose, ctx=self.ctx, hw=(cam.height, cam.width), _handle=h.value), added.value

    def prune(self, opacity_threshold: float) -> int:
        """GaussianMap::prune (gaussian_map.cpp:56-73): removed count; state stays aligned."""
        removed = C.c_int64()
        _check(lib().gs_map_prune(_vp(self.h), C.c_double(opacity_threshold), C.byref(removed)))
        return removed.value

    def max_active_degree(self) -> int:
        d = C.c_int()
        _check(lib().gs_map_max_active_degree(_vp(self.h), C.byref(d)))
        return d.value

    def apply_gradients(self, grads: "RenderGradients", lr: LearningRates | None = None):
        """GaussianMap::apply_gradients (gaussian_map.cpp:37-54)."""
        _check(lib().gs_apply_gradients(_vp(self.h), _vp(grads.h), C.byref(lr or LearningRates.default())))

    def device_planes(self):
        p, m, v, cap = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_int64()
        _check(lib().gs_map_device_planes(_vp(self.h), C.byref(p), C.byref(m), C.byref(v), C.byref(cap)))
        return p.value, m.value, v.value, cap.value


# --------------------------------------------------------------------------- gradients
class RenderGradients:
    """gsmap::RenderGradients (rasterizer.hpp:62-64) as device fp32 planes [59][capacity]."""

    def __init__(self, ctx: Context | None = None, external_ptr: int | None = None, capacity: int = 0):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        if external_ptr is not None:
            _check(lib().gs_grads_create_external(_vp(self.ctx.h), C.c_void_p(external_ptr), C.c_int64(capacity),
                                                  C.byref(h)))
        else:
            _check(lib().gs_grads_create(_vp(self.ctx.h), C.byref(h)))
        self.h = h.value
        self.n = 0

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gs_grads_destroy(_vp(self.h))
                self.h = None
        except Exception:
            pass

    def zero(self, m: GaussianMap):
        _check(lib().gs_grads_zero(_vp(self.h), _vp(m.h)))
        self.n = len(m)

    def read(self, n: int | None = None) -> np.ndarray:
        n = self.n if n is None else n
        out = np.zeros((n, 59))
        _check(lib().gs_grads_read(_vp(self.h), _p(out), C.c_int64(n)))
        return out

    def write(self, g: np.ndarray):
        g = np.ascontiguousarray(g, np.float64)
        _check(lib().gs_grads_write(_vp(self.h), _p(g), C.c_int64(g.shape[0])))
        self.n = g.shape[0]

    @property
    def per_gaussian(self) -> np.ndarray:
        return self.read()

    def device_planes(self):
        p, cap = C.c_void_p(), C.c_int64()
        _check(lib().gs_grads_device_planes(_vp(self.h), C.byref(p), C.byref(cap)))
        return p.value, cap.value


# --------------------------------------------------------------------------- render
class RenderOutput:
    """gsmap::RenderOutput (rasterizer.hpp:43-59). Images download lazily as fp64 HWC; the
    contributor CSR and the projected set are materialised only on request."""

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib().gs_frame_create(_vp(self.ctx.h), C.byref(h)))
        self.h = h.value
        self.cam = None
        self._imgs = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gs_frame_destroy(_vp(self.h))
                self.h = None
        except Exception:
            pass

    def _images(self):
        if self._imgs is None:
            H, W = self.cam.height, self.cam.width
            c = np.zeros((H, W, 3)); d = np.zeros((H, W)); v = np.zeros((H, W))
            _check(lib().gs_frame_read(_vp(self.h), _p(c), _p(d), _p(v)))
            self._imgs = (c, d, v)
        return self._imgs

    @property
    def color(self):
        return self._images()[0]

    @property
    def depth(self):
        return self._images()[1]

    @property
    def visibility(self):
        return self._images()[2]

    def stats(self) -> FrameStats:
        s = FrameStats()
        _check(lib().gs_frame_stats_get(_vp(self.h), C.byref(s)))
        return s

    def pixel_state(self):
        H, W = self.cam.height, self.cam.width
        nc = np.zeros((H, W), np.int32); t = np.zeros((H, W), np.float32)
        _check(lib().gs_frame_read_pixel_state(_vp(self.h), _p(nc), _p(t)))
        return nc, t

    def projected(self):
        n = self.stats().n_visible
        d = dict(index=np.zeros(n, np.int32), mean=np.zeros((n, 2)), rect=np.zeros((n, 4), np.int32),
                 conic=np.zeros((n, 3), np.float32), opacity=np.zeros(n, np.float32),
                 color=np.zeros((n, 3), np.float32), depth=np.zeros(n))
        _check(lib().gs_frame_read_projected(_vp(self.h), *[_p(d[k]) for k in
                                             ("index", "mean", "rect", "conic", "opacity", "color", "depth")]))
        return d

    def tiles(self):
        s = self.stats()
        off = np.zeros(s.tiles_x * s.tiles_y + 1, np.int64); ent = np.zeros(s.n_pairs, np.int32)
        _check(lib().gs_frame_read_tiles(_vp(self.h), _p(off), _p(ent)))
        return off, ent

    def csr(self):
        s = self.stats()
        off = np.zeros(s.width * s.height + 1, np.uint32)
        g = np.zeros(s.n_contrib, np.int32); a = np.zeros(s.n_contrib)
        _check(lib().gs_frame_materialize(_vp(self.h), _p(off), _p(g), _p(a)))
        return off, g, a

    def contributors(self, y: int, x: int):
        off, g, a = self.csr()
        p = y * self.cam.width + x
        return list(zip(g[off[p]:off[p + 1]].tolist(), a[off[p]:off[p + 1]].tolist()))

    def device_images(self):
        c, d, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().gs_frame_device_images(_vp(self.h), C.byref(c), C.byref(d), C.byref(v)))
        return c.value, d.value, v.value


class EvalMetrics(C.Structure):
    _fields_ = [("psnr", C.c_double), ("ssim", C.c_double), ("depth_rmse", C.c_double)]


def save_checkpoint(path: str, m: GaussianMap):
    m.save_checkpoint(path)


def load_checkpoint(path: str, ctx: Context | None = None) -> GaussianMap:
    return GaussianMap.load_checkpoint(path, ctx)


def evaluate_view(m: GaussianMap, pose: Pose, cam: Camera, gt_color: np.ndarray,
                  gt_depth: np.ndarray | None = None) -> dict:
    """One frame of evaluate_sequence (pipeline.cpp:46-60) on the device: psnr / ssim of the
    quantize_8bit render against gt_color (HWC) and depth_rmse against gt_depth (NaN if None)."""
    gc = np.ascontiguousarray(gt_color, np.float64)
    if gc.shape != (cam.height, cam.width, 3):
        raise ValueError("evaluate_view: gt colour shape does not match the camera")
    gd = None if gt_depth is None else np.ascontiguousarray(gt_depth, np.float64)
    if gd is not None and gd.shape != (cam.height, cam.width):
        raise ValueError("evaluate_view: gt depth shape does not match the camera")
    r = EvalMetrics()
    _check(lib().gs_evaluate_view(_vp(m.h), C.byref(pose), C.byref(cam), _p(gc), _p(gd), C.byref(r)))
    return dict(psnr=r.psnr, ssim=r.ssim, depth_rmse=r.depth_rmse)


def evaluate_sequence(m: GaussianMap, frames, cam: Camera) -> list[dict]:
    """evaluate_sequence (pipeline.cpp:41-64): frames yields (pose, colour HWC, gt depth or
    None, LiDAR points or None); without gt depth the frame's cloud is projected
    (project_sparse_depth) as the reference does. Returns EvalRecord dicts."""
    import time
    start = time.monotonic()
    out = []
    for i, (pose, color, gt_depth, cloud) in enumerate(frames):
        if gt_depth is None and cloud is not None:
            gt_depth = project_sparse_depth(cloud, pose, cam, m.ctx)
        r = evaluate_view(m, pose, cam, color, gt_depth)
        r.update(frame=i, iteration=m.global_step, wall_time_s=time.monotonic() - start)
        out.append(r)
    return out


def filter_points_by_visibility(points6: np.ndarray, m: GaussianMap, pose: Pose, cam: Camera,
                                tau_alpha: float) -> np.ndarray:
    """keyframe.cpp:49-74 on the device: the kept points, in order."""
    pts = np.ascontiguousarray(points6, np.float64)
    out = np.zeros_like(pts)
    kept = C.c_int64()
    _check(lib().gs_filter_points_by_visibility(_vp(m.h), _p(pts), C.c_int64(len(pts)), C.byref(pose), C.byref(cam),
                                                C.c_double(tau_alpha), _p(out), C.byref(kept)))
    return out[: kept.value]


def project_sparse_depth(points: np.ndarray, pose: Pose, cam: Camera, ctx: Context | None = None) -> np.ndarray:
    """sequence.cpp:246-259 on the device: points [n][>=3] (world xyz first) -> [h][w] min camera z."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, np.float64)
    if pts.ndim != 2 or pts.shape[1] < 3:
        raise ValueError("project_sparse_depth: points must be [n][>=3]")
    out = np.zeros((cam.height, cam.width))
    _check(lib().gs_project_sparse_depth(_vp(ctx.h), _p(pts), C.c_int64(len(pts)), C.c_int32(pts.shape[1]),
                                         C.byref(pose), C.byref(cam), _p(out)))
    return out


def render(m: GaussianMap, pose: Pose, cam: Camera, out: RenderOutput | None = None, pool=None) -> RenderOutput:
    """rasterizer.hpp:69-70. ``pool`` (the reference's ThreadPool*) is accepted and ignored."""
    out = out or RenderOutput(m.ctx)
    out.cam = Camera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    out._imgs = None
    _check(lib().gs_render(_vp(m.h), C.byref(pose), C.byref(cam), _vp(out.h)))
    return out


def render_backward(m: GaussianMap, pose: Pose, cam: Camera, out: RenderOutput, dl_dcolor, dl_ddepth,
                    pool=None, grads: RenderGradients | None = None) -> RenderGradients:
    """rasterizer.hpp:74-77: fresh RenderGradients for the cotangents (host fp64 HWC)."""
    dc = np.ascontiguousarray(dl_dcolor, np.float64)
    dd = np.ascontiguousarray(dl_ddepth, np.float64)
    if dc.ndim != 3 or dc.shape != (cam.height, cam.width, 3):
        raise ValueError("render_backward: dl_dcolor dimensions mismatch")
    if dd.shape != (cam.height, cam.width):
        raise ValueError("render_backward: dl_ddepth dimensions mismatch")
    g = grads or RenderGradients(m.ctx)
    _check(lib().gs_render_backward(_vp(m.h), C.byref(pose), C.byref(cam), _vp(out.h), _p(dc), _p(dd),
                                    cam.height, cam.width, _vp(g.h)))
    g.n = len(m)
    return g


# --------------------------------------------------------------------------- keyframes / loss / step
class Keyframe:
    """gsmap::Keyframe hot-path fields (map/keyframe.hpp:23-34) with its pyramid on the device."""

    def __init__(self, pose: Pose, color=None, sparse_depth=None, initial_iters: int = 0, levels: int = 2,
                 ctx: Context | None = None, device_planes: tuple | None = None, hw: tuple | None = None,
                 _handle=None):
        self.ctx = ctx or default_context()
        self.pose = pose
        if _handle is not None:  # adopted from gs_integrate_keyframe
            self.h = _handle
            self.shape = hw
            return
        h = C.c_void_p()
        if device_planes is not None:
            H, W = hw
            _check(lib().gs_keyframe_create_device(_vp(self.ctx.h), C.byref(pose), C.c_void_p(device_planes[0]),
                                                   C.c_void_p(device_planes[1]), H, W, initial_iters, levels,
                                                   C.byref(h)))
        else:
            color = np.ascontiguousarray(color, np.float64)
            sparse_depth = np.ascontiguousarray(sparse_depth, np.float64)
            H, W = color.shape[:2]
            _check(lib().gs_keyframe_create(_vp(self.ctx.h), C.byref(pose), _p(color), _p(sparse_depth), H, W,
                                            initial_iters, levels, C.byref(h)))
        self.h = h.value
        self.shape = (H, W)

    def close(self):
        """Release the keyframe's device pyramid now (otherwise at garbage collection)."""
        if getattr(self, "h", None):
            h, self.h = self.h, None
            _check(lib().gs_keyframe_destroy(_vp(h)))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def consumed_iters(self) -> int:
        c = C.c_int32()
        _check(lib().gs_keyframe_consumed(_vp(self.h), C.byref(c)))
        return c.value

    @consumed_iters.setter
    def consumed_iters(self, c: int):
        _check(lib().gs_keyframe_set_consumed(_vp(self.h), c))

    def level_shape(self, l: int):
        if not 0 <= l:
            raise ValueError("level out of range")
        H, W = self.shape
        for _ in range(l):
            H, W = (H + 1) // 2, (W + 1) // 2
        return H, W

    def host_level(self, l: int, color: np.ndarray, depth: np.ndarray):
        """(colour, depth) checked for gs_keyframe_upload_level: C-contiguous fp64 of the level's
        (H, W, 3) / (H, W) shape. The C side reads exactly that many doubles, so anything else
        is converted (a copy) or rejected here; the caller must keep the returned arrays alive
        until the upload is consumed (the copy is asynchronous)."""
        H, W = self.level_shape(l)
        color = np.ascontiguousarray(color, np.float64)
        depth = np.ascontiguousarray(depth, np.float64)
        if color.shape != (H, W, 3) or depth.shape != (H, W):
            raise ValueError(f"upload_level: level {l} needs colour ({H}, {W}, 3) and depth ({H}, {W}), "
                             f"got {color.shape} and {depth.shape}")
        return color, depth

    def upload_level(self, l: int, color: np.ndarray, depth: np.ndarray):
        """Overwrite pyramid level ``l`` from host fp64 HWC images (pinned memory recommended;
        the copy is asynchronous, so a converted copy is kept alive on the keyframe until the next
        upload of any level)."""
        color, depth = self.host_level(l, color, depth)
        self._pending_upload = (color, depth)
        _check(lib().gs_keyframe_upload_level(_vp(self.h), l, _p(color), _p(depth)))

    def level(self, l: int):
        H, W = self.level_shape(l)
        c = np.zeros((H, W, 3)); d = np.zeros((H, W))
        _check(lib().gs_keyframe_read_level(_vp(self.h), l, _p(c), _p(d)))
        return c, d


def compute_loss(out: RenderOutput, kf: Keyframe, level: int, cfg: TrainConfig, with_cotangents: bool = True):
    """mapper.cpp:146-212 -> dict(total, color_loss, depth_loss, l1, ssim, psnr, dl_dcolor, dl_ddepth)."""
    r = LossResult()
    H, W = out.cam.height, out.cam.width
    dc = np.zeros((H, W, 3)) if with_cotangents else None
    dd = np.zeros((H, W)) if with_cotangents else None
    _check(lib().gs_compute_loss(_vp(out.h), _vp(kf.h), level, C.byref(cfg), C.byref(r), _p(dc), _p(dd)))
    res = {k: getattr(r, k) for k, _ in LossResult._fields_}
    res["dl_dcolor"], res["dl_ddepth"] = dc, dd
    return res


def train_keyframe_step(m: GaussianMap, kf: Keyframe, cfg: TrainConfig, cam: Camera, pool=None,
                        prefetch: tuple | None = None):
    """mapper.cpp:214-238. Returns dict(level, loss, psnr) or None when the budget is spent.
    prefetch = (next_keyframe, level[, colour HWC fp64, depth fp64]) names the NEXT step
    (gs_train_step_prefetch): its render is enqueued while this step's report is read back (and
    used by the next call if the map and camera are unchanged), and the images, if given, are
    uploaded on the copy stream behind this step's work; they must stay alive until the next call."""
    rep = StepReport()
    if prefetch is not None:
        nk, nl, nc, nd = (tuple(prefetch) + (None, None))[:4]  # (keyframe, level[, colour, depth])
        if (nc is None) != (nd is None):
            raise ValueError("train_keyframe_step: pass both prefetch images or neither")
        if nc is not None:
            # checked / converted like upload_level; kept alive on the next keyframe until its
            # next upload (the copy runs asynchronously behind this step)
            nc, nd = nk.host_level(int(nl), nc, nd)
            nk._pending_upload = (nc, nd)
        _check(lib().gs_train_step_prefetch(_vp(m.h), _vp(kf.h), C.byref(cfg), C.byref(cam), _vp(nk.h), int(nl),
                                            _p(nc), _p(nd), C.byref(rep)))
    else:
        _check(lib().gs_train_step(_vp(m.h), _vp(kf.h), C.byref(cfg), C.byref(cam), C.byref(rep)))
    if not rep.ran:
        return None
    return dict(level=rep.level, loss=rep.loss, psnr=rep.psnr)


def train_accumulate(m: GaussianMap, kf: Keyframe, cfg: TrainConfig, cam: Camera, grads: RenderGradients,
                     frame: RenderOutput | None = None, sync: bool = False):
    """One view of a keyframe batch: render + loss + backward, gradients summed into ``grads``."""
    rep = StepReport()
    _check(lib().gs_train_accumulate(_vp(m.h), _vp(kf.h), C.byref(cfg), C.byref(cam),
                                     _vp(frame.h) if frame else None, _vp(grads.h), int(sync), C.byref(rep)))
    grads.n = len(m)
    if not rep.ran:
        return None
    return dict(level=rep.level, loss=rep.loss, psnr=rep.psnr)


# --------------------------------------------------------------------------- multi-GPU batch
class Comm:
    """An NCCL communicator of the context's device (gs_comm_*). Every rank calls
    ``Comm(ctx, uid, nranks, rank)`` with the same ``uid = comm_unique_id()`` (shared out of
    band); ``Comm.wrap(ctx, nccl_comm_ptr)`` borrows an existing ncclComm_t instead."""

    def __init__(self, ctx: Context, uid: bytes | None = None, nranks: int = 1, rank: int = 0, _handle=None):
        self.ctx = ctx
        if _handle is not None:
            self.h = _handle
        else:
            uid = comm_unique_id() if uid is None else uid
            buf = (C.c_uint8 * 128).from_buffer_copy(uid)
            h = C.c_void_p()
            _check(lib().gs_comm_create(_vp(ctx.h), buf, nranks, rank, C.byref(h)))
            self.h = h.value
        n, r = C.c_int32(), C.c_int32()
        _check(lib().gs_comm_size(_vp(self.h), C.byref(n), C.byref(r)))
        self.nranks, self.rank = n.value, r.value

    @classmethod
    def wrap(cls, ctx: Context, nccl_comm: int):
        h = C.c_void_p()
        _check(lib().gs_comm_wrap(_vp(ctx.h), C.c_void_p(nccl_comm), C.byref(h)))
        return cls(ctx, _handle=h.value)

    def close(self):
        if getattr(self, "h", None):
            h, self.h = self.h, None
            _check(lib().gs_comm_destroy(_vp(h)))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().gs_comm_unique_id(buf))
    return bytes(buf)


def train_batch(m: GaussianMap, keyframes, cfg: TrainConfig, cam: Camera, comm: Comm | None = None,
                sharded: bool = False):
    """gs_train_batch: this rank's views (each keyframe at its scheduled level) -> gradients
    summed on the device -> NCCL reduce -> ONE Adam step. Returns the per-view reports (None for
    a keyframe whose budget is spent)."""
    n = len(keyframes)
    arr = (C.c_void_p * max(n, 1))(*[k.h for k in keyframes])
    reps = (StepReport * max(n, 1))()
    _check(lib().gs_train_batch(_vp(m.h), arr, n, C.byref(cfg), C.byref(cam), _vp(comm.h) if comm else None,
                                1 if sharded else 0, reps))
    return [dict(level=r.level, loss=r.loss, psnr=r.psnr) if r.ran else None for r in reps[:n]]


def gather_optimizer_state(m: GaussianMap, comm: Comm):
    """Re-replicate the Adam state a sharded train_batch left on each rank's own range."""
    _check(lib().gs_comm_gather_optimizer_state(_vp(m.h), _vp(comm.h)))


def optimizer_sharded(m: GaussianMap) -> bool:
    s = C.c_int32()
    _check(lib().gs_map_optimizer_sharded(_vp(m.h), C.byref(s)))
    return bool(s.value)
