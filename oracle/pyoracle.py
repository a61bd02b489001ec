"""TEST INFRASTRUCTURE ONLY — ctypes view of the CPU fp64 oracle (oracle/_build/liborc.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may
import this module. The product (paper_2411_02703_b200) never does.

Layout conventions (shared with the product's C-ABI, include/gsmap_b200.h):
  * a Gaussian is 59 fp64 scalars in reference order (gaussian.hpp:16-26): position 3, rotation
    (w,x,y,z) 4, log_scale 3, opacity_logit 1, sh[16][3] 48; plus int32 active_degree.
  * images are row-major HWC fp64 (io/image.hpp:26-33).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")  # oracle/pyref.py rebinds this to oracle/_ref

GAUSS_DTYPE = np.dtype([("p", "<f8", (59,)), ("degree", "<i4"), ("pad", "<i4")])


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]

    def tuple(self):
        return (self.fx, self.fy, self.cx, self.cy, self.width, self.height)


class Pose(C.Structure):
    _fields_ = [("qw", C.c_double), ("qx", C.c_double), ("qy", C.c_double), ("qz", C.c_double),
                ("tx", C.c_double), ("ty", C.c_double), ("tz", C.c_double)]


class LR(C.Structure):
    _fields_ = [("position", C.c_double), ("rotation", C.c_double), ("log_scale", C.c_double),
                ("opacity", C.c_double), ("sh", C.c_double)]


class Cfg(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("lambda_d", C.c_double), ("pyramid_levels", C.c_int32),
                ("iters_per_level", C.c_int32), ("lr", LR)]


def default_lr() -> LR:
    return LR(1.6e-4, 1e-3, 5e-3, 5e-2, 2.5e-3)


def make_cfg(lam=0.2, lam_d=0.5, levels=2, ipl=0, lr: LR | None = None) -> Cfg:
    return Cfg(lam, lam_d, levels, ipl, lr or default_lr())


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class LogicError(OracleError):
    pass


_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class _Sym:
    """Attribute sink for a symbol the loaded build does not export (the reference build,
    oracle/_ref/libgsref.so, lacks the restatement-only helpers): declaring it is a no-op."""

    def __setattr__(self, k, v):
        pass


def _declare(real):
    class _Tolerant:
        def __getattr__(self, name):
            return getattr(real, name) if hasattr(real, name) else _Sym()

    L = _Tolerant()
    P = C.c_void_p
    dp = C.POINTER(C.c_double)
    L.orc_last_error.restype = C.c_char_p
    L.orc_map_create.restype = P
    L.orc_map_create.argtypes = [P, C.c_int64]
    L.orc_map_free.argtypes = [P]
    L.orc_map_size.restype = C.c_int64
    L.orc_map_size.argtypes = [P]
    L.orc_map_scene_extent.restype = C.c_double
    L.orc_map_scene_extent.argtypes = [P]
    L.orc_map_set_scene_extent.argtypes = [P, C.c_double]
    L.orc_map_global_step.restype = C.c_int64
    L.orc_map_global_step.argtypes = [P]
    L.orc_map_set_global_step.argtypes = [P, C.c_int64]
    L.orc_map_prune.restype = C.c_int64
    L.orc_map_prune.argtypes = [P, C.c_double, C.POINTER(C.c_int)]
    for name in ("orc_map_get", "orc_map_set", "orc_map_raise_sh_degree", "orc_map_max_active_degree",
                 "orc_maybe_upgrade_sh", "orc_out_free", "orc_out_images", "orc_out_csr",
                 "orc_out_projected", "orc_out_bins", "orc_keyframe_free", "orc_pool_free",
                 "orc_rng_free", "orc_map_get_adam", "orc_map_set_adam", "orc_keyframe_set_consumed"):
        setattr(getattr(L, name), "argtypes", None)
    L.orc_map_raise_sh_degree.argtypes = [P, C.c_int]
    L.orc_map_max_active_degree.argtypes = [P]
    L.orc_maybe_upgrade_sh.argtypes = [P, C.c_int]
    L.orc_out_num_contribs.restype = C.c_int64
    L.orc_out_num_contribs.argtypes = [P]
    L.orc_out_num_projected.restype = C.c_int64
    L.orc_out_num_projected.argtypes = [P]
    L.orc_out_num_bin_entries.restype = C.c_int64
    L.orc_out_num_bin_entries.argtypes = [P]
    L.orc_out_is_smooth.argtypes = [P, P]
    L.orc_keyframe_create.restype = P
    L.orc_keyframe_consumed.argtypes = [P]
    L.orc_pool_create.restype = P
    L.orc_pool_create.argtypes = [C.c_int]
    L.orc_pool_threads.argtypes = [P]
    L.orc_rng_create.restype = P
    L.orc_rng_create.argtypes = [C.c_uint32]
    L.orc_rng_uniform.restype = C.c_double
    L.orc_rng_uniform.argtypes = [P, C.c_double, C.c_double]
    L.orc_random_scene.restype = P
    L.orc_random_scene.argtypes = [P, C.c_int, C.POINTER(Camera), C.POINTER(Pose), C.c_double, C.c_double]
    L.orc_pose_make.argtypes = [C.c_double] * 7 + [C.POINTER(Pose)]
    L.orc_run_gradcheck.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp]


def _check(status: int):
    if status == 0:
        return
    msg = lib().orc_last_error().decode()
    if status == 1:
        raise InvalidArgument(msg)
    if status == 2:
        raise LogicError(msg)
    raise OracleError(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def pose(w=1.0, x=0.0, y=0.0, z=0.0, t=(0.0, 0.0, 0.0)) -> Pose:
    """gsmap::Pose(q, t): stores q.normalized() (types.hpp:53-54)."""
    out = Pose()
    _check(lib().orc_pose_make(w, x, y, z, t[0], t[1], t[2], C.byref(out)))
    return out


def camera(fx, fy, cx, cy, width, height) -> Camera:
    return Camera(fx, fy, cx, cy, width, height)


def validate_camera(cam: Camera):
    _check(lib().orc_camera_validate(C.byref(cam)))


def camera_scaled(cam: Camera, level: int) -> Camera:
    out = Camera()
    _check(lib().orc_camera_scaled(C.byref(cam), level, C.byref(out)))
    return out


def camera_center(p: Pose) -> np.ndarray:
    out = np.zeros(3)
    _check(lib().orc_pose_camera_center(C.byref(p), _ptr(out)))
    return out


def empty_gaussians(n: int) -> np.ndarray:
    g = np.zeros(n, dtype=GAUSS_DTYPE)
    g["p"][:, 3] = 1.0  # identity rotation (w=1)
    return g


def make_blob(pos, opacity, color, log_scale=-1.5) -> np.ndarray:
    """tests/test_rasterizer.cpp:19-27 make_blob."""
    g = empty_gaussians(1)
    g["p"][0, 0:3] = pos
    g["p"][0, 7:10] = log_scale
    g["p"][0, 10] = np.log(opacity / (1.0 - opacity))
    g["p"][0, 11:14] = (np.asarray(color, dtype=float) - 0.5) / 0.28209479177387814
    return g


class OracleMap:
    def __init__(self, gaussians: np.ndarray | None = None, handle=None):
        L = lib()
        if handle is not None:
            self.h = handle
        else:
            g = np.ascontiguousarray(gaussians if gaussians is not None else empty_gaussians(0), dtype=GAUSS_DTYPE)
            self.h = L.orc_map_create(_ptr(g), len(g))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_map_free(C.c_void_p(self.h))
            self.h = None

    def __len__(self):
        return lib().orc_map_size(self.h)

    @property
    def gaussians(self) -> np.ndarray:
        g = np.zeros(len(self), dtype=GAUSS_DTYPE)
        lib().orc_map_get(C.c_void_p(self.h), _ptr(g))
        return g

    @gaussians.setter
    def gaussians(self, g: np.ndarray):
        g = np.ascontiguousarray(g, dtype=GAUSS_DTYPE)
        assert len(g) == len(self)
        lib().orc_map_set(C.c_void_p(self.h), _ptr(g))

    def adam_state(self):
        n = len(self)
        m = np.zeros((n, 59)); v = np.zeros((n, 59)); s = np.zeros(n, dtype=np.int64)
        lib().orc_map_get_adam(C.c_void_p(self.h), _ptr(m), _ptr(v), _ptr(s))
        return m, v, s

    def set_adam_state(self, m, v, s):
        m = np.ascontiguousarray(m, dtype=np.float64); v = np.ascontiguousarray(v, dtype=np.float64)
        s = np.ascontiguousarray(s, dtype=np.int64)
        lib().orc_map_set_adam(C.c_void_p(self.h), _ptr(m), _ptr(v), _ptr(s))

    @property
    def scene_extent(self) -> float:
        return lib().orc_map_scene_extent(self.h)

    @scene_extent.setter
    def scene_extent(self, e: float):
        lib().orc_map_set_scene_extent(self.h, e)

    @property
    def global_step(self) -> int:
        return lib().orc_map_global_step(self.h)

    @global_step.setter
    def global_step(self, s: int):
        lib().orc_map_set_global_step(self.h, s)

    def append(self, g: np.ndarray):
        g = np.ascontiguousarray(g, dtype=GAUSS_DTYPE)
        _check(lib().orc_map_append(C.c_void_p(self.h), _ptr(g), C.c_int64(len(g))))

    def prune(self, thr: float) -> int:
        st = C.c_int(0)
        r = lib().orc_map_prune(self.h, thr, C.byref(st))
        _check(st.value)
        return r

    def raise_sh_degree(self, d: int):
        lib().orc_map_raise_sh_degree(C.c_void_p(self.h), d)

    def max_active_degree(self) -> int:
        return lib().orc_map_max_active_degree(C.c_void_p(self.h))

    def maybe_upgrade_sh(self, interval: int) -> int:
        return lib().orc_maybe_upgrade_sh(C.c_void_p(self.h), interval)

    def apply_gradients(self, grads: np.ndarray, lr: LR | None = None):
        grads = np.ascontiguousarray(grads, dtype=np.float64)
        _check(lib().orc_apply_gradients(C.c_void_p(self.h), _ptr(grads), C.c_int64(grads.shape[0]),
                                         C.byref(lr or default_lr())))

    def init_from_points(self, pts6: np.ndarray) -> int:
        pts6 = np.ascontiguousarray(pts6, dtype=np.float64)
        added = C.c_int64(0)
        _check(lib().orc_init_from_points(C.c_void_p(self.h), _ptr(pts6), C.c_int64(len(pts6)), C.byref(added)))
        return added.value


class RenderResult:
    """gsmap::RenderOutput (rasterizer.hpp:43-59) + the oracle's bin_tiles lists."""

    def __init__(self, handle, cam: Camera):
        self.h = handle
        self.cam = cam
        H, W = cam.height, cam.width
        L = lib()
        self.color = np.zeros((H, W, 3)); self.depth = np.zeros((H, W)); self.visibility = np.zeros((H, W))
        L.orc_out_images(C.c_void_p(handle), _ptr(self.color), _ptr(self.depth), _ptr(self.visibility))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_out_free(C.c_void_p(self.h))
            self.h = None

    def csr(self):
        L = lib()
        n = L.orc_out_num_contribs(self.h)
        off = np.zeros(self.cam.height * self.cam.width + 1, dtype=np.uint32)
        g = np.zeros(n, dtype=np.int32); a = np.zeros(n)
        L.orc_out_csr(C.c_void_p(self.h), _ptr(off), _ptr(g), _ptr(a))
        return off, g, a

    def projected(self):
        L = lib()
        n = L.orc_out_num_projected(self.h)
        d = dict(index=np.zeros(n, np.int32), mean=np.zeros((n, 2)), cov2d=np.zeros((n, 2, 2)),
                 cov_inv=np.zeros((n, 2, 2)), depth=np.zeros(n), radius=np.zeros(n, np.int32),
                 opacity=np.zeros(n), color=np.zeros((n, 3)), color_raw=np.zeros((n, 3)))
        L.orc_out_projected(C.c_void_p(self.h), *[_ptr(d[k]) for k in
                            ("index", "mean", "cov2d", "cov_inv", "depth", "radius", "opacity", "color", "color_raw")])
        return d

    def bins(self):
        """(tile_offsets[T+1], entries[K]) with entries = rank into projected (bin_tiles order)."""
        L = lib()
        k = L.orc_out_num_bin_entries(self.h)
        tx = (self.cam.width + 15) // 16; ty = (self.cam.height + 15) // 16
        off = np.zeros(tx * ty + 1, dtype=np.int64); ent = np.zeros(k, dtype=np.int32)
        L.orc_out_bins(C.c_void_p(self.h), _ptr(off), _ptr(ent))
        return off, ent

    def n_contrib(self) -> np.ndarray:
        off, _, _ = self.csr()
        return np.diff(off.astype(np.int64)).reshape(self.cam.height, self.cam.width)


def render(m: OracleMap, p: Pose, cam: Camera, threads: int = 1) -> RenderResult:
    h = C.c_void_p()
    _check(lib().orc_render(C.c_void_p(m.h), C.byref(p), C.byref(cam), threads, C.byref(h)))
    return RenderResult(h.value, cam)


def is_smooth(m: OracleMap, out: RenderResult) -> bool:
    return bool(lib().orc_out_is_smooth(C.c_void_p(m.h), C.c_void_p(out.h)))


def render_backward(m: OracleMap, p: Pose, cam: Camera, out: RenderResult, dcolor, ddepth,
                    threads: int = 1) -> np.ndarray:
    dcolor = np.ascontiguousarray(dcolor, dtype=np.float64)
    ddepth = np.ascontiguousarray(ddepth, dtype=np.float64)
    dh, dw = dcolor.shape[0], dcolor.shape[1]
    if dcolor.ndim != 3 or dcolor.shape[2] != 3:
        raise InvalidArgument("render_backward: dl_dcolor dimensions mismatch")
    g = np.zeros((len(m), 59))
    _check(lib().orc_render_backward(C.c_void_p(m.h), C.byref(p), C.byref(cam), C.c_void_p(out.h),
                                     _ptr(dcolor), _ptr(ddepth), dh, dw, threads, _ptr(g)))
    return g


def brute_force(m: OracleMap, p: Pose, cam: Camera):
    H, W = cam.height, cam.width
    c = np.zeros((H, W, 3)); d = np.zeros((H, W)); v = np.zeros((H, W))
    _check(lib().orc_brute_force(C.c_void_p(m.h), C.byref(p), C.byref(cam), _ptr(c), _ptr(d), _ptr(v)))
    return c, d, v


def psnr(a, b) -> float:
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    sh = a.shape + (1,) * (3 - a.ndim)
    if a.shape != b.shape:
        raise InvalidArgument("psnr: image dimensions mismatch")
    out = C.c_double()
    _check(lib().orc_psnr(_ptr(a), _ptr(b), sh[0], sh[1], sh[2], C.byref(out)))
    return out.value


def ssim(a, b, with_grad=False):
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape:
        raise InvalidArgument("ssim: image dimensions mismatch")
    sh = a.shape + (1,) * (3 - a.ndim)
    out = C.c_double()
    g = np.zeros(a.shape) if with_grad else None
    _check(lib().orc_ssim(_ptr(a), _ptr(b), sh[0], sh[1], sh[2], C.byref(out), _ptr(g) if with_grad else None))
    return (out.value, g) if with_grad else out.value


def depth_rmse(r, g):
    r = np.ascontiguousarray(r, np.float64); g = np.ascontiguousarray(g, np.float64)
    out = C.c_double(); e = C.c_int(0)
    _check(lib().orc_depth_rmse(_ptr(r), _ptr(g), r.shape[0], r.shape[1], C.byref(out), C.byref(e)))
    return out.value, bool(e.value)


def compute_loss(color, depth, vis, gt_color, gt_depth, cfg: Cfg):
    H, W = gt_color.shape[:2]
    arrs = [np.ascontiguousarray(x, np.float64) for x in (color, depth, vis, gt_color, gt_depth)]
    if arrs[0].shape != arrs[3].shape:
        raise InvalidArgument("compute_loss: rendered resolution does not match level")
    dC = np.zeros((H, W, 3)); dD = np.zeros((H, W)); s = np.zeros(5)
    _check(lib().orc_compute_loss(*[_ptr(a) for a in arrs], H, W, C.byref(cfg), _ptr(dC), _ptr(dD), _ptr(s)))
    return dict(total=s[0], color_loss=s[1], depth_loss=s[2], l1=s[3], ssim=s[4], dl_dcolor=dC, dl_ddepth=dD)


def build_pyramid(img, levels: int, depth: bool = False):
    img = np.ascontiguousarray(img, np.float64)
    H, W = img.shape[:2]
    c = 1 if img.ndim == 2 else img.shape[2]
    shapes = []
    h, w = H, W
    for _ in range(levels + 1):
        shapes.append((h, w)); h, w = (h + 1) // 2, (w + 1) // 2
    total = sum(a * b * c for a, b in shapes)
    out = np.zeros(total)
    _check(lib().orc_build_pyramid(_ptr(img), H, W, c, levels, int(depth), _ptr(out)))
    res, off = [], 0
    for (h, w) in shapes:
        n = h * w * c
        res.append(out[off:off + n].reshape((h, w) if img.ndim == 2 else (h, w, c)))
        off += n
    return res


class Keyframe:
    def __init__(self, p: Pose, color, sparse_depth, initial_iters: int, levels: int):
        color = np.ascontiguousarray(color, np.float64); sparse_depth = np.ascontiguousarray(sparse_depth, np.float64)
        st = C.c_int(0)
        L = lib()
        L.orc_keyframe_create.argtypes = [C.POINTER(Pose), C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        self.h = L.orc_keyframe_create(C.byref(p), _ptr(color), _ptr(sparse_depth), color.shape[0],
                                       color.shape[1], initial_iters, levels, C.byref(st))
        _check(st.value)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_keyframe_free(C.c_void_p(self.h))
            self.h = None

    @property
    def consumed_iters(self) -> int:
        return lib().orc_keyframe_consumed(C.c_void_p(self.h))

    @consumed_iters.setter
    def consumed_iters(self, c: int):
        lib().orc_keyframe_set_consumed(C.c_void_p(self.h), c)


class ThreadPool:
    def __init__(self, threads: int = 0):
        self.h = lib().orc_pool_create(threads)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_pool_free(C.c_void_p(self.h))
            self.h = None

    @property
    def threads(self) -> int:
        return lib().orc_pool_threads(C.c_void_p(self.h))


def train_keyframe_step(m: OracleMap, kf: Keyframe, cfg: Cfg, cam: Camera, pool: ThreadPool | None = None):
    ran = C.c_int(0); level = C.c_int(0); loss = C.c_double(); ps = C.c_double()
    _check(lib().orc_train_step(C.c_void_p(m.h), C.c_void_p(kf.h), C.byref(cfg), C.byref(cam),
                                C.c_void_p(pool.h) if pool else None, C.byref(ran), C.byref(level),
                                C.byref(loss), C.byref(ps)))
    if not ran.value:
        return None
    return dict(level=level.value, loss=loss.value, psnr=ps.value)


def project_sparse_depth(pts6, p: Pose, cam: Camera):
    pts6 = np.ascontiguousarray(pts6, np.float64)
    out = np.zeros((cam.height, cam.width))
    _check(lib().orc_project_sparse_depth(_ptr(pts6), C.c_int64(len(pts6)), C.byref(p), C.byref(cam), _ptr(out)))
    return out


def filter_points_by_visibility(pts6, m: OracleMap, p: Pose, cam: Camera, tau_alpha: float) -> np.ndarray:
    """keyframe.cpp:49-74: indices of the kept points."""
    pts6 = np.ascontiguousarray(pts6, np.float64)
    kept = np.zeros(max(len(pts6), 1), np.int64)
    nk = C.c_int64()
    _check(lib().orc_filter_points_by_visibility(C.c_void_p(m.h), _ptr(pts6), C.c_int64(len(pts6)), C.byref(p),
                                                 C.byref(cam), C.c_double(tau_alpha),
                                                 kept.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(nk)))
    return kept[: nk.value]


def save_checkpoint(path: str, m: OracleMap):
    """io/checkpoint.cpp:17-35 (format v1)."""
    _check(lib().orc_save_checkpoint(C.c_void_p(m.h), os.fsencode(path)))


def load_checkpoint(path: str) -> OracleMap:
    """io/checkpoint.cpp:37-71: a fresh map (fresh Adam state) holding the file's Gaussians."""
    h = C.c_void_p()
    _check(lib().orc_load_checkpoint(os.fsencode(path), C.byref(h)))
    return OracleMap(handle=h.value)


def evaluate_view(m: OracleMap, p: Pose, cam: Camera, gt_color, gt_depth=None) -> dict:
    """evaluate_sequence (pipeline.cpp:41-64) for one frame: psnr / ssim of the quantized render, depth_rmse."""
    gc = np.ascontiguousarray(gt_color, np.float64)
    gd = None if gt_depth is None else np.ascontiguousarray(gt_depth, np.float64)
    r = np.zeros(3)
    _check(lib().orc_evaluate_view(C.c_void_p(m.h), C.byref(p), C.byref(cam), _ptr(gc),
                                   None if gd is None else _ptr(gd), _ptr(r)))
    return dict(psnr=r[0], ssim=r[1], depth_rmse=r[2])


class Rng:
    """std::mt19937 with std::uniform_real_distribution<double> draws (libstdc++)."""

    def __init__(self, seed: int):
        self.h = lib().orc_rng_create(seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_rng_free(C.c_void_p(self.h))
            self.h = None

    def uniform(self, lo, hi) -> float:
        return lib().orc_rng_uniform(self.h, lo, hi)


def random_scene(rng: Rng, n: int, cam: Camera, p: Pose, lo=-2.5, hi=1.5) -> OracleMap:
    h = lib().orc_random_scene(rng.h, n, C.byref(cam), C.byref(p), lo, hi)
    return OracleMap(handle=h)


def run_gradcheck(seed=1, configs=60, core_configs=120, n_gaussians=25, image_size=32, params_per_config=8):
    r = np.zeros(4)
    _check(lib().orc_run_gradcheck(seed, configs, core_configs, n_gaussians, image_size, params_per_config,
                                   r.ctypes.data_as(C.POINTER(C.c_double))))
    return dict(max_rel_err_core=r[0], max_rel_err_render=r[1], configs_run=int(r[2]), configs_resampled=int(r[3]))


def build_covariance(q, ls):
    q = np.ascontiguousarray(q, np.float64); ls = np.ascontiguousarray(ls, np.float64)
    out = np.zeros(9)
    _check(lib().orc_build_covariance(_ptr(q), _ptr(ls), _ptr(out)))
    return out.reshape(3, 3)


def project_gaussian(g: np.ndarray, p: Pose, cam: Camera):
    g = np.ascontiguousarray(g, dtype=GAUSS_DTYPE)
    vis = C.c_int32(0); mean = np.zeros(2); cov = np.zeros(4); depth = C.c_double(); radius = C.c_int32()
    _check(lib().orc_project_gaussian(_ptr(g), C.byref(p), C.byref(cam), C.byref(vis), _ptr(mean), _ptr(cov),
                                      C.byref(depth), C.byref(radius)))
    if not vis.value:
        return None
    return dict(mean=mean, cov2d=cov.reshape(2, 2), depth=depth.value, radius=radius.value)


def eval_gaussian_2d(mean, cov, x) -> float:
    mean = np.ascontiguousarray(mean, np.float64); cov = np.ascontiguousarray(cov, np.float64).reshape(4)
    x = np.ascontiguousarray(x, np.float64)
    out = C.c_double()
    _check(lib().orc_eval_gaussian_2d(_ptr(mean), _ptr(cov), _ptr(x), C.byref(out)))
    return out.value


def eval_sh(coeffs48, degree: int, direction):
    c = np.ascontiguousarray(coeffs48, np.float64).reshape(48)
    d = np.ascontiguousarray(direction, np.float64)
    out = np.zeros(3)
    _check(lib().orc_eval_sh(_ptr(c), degree, _ptr(d), _ptr(out)))
    return out
