"""ctypes view of the synthetic measurement fixture (fixtures/_build/libgsfixture.so).

Restates proj/src/io/synthetic.cpp (scene + trajectory + LiDAR clouds) and builds the
colourised-LiDAR-initialised training map of SURVEY §8(d). Used identically by both bench
arms and by the tests; it is neither the product path nor the oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "libgsfixture.so")
GAUSS_DTYPE = np.dtype([("p", "<f8", (59,)), ("degree", "<i4"), ("pad", "<i4")])


class Spec(C.Structure):
    _fields_ = [("n_gaussians", C.c_int32), ("n_frames", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("seed", C.c_uint32), ("orbit", C.c_int32), ("extent", C.c_double), ("focal", C.c_double),
                ("lidar_noise", C.c_double)]


class _Cam(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class _Pose(C.Structure):
    _fields_ = [("qw", C.c_double), ("qx", C.c_double), ("qy", C.c_double), ("qz", C.c_double),
                ("tx", C.c_double), ("ty", C.c_double), ("tz", C.c_double)]


_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.gsf_last_error.restype = C.c_char_p
        _lib.gsf_scene_num_gaussians.restype = C.c_int64
        _lib.gsf_scene_num_gaussians.argtypes = [C.c_void_p]
        _lib.gsf_scene_num_points.restype = C.c_int64
        _lib.gsf_scene_num_points.argtypes = [C.c_void_p, C.c_int]
        _lib.gsf_scene_num_frames.argtypes = [C.c_void_p]
        _lib.gsf_scene_free.argtypes = [C.c_void_p]
        _lib.gsf_training_map.argtypes = [C.c_void_p, C.c_uint32, C.c_double, C.c_int, C.c_void_p]
        _lib.gsf_init_from_points.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
    return _lib


def _check(st):
    if st:
        raise ValueError(lib().gsf_last_error().decode())


class Scene:
    """generate_synthetic_scene(spec) without the GT renders (each arm renders them itself)."""

    def __init__(self, n_gaussians=500, width=160, height=120, focal=None, n_frames=20, seed=1,
                 extent=18.0, lidar_noise=0.06, trajectory="line"):
        focal = 0.8125 * width if focal is None else focal  # 130/160 (synthetic.hpp:17-19)
        spec = Spec(n_gaussians, n_frames, width, height, seed, 1 if trajectory == "orbit" else 0, extent, focal,
                    lidar_noise)
        h = C.c_void_p()
        _check(lib().gsf_scene_create(C.byref(spec), C.byref(h)))
        self.h = h.value
        L = lib()
        n = L.gsf_scene_num_gaussians(self.h)
        self.gaussians = np.zeros(n, GAUSS_DTYPE)
        L.gsf_scene_gaussians(C.c_void_p(self.h), self.gaussians.ctypes.data_as(C.c_void_p))
        cam = _Cam()
        L.gsf_scene_camera(C.c_void_p(self.h), C.byref(cam))
        self.camera = (cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
        self.n_frames = L.gsf_scene_num_frames(self.h)
        self.poses = []
        for f in range(self.n_frames):
            p = _Pose()
            L.gsf_scene_pose(C.c_void_p(self.h), f, C.byref(p))
            self.poses.append((p.qw, p.qx, p.qy, p.qz, p.tx, p.ty, p.tz))

    def __del__(self):
        if getattr(self, "h", None):
            lib().gsf_scene_free(self.h)
            self.h = None

    def cloud(self, f: int) -> np.ndarray:
        n = lib().gsf_scene_num_points(self.h, f)
        out = np.zeros((n, 6))
        lib().gsf_scene_points(C.c_void_p(self.h), f, out.ctypes.data_as(C.c_void_p))
        return out

    def sparse_depth(self, f: int, cam: tuple | None = None) -> np.ndarray:
        cam = cam or self.camera
        c = _Cam(*cam)
        out = np.zeros((c.height, c.width))
        lib().gsf_scene_sparse_depth(C.c_void_p(self.h), f, C.byref(c), out.ctypes.data_as(C.c_void_p))
        return out

    def training_map(self, seed: int = 2, noise: float = 0.06, threads: int = 0) -> np.ndarray:
        out = np.zeros(len(self.gaussians), GAUSS_DTYPE)
        _check(lib().gsf_training_map(self.h, seed, noise, threads, out.ctypes.data_as(C.c_void_p)))
        return out


def init_from_points(pts6: np.ndarray, threads: int = 0) -> np.ndarray:
    pts6 = np.ascontiguousarray(pts6, np.float64)
    out = np.zeros(len(pts6), GAUSS_DTYPE)
    _check(lib().gsf_init_from_points(pts6.ctypes.data_as(C.c_void_p), len(pts6), threads,
                                      out.ctypes.data_as(C.c_void_p)))
    return out
