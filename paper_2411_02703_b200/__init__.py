"""B200-native (sm_100a) drop-in for the LVI-GS mapping hot path: differentiable tile
rasterizer (forward + backward), pyramid L1/SSIM/LiDAR-depth loss and the per-Gaussian Adam
step, behind a C-ABI (include/gsmap_b200.h) mirroring proj/include/gsmap's interface.

The kernels live in csrc/ and build in-tree into libgsmap_b200.so; see DESIGN.md.
"""
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libgsmap_b200.so")


def build(verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a into the in-tree shared library."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.check_call(["make", "-j8", "-C", os.path.join(PKG_DIR, "csrc")], stdout=out)
    return LIB_PATH
