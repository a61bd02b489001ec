"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a GPU and exports
every entry point include/gsmap_b200.h declares; errors come back as status codes, not crashes."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gsmap_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(gs_[a-z0-9_]+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2411_02703_b200 import gsmap
    if not os.path.exists(gsmap.LIB_PATH):
        import paper_2411_02703_b200 as pkg
        pkg.build()
    return gsmap.lib()


def test_header_declares_the_hot_path(lib):
    names = declared_symbols()
    for must in ("gs_render", "gs_render_backward", "gs_apply_gradients", "gs_compute_loss", "gs_train_step",
                 "gs_map_append", "gs_last_error", "gs_frame_materialize", "gs_train_accumulate"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_errors_are_status_codes(lib):
    import ctypes as C
    from paper_2411_02703_b200 import gsmap
    cam = gsmap.Camera(0.0, 1.0, 0.0, 0.0, 4, 4)
    assert lib.gs_camera_validate(C.byref(cam)) == gsmap.GS_EINVAL
    assert b"focal" in lib.gs_last_error()
    out = gsmap.Camera()
    assert lib.gs_camera_scaled(C.byref(gsmap.Camera(130, 130, 79.5, 59.5, 160, 120)), 1, C.byref(out)) == 0
    assert (out.width, out.height) == (80, 60)
    assert out.cx == pytest.approx((79.5 + 0.5) / 2 - 0.5)


def test_no_cpu_fallback_without_gpu(lib):
    """On a machine without a CUDA device the product fails loudly instead of computing on CPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    from paper_2411_02703_b200 import gsmap
    with pytest.raises(gsmap.CudaError):
        gsmap.Context(0)


def test_cpp_shim_compiles(lib):
    """The C++ host shim (include/gsmap_b200.hpp) builds against the C-ABI library."""
    import subprocess
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "_build", "test_shim"))
