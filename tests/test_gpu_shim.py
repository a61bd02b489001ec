"""Runs the reference's rasterizer/mapper known-answer tests written against the C++ shim
(tests/cpp/test_shim.cpp) on the GPU: the host side in C++, calling the kernels through the
C-ABI exactly as the reference's mapping thread would."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_cpp_shim_kats():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "_build", "test_shim")], capture_output=True, text=True,
                       timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 9
