"""The reference's OWN unit tests (proj/tests/test_rasterizer.cpp, test_mapper.cpp,
test_keyframe.cpp), compiled unchanged and linked against the reference with its five hot-path
definitions replaced at link time by the B200 backend (integration/gsmap_b200_backend.cpp,
integration/Makefile): the drop-in boundary exercised by unchanged reference callers.

Bar: every test case passes except the ones that need fp64 arithmetic the fp32 device does not
have (SURVEY §8c / north_star: 1e-4 on images, 1e-3 on gradients), each listed with its reason;
at the north_star tolerance (every Approx epsilon floored at 1e-4) the closed-form KATs pass too.
The reference's own CPU build is run beside it for the same table."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = os.path.join(ROOT, "integration", "_build", "ref_tests_b200")
CPU = os.path.join(ROOT, "integration", "_build", "ref_tests_cpu")

# test case -> why the fp32 device cannot meet the reference's fp64 assertion
FP64_ONLY = {
    "render: single on-axis Gaussian composites one term": "Approx(...).epsilon(1e-12) on an fp32 image",
    "render_backward: single-Gaussian opacity gradient matches the closed form":
        "epsilon 1e-9 closed form and a 1e-5 check against an fp64 finite difference",
    "gradient check: full render against finite differences (sampled)":
        "central differences (step 1e-4) of an fp32 render resolve ~1e-3 of the gradient",
    "compute_loss gradients match finite differences of the scalar":
        "central differences with step 1e-6 on fp32 depth images",
    "compute_loss: perfect render gives zero loss and zero gradients":
        "exact zeros; fails on the reference's own CPU build too (metrics.cpp:131-133 rounds two paths)",
}
# still failing with every epsilon floored at 1e-4: finite differences finer than fp32 resolves
FD_ONLY = {
    "gradient check: full render against finite differences (sampled)",
    "compute_loss gradients match finite differences of the scalar",
    "compute_loss: perfect render gives zero loss and zero gradients",
}


def run(binary, env=None):
    if not os.path.exists(binary):
        pytest.skip(f"{binary} not built (integration/Makefile needs /root/reference at build time)")
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([binary], capture_output=True, text=True, env=e, timeout=600)
    cases = {name: verdict for verdict, name in re.findall(r"^\[(PASS|FAIL)\] (.+?)  \(", p.stdout, re.M)}
    summary = re.findall(r"^\[doctest\] .*$", p.stdout, re.M)
    print("\n".join(summary))
    return cases, p.stdout


@pytest.mark.gpu
def test_reference_unit_tests_on_b200_backend():
    cases, out = run(B200)
    assert len(cases) == 41, out[-2000:]
    failed = {k for k, v in cases.items() if v == "FAIL"}
    for k in sorted(failed):
        print(f"  fp64-only: {k}: {FP64_ONLY.get(k, 'UNEXPECTED')}")
    assert failed <= set(FP64_ONLY), f"unexpected failures: {sorted(failed - set(FP64_ONLY))}"
    assert len(cases) - len(failed) >= 36


@pytest.mark.gpu
def test_reference_unit_tests_on_b200_backend_at_north_star_tolerance():
    cases, out = run(B200, {"DOCTEST_EPSILON_FLOOR": "1e-4"})
    failed = {k for k, v in cases.items() if v == "FAIL"}
    assert failed <= FD_ONLY, f"unexpected failures at 1e-4: {sorted(failed - FD_ONLY)}"


def test_reference_unit_tests_on_reference_cpu_build():
    """The same binary's other link: the unchanged reference (CPU, this container)."""
    cases, out = run(CPU)
    failed = {k for k, v in cases.items() if v == "FAIL"}
    assert failed == {"compute_loss: perfect render gives zero loss and zero gradients"}, sorted(failed)
