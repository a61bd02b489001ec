"""TEST INFRASTRUCTURE ONLY — the reference ITSELF behind the oracle's Python interface.

``oracle/_ref/libgsref.so`` is the reference's own source tree (/root/reference/proj/src,
unchanged) compiled by ``oracle/ref/Makefile`` against ``oracle/ref_eigen`` (a restatement of
the Eigen 3.4 subset it uses; Eigen is not installed here). It exports the oracle's flat C-ABI
(``orc_*``, implemented in ``oracle/ref/ref_capi.cpp`` over the reference's public API), so this
module is a second, independent instance of ``oracle/pyoracle.py`` bound to it: every wrapper
(``render``, ``render_backward``, ``compute_loss``, ``train_keyframe_step`` ...) runs the
reference's code. Tests use it to pin the restatement (``tests/test_ref_pin_cpu.py``) and
``tests/golden/make_golden.py`` uses it to produce the golden vectors.

Only tests/, __graft_entry__ (build) and bench.py's reference arm may import this module.
Helpers the reference has no public equivalent for (tile bins, optimizer-state setters,
``evaluate_view``) raise ``AttributeError`` here.
"""
from __future__ import annotations

import importlib.util
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(_HERE, "_ref", "libgsref.so")
REF_SOURCES = "/root/reference/proj"


def available() -> bool:
    """The reference build exists (it is built here, where /root/reference is, and travels)."""
    if os.path.exists(REF_LIB):
        return True
    if os.path.isdir(REF_SOURCES):
        build()
        return os.path.exists(REF_LIB)
    return False


def build():
    subprocess.check_call(["make", "-s", "-j8", "-C", os.path.join(_HERE, "ref")])


def load():
    """A fresh module object with pyoracle's wrappers, bound to the reference build."""
    if not available():
        raise ImportError("oracle/_ref/libgsref.so is not built and /root/reference is absent")
    spec = importlib.util.spec_from_file_location("pyoracle_ref", os.path.join(_HERE, "pyoracle.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod._LIB_PATH = REF_LIB
    kind = mod.lib().orc_build_kind
    kind.restype = __import__("ctypes").c_char_p
    assert kind().decode().startswith("reference"), "pyref loaded the restatement instead of the reference"
    return mod
