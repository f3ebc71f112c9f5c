"""Loader for the reference's own compiled kernels (TEST INFRASTRUCTURE ONLY).

oracle/_ref/_ext*.so is /root/reference/pkg/src/fieldbridge/_kernels/_ext.pyx
cythonized and compiled by `make -C oracle ref` with the reference's flags
(setup.py:5-12).  The built module travels to the GPU box; the reference
sources do not, and nothing here reads /root/reference at run time.
"""

import glob
import importlib.util
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_mod = None


def available():
    return bool(glob.glob(os.path.join(_HERE, "_ref", "_ext*.so")))


def ext():
    """The reference `fieldbridge._kernels._ext` module (compiled Cython)."""
    global _mod
    if _mod is None:
        paths = glob.glob(os.path.join(_HERE, "_ref", "_ext*.so"))
        if not paths:
            raise ImportError("oracle/_ref not built (make -C oracle ref)")
        name = "fieldbridge._kernels._ext"
        spec = importlib.util.spec_from_file_location(name, paths[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _mod = mod
    return _mod


def import_reference_package(ref_src="/root/reference/pkg/src"):
    """Import the reference Python package `fieldbridge` (THIS container only;
    used by tests/golden/make_golden.py) with the compiled _ext backend."""
    if "fieldbridge" in sys.modules:
        return sys.modules["fieldbridge"]
    sys.modules["fieldbridge._kernels._ext"] = ext()
    if ref_src not in sys.path:
        sys.path.insert(0, ref_src)
    import fieldbridge

    assert fieldbridge._kernels.BACKEND == "ext", fieldbridge._kernels.BACKEND
    return fieldbridge
