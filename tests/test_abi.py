"""CPU: the C-ABI library loads and exports every function include/*.h
declares (no compute calls: there is no GPU here), and the ctypes structs
match the header's layout."""

import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT

HEADERS = sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))


def _declared_functions():
    text = "".join(open(h).read() for h in HEADERS)
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = _declared_functions()
    for required in ("fm_grid_build", "fm_support_count", "fm_support_fill", "fm_rbf_weights",
                     "fm_fit_many", "fm_build_operator", "fm_transfer_values", "fm_apply",
                     "fm_offsets_from_counts", "fm_target_order"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2510_18838_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail(f"{_lib.LIB_PATH} not built (python -m paper_2510_18838_b200._build)")
    L = _lib.lib()
    for name in _declared_functions():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_pure_host_entry_points():
    from paper_2510_18838_b200 import _lib

    L = _lib.lib()
    assert L.fm_version() >= 10000
    assert L.fm_error_string(-3).decode().startswith("unsupported")
    assert [L.fm_n_monomials(2, p) for p in range(4)] == [1, 3, 6, 10]
    assert L.fm_n_monomials(3, 3) == 20 and L.fm_n_monomials(5, 2) == 21
    assert L.fm_grid_workspace(1000, 1000) >= 3 * 4000
    assert L.fm_scan_workspace(0) > 0


def test_struct_layouts():
    from paper_2510_18838_b200._lib import FmFit, FmGrid, FmRbf, FmSelect

    assert ctypes.sizeof(FmGrid) == 4 + 4 + 5 * 8 * 3 + 8
    assert ctypes.sizeof(FmSelect) == 4 + 4 + 4 * 8
    assert ctypes.sizeof(FmRbf) == 16
    assert ctypes.sizeof(FmFit) == 24


def test_grid_geometry_c_equals_python():
    """fm_grid_geometry (host-only C, used on the hot path) reproduces
    locate.grid_geometry -- the reference's _pad_bbox/_grid_shape for dim 2,
    equal-side cells otherwise -- bit for bit, including degenerate boxes."""
    import numpy as np

    from paper_2510_18838_b200 import _lib
    from paper_2510_18838_b200.locate import grid_geometry

    L = _lib.lib()
    rs = np.random.RandomState(0)
    for _ in range(2000):
        dim = int(rs.randint(1, 6))
        lo = rs.uniform(-10, 10, dim)
        ext = rs.uniform(0, 20, dim) * 10.0 ** rs.randint(-6, 3, dim)
        hi = lo + np.where(rs.rand(dim) < 0.1, 0.0, ext)
        n = int(rs.randint(1, 10 ** 7))
        cpp = float(rs.choice([0.25, 1.0, 4.0, 0.7]))
        g = grid_geometry(lo, hi, n, cpp).to_ctypes()
        out = _lib.FmGrid()
        assert L.fm_grid_geometry(dim, lo.ctypes.data, hi.ctypes.data, n, cpp,
                                  ctypes.byref(out), None, None) == 0
        assert out.dim == g.dim and out.ncell == g.ncell
        for a in range(5):
            assert out.n[a] == g.n[a] and out.lo[a] == g.lo[a] and out.inv_d[a] == g.inv_d[a]
