"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.  It is the checker, never the thing measured or shipped;
the product package (paper_2510_18838_b200) does not import it.

Functions mirror the reference's `fieldbridge._kernels` signatures
(/root/reference/pkg/src/fieldbridge/_kernels/_ext.pyx:65, 203-207, 238-243,
291-293) and add `*_nd` variants for dimension != 2 and several field
components.  The C code is oracle/fb_oracle.c; LAPACK dgelsy is the very
same scipy-openblas routine the reference calls through
scipy.linalg.cython_lapack (_ext.pyx:14).

Parity status: pinned.  tests/test_oracle.py checks these functions bitwise
against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and, when oracle/_ref is built, against the
reference's compiled _ext module directly.
"""

import ctypes
import glob
import os
import subprocess

import numpy as np

from .pointgrid import OraclePointGrid

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")

RBF_GAUSSIAN = 0
RBF_C4 = 1
RBF_CONST = 2
RBF_IDENTITY = 3
RBF_MULTIQUADRIC = 4
RBF_INVERSE_MULTIQUADRIC = 5
RBF_THIN_PLATE_SPLINE = 6
RBF_CUBIC_SPLINE = 7
FIT_OK = 0
FIT_SINGULAR = 1
FIT_EMPTY = 2

_lib = None


def build():
    """Compile oracle/fb_oracle.c into oracle/_build/liborc.so."""
    subprocess.check_call(["make", "-s", "-C", _HERE, "liborc"])


def _scipy_dgelsy_ptr():
    import scipy
    import scipy.linalg  # noqa: F401  (loads the openblas shared object)
    libdir = os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)), "scipy.libs")
    cands = sorted(glob.glob(os.path.join(libdir, "libscipy_openblas*.so")))
    if not cands:
        raise RuntimeError("scipy-openblas not found; cannot bind dgelsy")
    blas = ctypes.CDLL(cands[0])
    return ctypes.cast(blas.scipy_dgelsy_, ctypes.c_void_p).value


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_set_dgelsy.argtypes = [ctypes.c_void_p]
        L.orc_set_dgelsy(_scipy_dgelsy_ptr())
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i64(x):
    return ctypes.c_int64(int(x))


def _threads(nthreads):
    return int(nthreads) if nthreads else 1


# ------------------------------------------------------------------ rbf
def rbf_weights(kind, a, r_c, r):
    """_ext.pyx:65-75."""
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    out = np.empty(r.shape[0])
    if kind < 0 or kind > 7:
        raise ValueError(f"unknown rbf kind code {kind}")
    lib().orc_rbf(ctypes.c_int(kind), ctypes.c_double(a), ctypes.c_double(r_c), _p(r),
                  _i64(r.shape[0]), _p(out))
    return out


# --------------------------------------------------------------- search
def _grid_arrays(n, lo, d):
    n = np.ascontiguousarray(n, dtype=np.int64)
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    inv_d = np.ascontiguousarray(1.0 / np.asarray(d, dtype=np.float64))
    return n, lo, inv_d


def supports_nd(targets, grid, selection, nthreads=1):
    """Fixed (r_c float) or adaptive ((min_pts, r0, growth, r_max) tuple)
    radius supports on an OraclePointGrid; returns the reference tuple."""
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, grid.dim)
    return _supports(targets, grid.points, grid.n, grid.lo, grid.d, grid.cell_offsets,
                     grid.cell_items, selection, nthreads)


def _supports(targets, pts, n, lo, d, cell_off, cell_items, selection, nthreads):
    L = lib()
    dim = targets.shape[1]
    nt = targets.shape[0]
    n, lo, inv_d = _grid_arrays(n, lo, d)
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    cell_off = np.ascontiguousarray(cell_off, dtype=np.int64)
    cell_items = np.ascontiguousarray(cell_items, dtype=np.int64)
    counts = np.zeros(nt, dtype=np.int64)
    nth = _threads(nthreads)
    if isinstance(selection, tuple):
        min_pts, r0, growth, r_max = selection
        radii = np.zeros(nt, dtype=np.float64)
        status = np.zeros(nt, dtype=np.uint8)
        L.orc_adaptive_count(
            ctypes.c_int(dim), _p(targets), _i64(nt), _p(pts), _p(n), _p(lo), _p(inv_d),
            _p(cell_off), _p(cell_items), _i64(min_pts), ctypes.c_double(r0),
            ctypes.c_double(growth), ctypes.c_double(r_max), _p(counts), _p(radii),
            _p(status), ctypes.c_int(nth))
        r_c = 0.0
        radii_arg = _p(radii)
    else:
        r_c = float(selection)
        L.orc_fixed_count(ctypes.c_int(dim), _p(targets), _i64(nt), _p(pts), _p(n),
                          _p(lo), _p(inv_d), _p(cell_off), _p(cell_items),
                          ctypes.c_double(r_c), _p(counts), ctypes.c_int(nth))
        radii = None
        radii_arg = None
    offsets = np.zeros(nt + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    idx = np.empty(offsets[-1], dtype=np.int64)
    dist = np.empty(offsets[-1], dtype=np.float64)
    L.orc_fill(ctypes.c_int(dim), _p(targets), _i64(nt), _p(pts), _p(n), _p(lo),
               _p(inv_d), _p(cell_off), _p(cell_items), ctypes.c_double(r_c), radii_arg,
               _p(offsets), _p(idx), _p(dist), ctypes.c_int(nth))
    if radii is None:
        return offsets, idx, dist
    return offsets, idx, dist, radii, status


def fixed_radius_supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny, cell_off, cell_items,
                          r_c, nthreads=1):
    """_ext.pyx:203-235 (same signature)."""
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 2)
    return _supports(targets, pts, [nx, ny], [gx0, gy0], [gdx, gdy], cell_off,
                     cell_items, float(r_c), nthreads)


def adaptive_radius_supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny, cell_off,
                             cell_items, min_pts, r0, growth, r_max, nthreads=1):
    """_ext.pyx:238-288 (same signature)."""
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 2)
    return _supports(targets, pts, [nx, ny], [gx0, gy0], [gdx, gdy], cell_off,
                     cell_items, (int(min_pts), float(r0), float(growth), float(r_max)),
                     nthreads)


# ------------------------------------------------------------------ fit
def n_monomials(dim, degree):
    return int(lib().orc_n_monomials(ctypes.c_int(dim), ctypes.c_int(degree)))


def monomial_table(dim, degree):
    k = n_monomials(dim, degree)
    parent = np.zeros(k, dtype=np.int32)
    var = np.zeros(k, dtype=np.int32)
    deg = np.zeros(k, dtype=np.int32)
    lib().orc_monomial_table(ctypes.c_int(dim), ctypes.c_int(degree), _p(parent), _p(var),
                             _p(deg))
    return parent, var, deg


def fit_many_nd(targets, sup_off, sup_idx, sup_w, src, src_val, degree, lam, centering,
                nthreads=1):
    """_ext.pyx:291-426 generalised: src (ns, dim); src_val (ns,) or (ns, C).
    Returns values (nt,) / (nt, C), coeffs (nt, k) / (nt, C, k), status (nt,)."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    dim = src.shape[1]
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, dim)
    sv = np.ascontiguousarray(src_val, dtype=np.float64)
    scalar = sv.ndim == 1
    sv2 = sv.reshape(sv.shape[0], -1)
    ncomp = sv2.shape[1]
    nt = targets.shape[0]
    k = n_monomials(dim, degree)
    sup_off = np.ascontiguousarray(sup_off, dtype=np.int64)
    sup_idx = np.ascontiguousarray(sup_idx, dtype=np.int64)
    sup_w = np.ascontiguousarray(sup_w, dtype=np.float64)
    values = np.empty((nt, ncomp))
    coeffs = np.empty((nt, ncomp, k))
    status = np.zeros(nt, dtype=np.uint8)
    rc = lib().orc_fit_many(
        ctypes.c_int(dim), ctypes.c_int(degree), ctypes.c_double(lam),
        ctypes.c_int(1 if centering else 0), _p(targets), _i64(nt), _p(sup_off),
        _p(sup_idx), _p(sup_w), _p(src), _p(sv2), ctypes.c_int(ncomp), _p(values),
        _p(coeffs), _p(status), ctypes.c_int(_threads(nthreads)))
    if rc != 0:
        raise RuntimeError(f"oracle fit_many failed ({rc})")
    if scalar:
        return values[:, 0], coeffs[:, 0, :], status
    return values, coeffs, status


def fit_many(targets, sup_off, sup_idx, sup_w, src_xy, src_val, degree, lam, centering,
             nthreads=1):
    """_ext.pyx:291-426 (same signature, 2-D)."""
    return fit_many_nd(targets, sup_off, sup_idx, sup_w, src_xy, src_val, degree, lam,
                       centering, nthreads)


# ---------------------------------------------------- pipeline helpers
def rbf_for_supports(kind, a, off, dist, radius):
    """pointwise.py:179-183/250/266-269: weights at the effective cutoff
    (scalar fixed radius, or per-target radii)."""
    if kind == RBF_IDENTITY:
        return np.ones_like(dist)
    if np.ndim(radius) == 0:
        return rbf_weights(kind, a, float(radius), dist)
    off = np.ascontiguousarray(off, dtype=np.int64)
    dist = np.ascontiguousarray(dist, dtype=np.float64)
    radius = np.ascontiguousarray(radius, dtype=np.float64)
    w = np.empty_like(dist)
    if kind < 0 or kind > 7:
        raise ValueError(f"unknown rbf kind code {kind}")
    lib().orc_rbf_per_target(ctypes.c_int(kind), ctypes.c_double(a), _p(off),
                             _i64(off.shape[0] - 1), _p(radius), _p(dist), _p(w))
    return w


def r_max_for(points, targets):
    """pointwise.py:253-255 (any dim: hypot generalised to the 2-norm)."""
    span = np.vstack([points, targets])
    lo, hi = span.min(axis=0), span.max(axis=0)
    if span.shape[1] == 2:
        ext = float(np.hypot(hi[0] - lo[0], hi[1] - lo[1]))
    else:
        ext = float(np.sqrt(np.sum((hi - lo) ** 2)))
    return 1.0000001 * ext + 1e-300


def transfer(src, vals, targets, degree, kind, a, selection, lam=0.0, centering=True,
             nthreads=1):
    """Whole hot path on the CPU: grid -> supports -> weights -> fit.
    `selection` is ('fixed', r_c) or ('adaptive', min_pts, r0, growth).
    Returns (values, status, (off, idx, dist, w))."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, src.shape[1])
    grid = OraclePointGrid(src)
    if selection[0] == "fixed":
        off, idx, dist = supports_nd(targets, grid, float(selection[1]), nthreads)
        radius = float(selection[1])
    else:
        _, min_pts, r0, growth = selection
        off, idx, dist, radii, _st = supports_nd(
            targets, grid, (int(min_pts), float(r0), float(growth), r_max_for(src, targets)),
            nthreads)
        radius = radii
    w = np.abs(rbf_for_supports(kind, a, off, dist, radius))
    values, _c, status = fit_many_nd(targets, off, idx, w, src, vals, degree, lam,
                                     centering, nthreads)
    return values, status, (off, idx, dist, w)


def locate_batch(points, tri_xy, tri_verts, tri_edges, vert_gid, tri_gid, inv2a, epsfac,
                 gx0, gy0, gdx, gdy, nx, ny, cell_off, cell_items, tol):
    """_ext.pyx:88-152 (same signature and outputs as the reference)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    found = np.zeros(n, dtype=np.uint8)
    elem = np.full(n, -1, dtype=np.int64)
    dim = np.full(n, -1, dtype=np.int64)
    ent = np.full(n, -1, dtype=np.int64)
    bary = np.full((n, 3), np.nan, dtype=np.float64)
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
    a = [f64(tri_xy), i64(tri_verts), i64(tri_edges), i64(vert_gid), i64(tri_gid), f64(inv2a),
         f64(epsfac), i64(cell_off), i64(cell_items)]
    L = lib()
    L.orc_locate_batch(_p(pts), ctypes.c_int64(n), _p(a[0]), _p(a[1]), _p(a[2]), _p(a[3]),
                       _p(a[4]), _p(a[5]), _p(a[6]), ctypes.c_double(gx0), ctypes.c_double(gy0),
                       ctypes.c_double(gdx), ctypes.c_double(gdy), ctypes.c_int64(nx),
                       ctypes.c_int64(ny), _p(a[7]), _p(a[8]), ctypes.c_double(tol), _p(found),
                       _p(elem), _p(dim), _p(ent), _p(bary))
    return found.astype(bool), elem, dim, ent, bary


def patch_supports(seed, edge_tris, tris, layers, centroids):
    """Element-patch supports (pointwise.py:190-230, _select_batch's patch
    branch 271-296): per seed element, the elements within `layers` hops over
    interior-edge adjacency (both directions, 195-200), sorted (226); dofs are
    those elements (centroids) or np.unique of their vertices (229).  Plain
    Python BFS -- small cases only.  Returns (offsets int64 (nt+1), idx int64)."""
    et = np.asarray(edge_tris, dtype=np.int64)
    interior = et[:, 1] >= 0
    nbrs = {}
    for a, b in zip(et[interior, 0].tolist(), et[interior, 1].tolist()):
        nbrs.setdefault(a, []).append(b)
        nbrs.setdefault(b, []).append(a)
    tris = np.asarray(tris, dtype=np.int64)
    off = [0]
    parts = []
    for s in np.asarray(seed, dtype=np.int64).tolist():
        seen = {s}
        frontier = [s]
        for _ in range(layers):
            nxt = []
            for t in frontier:
                for nb in nbrs.get(t, ()):
                    if nb not in seen:
                        seen.add(nb)
                        nxt.append(nb)
            frontier = nxt
        elems = np.array(sorted(seen), dtype=np.int64)
        dofs = elems if centroids else np.unique(tris[elems].reshape(-1))
        parts.append(dofs)
        off.append(off[-1] + dofs.size)
    idx = np.concatenate(parts) if parts else np.empty(0, np.int64)
    return np.array(off, dtype=np.int64), idx.astype(np.int64)
