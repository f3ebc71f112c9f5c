"""Drop-in for the reference's kernel seam `fieldbridge._kernels`.

The reference binds these names to its Cython extension or numpy fallback
(_kernels/__init__.py:9-42).  Here they keep the exact signatures, argument
meaning, dtypes and return layout of _ext.pyx (65, 203-207, 238-243,
291-293) but run on the B200 through libfieldmap.so: host numpy in, host
numpy out, device in between.  A maintainer can therefore do

    import fieldbridge._kernels as K
    from paper_2510_18838_b200 import _kernels as B
    for name in ("rbf_weights", "fixed_radius_supports",
                 "adaptive_radius_supports", "fit_many"):
        setattr(K, name, getattr(B, name))

and the reference's pointwise/locate code (which resolves `_kernels.<fn>`
at call time, pointwise.py:17, 240, 256, 302) runs on the GPU (see
INTEGRATION.md).  `locate_batch` (element localization, the seam's other
search export) is here too, bitwise equal to
_ext.pyx:88-152; `clip_batch` (conservative transfer) is OUT.

fixed/adaptive_radius_supports receive the caller's grid geometry and use
it for the device grid; the caller's host CSR (cell_off, cell_items) is not
needed because the device rebuilds it (results do not depend on it).
"""

import numpy as np
import torch

from . import device as D
from .locate import GridGeometry

BACKEND = "b200"

# RBF kind codes and fit status codes (_ext.pyx:18-29)
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


def rbf_weights(kind, a, r_c, r):
    """Evaluate the radial weight for distances ``r`` (cutoff at r > r_c)."""
    r_arr = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
    if kind < 0 or kind > 7:
        raise ValueError(f"unknown rbf kind code {kind}")
    if r_arr.shape[0] == 0:
        return np.empty(0)
    out = D.rbf_weights(kind, a, r_c, D.to_device(r_arr))
    return out.cpu().numpy()


def _cloud_from_ref_grid(pts, gx0, gy0, gdx, gdy, nx, ny):
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    geom = GridGeometry(2, (int(nx), int(ny)), np.array([gx0, gy0], dtype=np.float64),
                        np.array([gx0 + nx * gdx, gy0 + ny * gdy], dtype=np.float64),
                        np.array([gdx, gdy], dtype=np.float64))
    return D.SourceCloud(pts, geom=geom)


def _supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny, sel):
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 2)
    if targets.shape[0] == 0:
        return None, np.zeros(1, np.int64), np.empty(0, np.int64), np.empty(0)
    cloud = _cloud_from_ref_grid(pts, gx0, gy0, gdx, gdy, nx, ny)
    t = D.to_device(targets)
    perm = cloud.target_order(t)
    cnt = D.count_supports(cloud, t, sel, perm)
    idx, dist, _ = D.fill_supports(cloud, t, sel, cnt, perm)
    return cnt, cnt.offsets.cpu().numpy(), idx.cpu().numpy(), dist.cpu().numpy()


def fixed_radius_supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny, cell_off, cell_items, r_c):
    """Per-target source ids with distance < r_c, ids ascending (_ext.pyx:203-235)."""
    _, off, idx, dist = _supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny, D.fixed(r_c))
    return off, idx, dist


def adaptive_radius_supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny, cell_off, cell_items,
                             min_pts, r0, growth, r_max):
    """Grow the radius geometrically until min_pts sources fall inside (_ext.pyx:238-288)."""
    cnt, off, idx, dist = _supports(targets, pts, gx0, gy0, gdx, gdy, nx, ny,
                                    D.adaptive(min_pts, r0, growth, r_max))
    if cnt is None:
        return off, idx, dist, np.zeros(0), np.zeros(0, np.uint8)
    return off, idx, dist, cnt.radii.cpu().numpy(), cnt.status.cpu().numpy()


def fit_many(targets, sup_off, sup_idx, sup_w, src_xy, src_val, degree, lam, centering):
    """Weighted ridge polynomial fit per target (_ext.pyx:291-426)."""
    src_xy = np.ascontiguousarray(src_xy, dtype=np.float64)
    dim = src_xy.shape[1] if src_xy.ndim == 2 else 2
    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, dim)
    sup_off = np.ascontiguousarray(sup_off, dtype=np.int64)
    nt = targets.shape[0]
    from . import _lib

    k = _lib.lib().fm_n_monomials(dim, int(degree))
    if nt == 0:
        return np.empty(0), np.empty((0, k)), np.empty(0, np.uint8)
    max_m = int(np.max(np.diff(sup_off))) if nt else 0
    values, coeffs, status, _ = D.fit_many(
        D.to_device(targets), torch.from_numpy(sup_off).to(D._dev()),
        torch.from_numpy(np.ascontiguousarray(sup_idx, dtype=np.int64)).to(D._dev()),
        D.to_device(np.ascontiguousarray(sup_w, dtype=np.float64)), D.to_device(src_xy),
        D.to_device(np.ascontiguousarray(src_val, dtype=np.float64)), int(degree), float(lam),
        bool(centering), max_m)
    return values.cpu().numpy(), coeffs.cpu().numpy(), status.cpu().numpy()


def locate_batch(points, tri_xy, tri_verts, tri_edges, vert_gid, tri_gid, inv2a, epsfac,
                 gx0, gy0, gdx, gdy, nx, ny, cell_off, cell_items, tol):
    """Grid-accelerated point localization with entity classification
    (_ext.pyx:88-152): (found bool, elem, dim, ent int64, bary (n, 3) f64)."""
    from . import _lib as L

    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    n = pts.shape[0]
    if n == 0:
        return (np.zeros(0, dtype=bool), np.full(0, -1, np.int64), np.full(0, -1, np.int64),
                np.full(0, -1, np.int64), np.full((0, 3), np.nan))
    f64 = lambda a: D.to_device(np.ascontiguousarray(a, dtype=np.float64))  # noqa: E731
    i64 = lambda a: torch.from_numpy(  # noqa: E731
        np.ascontiguousarray(a, dtype=np.int64)).to(D._dev())
    dev = [f64(pts), f64(tri_xy), i64(tri_verts), i64(tri_edges), i64(vert_gid), i64(tri_gid),
           f64(inv2a), f64(epsfac), i64(cell_off), i64(cell_items)]
    found = torch.empty(n, dtype=torch.uint8, device=dev[0].device)
    elem = torch.empty(n, dtype=torch.int64, device=dev[0].device)
    dim = torch.empty_like(elem)
    ent = torch.empty_like(elem)
    bary = torch.empty((n, 3), dtype=torch.float64, device=dev[0].device)
    P = L.ptr
    L.check(L.lib().fm_locate_batch(P(dev[0]), n, *[P(a) for a in dev[1:8]], float(gx0),
                                    float(gy0), float(gdx), float(gdy), int(nx), int(ny),
                                    P(dev[8]), P(dev[9]), float(tol), P(found), P(elem), P(dim),
                                    P(ent), P(bary), D._stream()), "fm_locate_batch")
    return (found.cpu().numpy().astype(bool), elem.cpu().numpy(), dim.cpu().numpy(),
            ent.cpu().numpy(), bary.cpu().numpy())


def patch_supports(seed, tris, edge_tris, layers, centroids):
    """ElementPatch support CSR for seed elements (the loop of _select_batch's
    patch branch over _PatchTopology.patch_dofs, pointwise.py:212-230,
    286-296): (offsets int64 (nt+1), idx int64, counts int64 (nt)), computed
    by fm_patch_count / fm_patch_fill.  A patch larger than the kernel's
    per-target bound raises FieldmapError."""
    from ._lib import FieldmapError

    topo = D.PatchTopology.from_mesh_arrays(np.ascontiguousarray(tris, dtype=np.int64),
                                            np.ascontiguousarray(edge_tris, dtype=np.int64))
    off, idx, counts = D.patch_supports(topo, np.ascontiguousarray(seed, dtype=np.int64),
                                        layers, centroids)
    counts = counts.cpu().numpy()
    if (counts < 0).any():
        i = int(np.argmax(counts < 0))
        if counts[i] == -2:
            raise ValueError(f"seed of target {i} is not an element id (not located?)")
        raise FieldmapError(f"element patch of target {i} exceeds the kernel's per-target "
                            "bound (FM_PATCH_MAX_ELEMS / FM_PATCH_MAX_DOFS)")
    return off.cpu().numpy(), idx.cpu().numpy(), counts
