"""Source grid geometry and the PointGrid drop-in (a1 host side).

The reference's PointGrid (locate.py:144-161) is built with numpy on the
host.  Here the host only decides the geometry -- padded bbox (_pad_bbox,
locate.py:50-62) and cell counts (_grid_shape, locate.py:34-47), identical
formulas for dim 2 -- and the binning itself (cell keys, counting sort,
in-cell id order) runs on the device in fm_grid_build.

`PointGrid` / `build_point_grid` keep the reference's attribute surface
(lo, hi, nx, ny, dx, dy, points, cell_offsets, cell_items) for callers that
pass a grid into fit_point_cloud / PreparedTransfer; the CSR arrays are
materialised lazily from the device grid.
"""

from dataclasses import dataclass

import numpy as np

from ._lib import FM_MAX_DIM, FmGrid


def _grid_shape_2d(lo, hi, n_items, per_item):
    """locate.py:34-47."""
    w = max(hi[0] - lo[0], 0.0)
    h = max(hi[1] - lo[1], 0.0)
    target = max(1.0, per_item * n_items)
    if w <= 0.0 and h <= 0.0:
        return 1, 1
    if w <= 0.0:
        return 1, max(1, int(round(target)))
    if h <= 0.0:
        return max(1, int(round(target))), 1
    nx = max(1, int(round(np.sqrt(target * w / h))))
    ny = max(1, int(round(target / nx)))
    return nx, ny


def _pad_bbox(lo, hi):
    """locate.py:50-62 (any number of axes)."""
    lo = np.asarray(lo, dtype=float).copy()
    hi = np.asarray(hi, dtype=float).copy()
    span = max(float(np.max(hi - lo)), 1.0)
    pad = 1e-12 * span
    for k in range(lo.size):
        if hi[k] - lo[k] <= 0.0:
            lo[k] -= 0.5 * max(span, 1.0)
            hi[k] += 0.5 * max(span, 1.0)
        else:
            lo[k] -= pad
            hi[k] += pad
    return lo, hi


@dataclass(frozen=True)
class GridGeometry:
    dim: int
    n: tuple
    lo: np.ndarray
    hi: np.ndarray
    d: np.ndarray

    @property
    def ncell(self):
        return int(np.prod(self.n))

    @property
    def inv_d(self):
        return 1.0 / self.d

    def to_ctypes(self):
        g = FmGrid()
        g.dim = self.dim
        for a in range(FM_MAX_DIM):
            g.n[a] = int(self.n[a]) if a < self.dim else 1
            g.lo[a] = float(self.lo[a]) if a < self.dim else 0.0
            g.inv_d[a] = float(1.0 / self.d[a]) if a < self.dim else 1.0
        g.ncell = self.ncell
        return g


def grid_geometry(bbox_lo, bbox_hi, n_points, cells_per_point=1.0):
    """Geometry of the PointGrid the reference would build (dim 2), or its
    isotropic generalisation (cells of equal side) for other dims."""
    if cells_per_point <= 0:
        raise ValueError("cells_per_point must be > 0")
    lo, hi = _pad_bbox(bbox_lo, bbox_hi)
    dim = lo.size
    if dim == 2:
        shape = _grid_shape_2d(lo, hi, n_points, cells_per_point)
    else:
        target = max(1.0, cells_per_point * n_points)
        ext = hi - lo
        side = (float(np.prod(ext)) / target) ** (1.0 / dim)
        shape = tuple(max(1, int(round(e / side))) for e in ext)
    n = np.asarray(shape, dtype=np.int64)
    # locate.py:75-76: dx = (hi - lo) / nx
    d = np.array([(hi[a] - lo[a]) / n[a] for a in range(dim)], dtype=np.float64)
    return GridGeometry(dim, tuple(int(x) for x in n), lo, hi, d)


class PointGrid:
    """Bucket grid over a point cloud for radius queries (locate.py:144-161).

    Device-built; the host CSR attributes are computed on first access."""

    def __init__(self, points, cells_per_point=1.0):
        points = np.ascontiguousarray(points, dtype=np.float64)
        if points.ndim != 2 or points.shape[1] != 2 or points.shape[0] == 0:
            raise ValueError("points must be a nonempty (n, 2) array")
        self.points = points
        self.cells_per_point = cells_per_point
        self.geom = grid_geometry(points.min(axis=0), points.max(axis=0), points.shape[0],
                                  cells_per_point)
        self.lo = self.geom.lo
        self.hi = self.geom.hi
        self.nx, self.ny = self.geom.n
        self.dx, self.dy = float(self.geom.d[0]), float(self.geom.d[1])
        self._cloud = None

    def cloud(self):
        """The device-resident SourceCloud for this grid (built once)."""
        if self._cloud is None:
            from .device import SourceCloud

            self._cloud = SourceCloud(self.points, self.cells_per_point,
                                      bbox=(self.points.min(axis=0), self.points.max(axis=0)))
        return self._cloud

    @property
    def bbox(self):
        return np.array([self.lo, self.hi])

    @property
    def cell_offsets(self):
        return self.cloud().cell_start.to("cpu").numpy().astype(np.int64)

    @property
    def cell_items(self):
        return self.cloud().sorted_ids.to("cpu").numpy().astype(np.int64)


def build_point_grid(points, cells_per_point=1.0):
    """locate.py:171-172."""
    return PointGrid(points, cells_per_point)


# locate.py:31: element bboxes are padded by this fraction of the diameter
BBOX_PAD_REL = 1e-9


class ElementGrid:
    """The reference's element acceleration grid (`UniformGrid` /
    `build_grid`, locate.py:111-141, 164-168, CSR layout 65-84), built with
    tensor ops on the device: each element enters every cell its padded bbox
    overlaps; cells row-major (iy*nx + ix), items ascending per cell.  Same
    geometry and arithmetic as the reference, so `fm_locate_batch` on it
    returns what the reference's `locate_arrays` returns."""

    def __init__(self, mesh, cells_per_element=1.0, device=None):
        import torch

        if cells_per_element <= 0:
            raise ValueError("cells_per_element must be > 0")
        bbox = np.asarray(mesh.bbox, dtype=np.float64)
        lo, hi = _pad_bbox(bbox[0], bbox[1])
        nx, ny = _grid_shape_2d(lo, hi, int(mesh.tri_xy.shape[0]), cells_per_element)
        self.lo, self.hi, self.nx, self.ny = lo, hi, nx, ny
        self.dx = (hi[0] - lo[0]) / nx
        self.dy = (hi[1] - lo[1]) / ny
        self.mesh = mesh
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(np.array(mesh.tri_xy, dtype=np.float64), device=dev)
        pad = BBOX_PAD_REL * torch.as_tensor(
            np.array(mesh.diameters, dtype=np.float64), device=dev)

        def span(axis, d, n):
            c = t[:, :, axis]
            c0 = ((c.amin(dim=1) - pad - float(lo[axis])) / d).to(torch.int64).clamp(0, n - 1)
            c1 = ((c.amax(dim=1) + pad - float(lo[axis])) / d).to(torch.int64).clamp(0, n - 1)
            return c0, c1

        ex0, ex1 = span(0, self.dx, nx)
        ey0, ey1 = span(1, self.dy, ny)
        wx = ex1 - ex0 + 1
        counts = wx * (ey1 - ey0 + 1)
        ne = t.shape[0]
        items = torch.repeat_interleave(torch.arange(ne, device=dev), counts)
        start = torch.cumsum(counts, 0) - counts
        k = torch.arange(items.shape[0], device=dev) - start[items]
        cells = (ey0[items] + k // wx[items]) * nx + ex0[items] + k % wx[items]
        # (cell, id) order: entries are generated in ascending id, so a stable
        # sort by cell is the reference's lexsort (locate.py:79)
        order = torch.argsort(cells, stable=True)
        self.cell_items = items[order].contiguous()
        off = torch.zeros(nx * ny + 1, dtype=torch.int64, device=dev)
        torch.cumsum(torch.bincount(cells, minlength=nx * ny), 0, out=off[1:])
        self.cell_offsets = off
