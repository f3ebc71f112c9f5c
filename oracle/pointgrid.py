"""CPU restatement of the reference's source binning (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product path never does.

Restates /root/reference/pkg/src/fieldbridge/locate.py:
  _grid_shape  locate.py:34-47
  _pad_bbox    locate.py:50-62
  _CsrGrid     locate.py:65-99   (lexsort by (cell, id), add.at + cumsum)
  PointGrid    locate.py:144-161 (cells_per_point = 1)

For dim == 2 the geometry and the CSR are identical to the reference's
PointGrid (pinned in tests/test_oracle.py).  dim != 2 is an extension
(the reference rejects it, locate.py:149-150): the padded bbox is split
into cells of equal side (volume / target)^(1/dim).
"""

import numpy as np


def grid_shape_2d(lo, hi, n_items, per_item):
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


def pad_bbox(lo, hi):
    """locate.py:50-62, for any number of axes."""
    lo = np.asarray(lo, dtype=float).copy()
    hi = np.asarray(hi, dtype=float).copy()
    span = max(max(hi - lo), 1.0)
    pad = 1e-12 * span
    for k in range(lo.size):
        if hi[k] - lo[k] <= 0.0:
            lo[k] -= 0.5 * max(span, 1.0)
            hi[k] += 0.5 * max(span, 1.0)
        else:
            lo[k] -= pad
            hi[k] += pad
    return lo, hi


class OraclePointGrid:
    """locate.py:144-161 (PointGrid) restated; `dim` may be 1..5."""

    def __init__(self, points, cells_per_point=1.0):
        points = np.ascontiguousarray(points, dtype=np.float64)
        if points.ndim != 2 or points.shape[0] == 0:
            raise ValueError("points must be a nonempty (n, d) array")
        self.dim = points.shape[1]
        lo, hi = pad_bbox(points.min(axis=0), points.max(axis=0))
        n = points.shape[0]
        if self.dim == 2:
            shape = grid_shape_2d(lo, hi, n, cells_per_point)
        else:
            target = max(1.0, cells_per_point * n)
            ext = hi - lo
            side = (np.prod(ext) / target) ** (1.0 / self.dim)
            shape = tuple(max(1, int(round(e / side))) for e in ext)
        self.n = np.asarray(shape, dtype=np.int64)
        self.lo = lo
        self.hi = hi
        self.d = (hi - lo) / self.n
        self.inv_d = 1.0 / self.d
        ncell = int(np.prod(self.n))
        # locate.py:155-158: cell = trunc((p - lo) / d) clipped, axis 0 fastest
        cells = np.zeros(n, dtype=np.int64)
        stride = 1
        for a in range(self.dim):
            ia = np.clip(((points[:, a] - lo[a]) / self.d[a]).astype(np.int64), 0,
                         self.n[a] - 1)
            cells += ia * stride
            stride *= int(self.n[a])
        items = np.arange(n, dtype=np.int64)
        order = np.lexsort((items, cells))  # locate.py:79
        cells = cells[order]
        self.cell_items = np.ascontiguousarray(items[order])
        self.cell_offsets = np.zeros(ncell + 1, dtype=np.int64)
        np.add.at(self.cell_offsets, cells + 1, 1)
        np.cumsum(self.cell_offsets, out=self.cell_offsets)
        self.points = points

    # 2-D attribute names of the reference's _CsrGrid (locate.py:68)
    @property
    def nx(self):
        return int(self.n[0])

    @property
    def ny(self):
        return int(self.n[1])

    @property
    def dx(self):
        return float(self.d[0])

    @property
    def dy(self):
        return float(self.d[1])
