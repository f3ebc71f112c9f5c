"""Synthetic point clouds of the shapes the benchmark configs name.

Restates the coordinate part of the reference's mesh generators
(/root/reference/pkg/src/fieldbridge/generate.py) so the bench and the GPU
tests can build the C1/C2 inputs on a box without the reference:

  square(n)                      generate.py:28-44
  disk(radius, n_rings)          generate.py:47-80 (_disk_rings), 83-88
  disk_graded(radius, n, expo)   generate.py:91-101
  centroids / mean_edge_length   mesh.py:95 (`(p0 + p1 + p2) / 3.0`),
                                 mesh.py:128-131, build_mesh edge table
                                 mesh.py:220-224, CW re-orientation 186-192

The loops are vectorised, but every float is produced by the same IEEE
operation sequence as the reference (ring angles with math.cos/math.sin),
so coordinates, centroids and the mean edge length are bitwise equal to the
reference's (tests/test_synth.py pins them against tests/golden/).
"""

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class PointMesh:
    """Vertex coordinates plus CCW triangles (only what the hot path reads)."""

    coords: np.ndarray
    tris: np.ndarray

    @property
    def nverts(self):
        return self.coords.shape[0]

    @property
    def nelems(self):
        return self.tris.shape[0]

    def centroids(self):
        p0 = self.coords[self.tris[:, 0]]
        p1 = self.coords[self.tris[:, 1]]
        p2 = self.coords[self.tris[:, 2]]
        return np.ascontiguousarray((p0 + p1 + p2) / 3.0)

    @property
    def edges(self):
        t = self.tris
        raw = np.concatenate([t[:, [1, 2]], t[:, [2, 0]], t[:, [0, 1]]])
        raw = np.sort(raw, axis=1)
        # lexicographic unique rows (np.unique(axis=0) order) via 1-D keys
        nv = np.int64(self.nverts)
        key = np.unique(raw[:, 0] * nv + raw[:, 1])
        return np.column_stack([key // nv, key % nv])

    @property
    def mean_edge_length(self):
        p = self.coords[self.edges]
        return float(np.linalg.norm(p[:, 1] - p[:, 0], axis=1).mean())


def _orient_ccw(coords, tris):
    p0, p1, p2 = (coords[tris[:, k]] for k in range(3))
    signed = 0.5 * ((p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1])
                    - (p1[:, 1] - p0[:, 1]) * (p2[:, 0] - p0[:, 0]))
    cw = signed < 0
    if cw.any():
        tris = tris.copy()
        tris[cw] = tris[cw][:, [0, 2, 1]]
    return tris


def square(n):
    """generate.py:28-44: unit square, (n+1)^2 vertices, 2n^2 triangles."""
    side = np.linspace(0.0, 1.0, n + 1)
    xx, yy = np.meshgrid(side, side)
    coords = np.column_stack([xx.reshape(-1), yy.reshape(-1)])
    j, i = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v00 = (j * (n + 1) + i).reshape(-1)
    v10 = v00 + 1
    v01 = v00 + (n + 1)
    v11 = v01 + 1
    tris = np.empty((2 * n * n, 3), dtype=np.int64)
    tris[0::2] = np.column_stack([v00, v10, v11])
    tris[1::2] = np.column_stack([v00, v11, v01])
    return PointMesh(np.ascontiguousarray(coords), _orient_ccw(coords, tris))


def _disk_rings(n_rings, ring_radius):
    k = n_rings
    nv = 1 + 3 * k * (k + 1)
    coords = np.empty((nv, 2), dtype=np.float64)
    coords[0] = (0.0, 0.0)
    ring_start = np.zeros(k + 1, dtype=np.int64)
    pos = 1
    cos, sin, pi = math.cos, math.sin, math.pi
    for i in range(1, k + 1):
        ring_start[i] = pos
        r = ring_radius(i)
        m = 6 * i
        # `2.0 * math.pi * j / m` and math.cos/sin exactly as generate.py:56-57
        ang = [2.0 * pi * j / m for j in range(m)]
        coords[pos:pos + m, 0] = [r * cos(a) for a in ang]
        coords[pos:pos + m, 1] = [r * sin(a) for a in ang]
        pos += m
    parts = []
    for i in range(1, k + 1):
        outer = ring_start[i]
        mo = 6 * i
        inner = ring_start[i - 1]
        mi = 6 * (i - 1)
        s = np.repeat(np.arange(6), i)
        t = np.tile(np.arange(i), 6)
        o0 = outer + (s * i + t) % mo
        o1 = outer + (s * i + t + 1) % mo
        n0 = np.full_like(o0, inner) if i == 1 else inner + (s * (i - 1) + t) % mi
        blk = np.full((6 * i, 2, 3), -1, dtype=np.int64)
        blk[:, 0] = np.column_stack([o0, o1, n0])
        if i > 1:
            n1 = inner + (s * (i - 1) + t + 1) % mi
            has_b = t < i - 1
            blk[has_b, 1] = np.column_stack([n0, o1, n1])[has_b]
        blk = blk.reshape(-1, 3)
        parts.append(blk[blk[:, 0] >= 0])
    tris = np.concatenate(parts)
    return PointMesh(coords, _orient_ccw(coords, tris))


def disk(radius=1.0, n_rings=4):
    """generate.py:83-88."""
    return _disk_rings(n_rings, lambda i: radius * i / n_rings)


def disk_graded(radius=1.0, n_rings=4, exponent=0.6):
    """generate.py:91-101."""
    return _disk_rings(n_rings, lambda i: radius * (i / n_rings) ** exponent)


def sincos_field(coords, ncomp=1):
    """f_c = sin((c+1) x) cos(y) + 2 (config.py:29-30 for c = 0); (n, C)."""
    x = coords[:, 0]
    y = coords[:, 1]
    out = np.empty((coords.shape[0], ncomp), dtype=np.float64)
    for c in range(ncomp):
        out[:, c] = np.sin((c + 1) * x) * np.cos(y) + 2.0
    return out
