import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfieldmap.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def disk_small():
    from paper_2510_18838_b200 import synth

    return synth.disk(1.0, 8)  # 217 vertices, 384 elements (reference conftest.py:21-23)


class PointField:
    """Duck-typed stand-in for the reference's Field (mesh.py:269-309): the
    hot path only reads dof_points(), values, mesh and location."""

    def __init__(self, mesh, values, location="vertices"):
        self.mesh = None  # point-cloud sources (ElementPatch not used here)
        self._pts = mesh.coords if location == "vertices" else mesh.centroids()
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.location = location

    def dof_points(self):
        return self._pts

    def with_values(self, values):
        f = PointField.__new__(PointField)
        f.mesh, f._pts, f.location = self.mesh, self._pts, self.location
        f.values = np.ascontiguousarray(values, dtype=np.float64)
        return f


def sample_field(mesh, fn, location="vertices"):
    pts = mesh.coords if location == "vertices" else mesh.centroids()
    return PointField(mesh, np.asarray(fn(pts[:, 0], pts[:, 1]), dtype=np.float64), location)
