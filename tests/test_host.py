"""CPU: host-side logic of the package -- spec validation (pointwise.py:75-161),
grid geometry (locate.py:34-62), synthetic inputs, error labels."""

import numpy as np
import pytest

from conftest import golden
from paper_2510_18838_b200 import pointwise as P
from paper_2510_18838_b200 import synth
from paper_2510_18838_b200.locate import PointGrid, grid_geometry


def test_spec_validation_mirrors_reference():
    with pytest.raises(ValueError):
        P.RadialBasisSpec(P.RbfKind.C4, a=0.0)
    with pytest.raises(ValueError):
        P.RadialBasisSpec(P.RbfKind.C4, r_c=-1.0)
    with pytest.raises(ValueError):
        P.FixedRadius(0.0)
    with pytest.raises(ValueError):
        P.AdaptiveRadius(0, 0.1)
    with pytest.raises(ValueError):
        P.AdaptiveRadius(3, 0.0)
    with pytest.raises(ValueError):
        P.AdaptiveRadius(3, 0.1, growth=1.0)
    with pytest.raises(ValueError):
        P.ElementPatch(0)
    rbf = P.RadialBasisSpec(P.RbfKind.C4)
    with pytest.raises(ValueError):
        P.FitSpec(4, rbf, P.FixedRadius(1.0))
    with pytest.raises(ValueError):
        P.FitSpec(1, rbf, P.FixedRadius(1.0), lam=-1.0)
    with pytest.raises(TypeError):
        P.FitSpec(1, rbf, "radius")
    with pytest.raises(ValueError):
        P.FitSpec(2, rbf, P.AdaptiveRadius(5, 0.1))  # 6 monomials
    P.FitSpec(3, rbf, P.AdaptiveRadius(10, 0.1))  # degree 3: extension


def test_n_monomials():
    assert [P.n_monomials(d) for d in range(4)] == [1, 3, 6, 10]
    assert P.n_monomials(3, dim=3) == 20
    assert P.n_monomials(2, dim=5) == 21


def test_grid_geometry_is_the_reference_pointgrid():
    g = golden("disk_small")
    pts = g["coords"]
    geom = grid_geometry(pts.min(axis=0), pts.max(axis=0), pts.shape[0])
    assert np.array_equal(geom.lo, g["grid_lo"])
    assert np.array_equal(np.array(geom.n), g["grid_n"])
    assert np.array_equal(geom.d, g["grid_d"])
    pg = PointGrid(pts)
    assert (pg.nx, pg.ny) == tuple(g["grid_n"])
    assert (pg.dx, pg.dy) == tuple(g["grid_d"])


def test_grid_geometry_degenerate_and_nd():
    geom = grid_geometry(np.array([0.0, 1.0]), np.array([0.0, 1.0]), 1)
    assert geom.n == (1, 1)
    geom = grid_geometry(np.zeros(5), np.ones(5), 100000)
    assert geom.dim == 5 and 30000 < geom.ncell < 300000
    with pytest.raises(ValueError):
        PointGrid(np.zeros((0, 2)))


def test_synth_matches_reference_meshes():
    g = golden("disk_small")
    m = synth.disk(1.0, 8)
    assert np.array_equal(m.coords, g["coords"])
    assert np.array_equal(m.tris, g["tris"])
    assert np.array_equal(m.centroids(), g["centroids"])
    assert m.mean_edge_length == float(g["mean_edge_length"])
    assert synth.square(99).mean_edge_length == float(golden("c1")["mean_edge_length"])
    assert synth.disk_graded(1.0, 30, 0.6).mean_edge_length == float(
        golden("adaptive")["mean_edge_length"])


def test_point_label_and_r_max():
    pts = np.array([[0.5, 0.25], [1.0, 2.0]])
    assert P._point_label(pts, 1) == "target 1 at (1, 2)"
    r = P._r_max(np.array([[0.0, 0.0]]), np.array([[3.0, 4.0]]))
    assert r == 1.0000001 * 5.0 + 1e-300


def test_element_patch_rejects_point_clouds_without_gpu():
    # pointwise.py:360-370: the FieldError comes before any device work
    src = np.random.RandomState(4).uniform(0, 1, size=(30, 2))
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.CONST), P.ElementPatch(1))
    with pytest.raises(P.FieldError):
        P.fit_point_cloud(src, np.ones(30), [(0.5, 0.5)], spec)


def test_fit_point_cloud_input_errors_without_gpu():
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(0.1))
    with pytest.raises(P.InsufficientSourcesError):
        P.fit_point_cloud(np.zeros((0, 2)), np.zeros(0), [(0.5, 0.5)], spec)
    with pytest.raises(P.FieldError):
        P.fit_point_cloud(np.zeros((3, 2)), np.zeros(2), [(0.5, 0.5)], spec)


def test_eval_rbf_argument_errors_without_gpu():
    with pytest.raises(ValueError):
        P.eval_rbf(P.RadialBasisSpec(P.RbfKind.C4, r_c=1.0), -0.1)
    with pytest.raises(ValueError):
        P.eval_rbf(P.RadialBasisSpec(P.RbfKind.C4), 0.1)
    assert P.eval_rbf(P.RadialBasisSpec(P.RbfKind.IDENTITY), 123.0) == 1.0
