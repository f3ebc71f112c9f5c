"""CPU: pin the oracle (oracle/fb_oracle.c + oracle/pointgrid.py) against the
reference's own outputs (tests/golden, made by tests/golden/make_golden.py)
and, when oracle/_ref is built, against the reference's compiled _ext."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from oracle import ref
from oracle.pointgrid import OraclePointGrid
from paper_2510_18838_b200 import synth


def test_rbf_table_bitwise():
    g = golden("rbf")
    for kind in range(8):
        assert np.array_equal(O.rbf_weights(kind, 2.0, 0.7, g["r"]), g[f"w{kind}"]), kind


def test_pointgrid_matches_reference_grid():
    g = golden("disk_small")
    pg = OraclePointGrid(g["coords"])
    assert np.array_equal(pg.lo, g["grid_lo"])
    assert np.array_equal(pg.n, g["grid_n"])
    assert np.array_equal(pg.d, g["grid_d"])
    assert np.array_equal(pg.cell_offsets, g["cell_offsets"])
    assert np.array_equal(pg.cell_items, g["cell_items"])


def test_radius_query_bitwise_disk_small():
    # reference test_locate.py:128-141
    g = golden("disk_small")
    pg = OraclePointGrid(g["coords"])
    t = np.ascontiguousarray(g["centroids"][:50])
    off, idx, dist = O.fixed_radius_supports(t, pg.points, pg.lo[0], pg.lo[1], pg.dx, pg.dy,
                                             pg.nx, pg.ny, pg.cell_offsets, pg.cell_items, 0.3)
    assert np.array_equal(off, g["rq_off"])
    assert np.array_equal(idx, g["rq_idx"])
    assert np.array_equal(dist, g["rq_dist"])


def _c1_inputs():
    m = synth.square(99)
    src = m.coords
    tg = np.random.RandomState(0).uniform(0, 1, (10000, 2))
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    return src, tg, vals


def test_c1_supports_and_values_bitwise():
    g = golden("c1")
    src, tg, vals = _c1_inputs()
    h = float(g["mean_edge_length"])
    got, st, (off, idx, dist, w) = O.transfer(src, vals, tg, 2, O.RBF_C4, 2.0, ("fixed", 2 * h),
                                               nthreads=4)
    assert (st == 0).all()
    assert np.array_equal(np.diff(off), g["counts"].astype(np.int64))
    assert off[-1] == int(g["nnz"])
    k = int(g["off1000"][-1])
    assert np.array_equal(idx[:k], g["idx1000"])
    assert np.array_equal(dist[:k], g["dist1000"])
    assert np.array_equal(got, g["values"])


@pytest.mark.parametrize("deg", [0, 1, 2])
@pytest.mark.parametrize("lam", [0.0, 1e-6])
@pytest.mark.parametrize("cen", [True, False])
def test_fit_many_variants_bitwise(deg, lam, cen):
    g = golden("c1")
    src, tg, vals = _c1_inputs()
    h = float(g["mean_edge_length"])
    n = 600
    off = g["off1000"][:n + 1]
    idx = g["idx1000"][:off[-1]]
    dist = g["dist1000"][:off[-1]]
    w = np.abs(O.rbf_weights(O.RBF_C4, 2.0, 2 * h, dist))
    v, c, st = O.fit_many(tg[:n], off, idx, w, src, vals, deg, lam, cen)
    key = f"d{deg}_l{'r' if lam else '0'}_{'c' if cen else 'u'}"
    assert np.array_equal(st, g["fit_s_" + key])
    assert np.array_equal(v, g["fit_v_" + key], equal_nan=True)
    assert np.array_equal(c, g["fit_c_" + key], equal_nan=True)


def test_adaptive_bitwise():
    g = golden("adaptive")
    src = synth.disk_graded(1.0, 30, 0.6).coords
    tg = synth.disk(1.0, 30).coords
    h = float(g["mean_edge_length"])
    pg = OraclePointGrid(src)
    off, idx, dist, radii, status = O.supports_nd(tg, pg, (12, h, 1.5, float(g["r_max"])))
    for name, a in (("off", off), ("idx", idx), ("dist", dist), ("radii", radii),
                    ("status", status)):
        assert np.array_equal(a, g[name]), name


def test_random_cloud_gaussian_mq_values():
    g = golden("random_clouds")
    src, tg = g["src"], g["tg"]
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    for kind, name in ((O.RBF_GAUSSIAN, "gaussian"), (O.RBF_MULTIQUADRIC, "multiquadric")):
        got, st, _ = O.transfer(src, vals, tg, 2, kind, 2.0,
                                ("adaptive", 12, 1.5 / np.sqrt(src.shape[0]), 1.5))
        # exp() of glibc vs the reference's libm call are the same function here
        assert np.array_equal(got, g[name]), name


def test_singular_status_matches_reference():
    g = golden("singular")
    off = g["off"]
    for i in range(len(g["degs"])):
        sl = slice(off[i], off[i + 1])
        m = off[i + 1] - off[i]
        v, _c, st = O.fit_many(g["tg"][i:i + 1], np.array([0, m]), np.arange(m), g["w"][sl],
                               g["pts"][sl], g["vals"][sl], int(g["degs"][i]), 0.0, True)
        assert st[0] == g["status"][i]
        assert np.array_equal(v, g["values"][i:i + 1], equal_nan=True)


def test_monomial_table_extension():
    parent, var, deg = O.monomial_table(2, 3)
    # [1, x, y, x^2, xy, y^2, x^3, x^2y, xy^2, y^3]
    assert list(deg) == [0, 1, 1, 2, 2, 2, 3, 3, 3, 3]
    assert list(parent) == [-1, 0, 0, 1, 1, 2, 3, 3, 4, 5]
    assert list(var) == [-1, 0, 1, 0, 1, 1, 0, 1, 1, 1]
    assert O.n_monomials(3, 3) == 20 and O.n_monomials(5, 2) == 21


def test_extension_polynomial_reproduction_3d_degree3():
    rng = np.random.RandomState(3)
    src = rng.uniform(0, 1, (4000, 3))
    tg = rng.uniform(0.2, 0.8, (200, 3))

    def f(p):
        x, y, z = p[:, 0], p[:, 1], p[:, 2]
        return 1 + x - 2 * y * z + x * x * z - 0.5 * y ** 3

    got, st, _ = O.transfer(src, f(src), tg, 3, O.RBF_C4, 2.0, ("adaptive", 40, 0.05, 1.5))
    assert (st == 0).all()
    assert np.max(np.abs(got - f(tg))) < 1e-9


def test_multicomponent_equals_columns():
    src, tg, vals = _c1_inputs()
    tg = tg[:300]
    V = np.stack([vals, 2 * vals - 1, np.cos(src[:, 0])], 1)
    h = float(golden("c1")["mean_edge_length"])
    got, st, _ = O.transfer(src, V, tg, 2, O.RBF_C4, 2.0, ("fixed", 2 * h))
    for c in range(3):
        one, _, _ = O.transfer(src, V[:, c].copy(), tg, 2, O.RBF_C4, 2.0, ("fixed", 2 * h))
        assert np.array_equal(got[:, c], one)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_oracle_equals_reference_ext_adaptive_fit():
    E = ref.ext()
    src = synth.disk_graded(1.0, 20, 0.6).coords
    tg = synth.disk(1.0, 20).coords
    pg = OraclePointGrid(src)
    h = synth.disk_graded(1.0, 20, 0.6).mean_edge_length
    r_max = O.r_max_for(src, tg)
    want = E.adaptive_radius_supports(tg, pg.points, pg.lo[0], pg.lo[1], pg.dx, pg.dy, pg.nx,
                                      pg.ny, pg.cell_offsets, pg.cell_items, 12, h, 1.5, r_max)
    got = O.adaptive_radius_supports(tg, pg.points, pg.lo[0], pg.lo[1], pg.dx, pg.dy, pg.nx,
                                     pg.ny, pg.cell_offsets, pg.cell_items, 12, h, 1.5, r_max)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    off, idx, dist, radii, _ = got
    w = np.abs(O.rbf_for_supports(O.RBF_GAUSSIAN, 2.0, off, dist, radii))
    vals = np.cos(3 * src[:, 0]) + src[:, 1]
    for deg in (1, 2):
        a = O.fit_many(tg, off, idx, w, src, vals, deg, 0.0, True)
        b = E.fit_many(tg, off, idx, w, src, vals, deg, 0.0, True)
        for x, y in zip(a, b):
            assert np.array_equal(x, y, equal_nan=True)


def _locate_case(d, name, tol, fn):
    g = d[f"{name}_grid"]
    gn = d[f"{name}_grid_n"]
    return fn(d[f"{name}_pts"], d[f"{name}_tri_xy"], d[f"{name}_tris"], d[f"{name}_tri_edges"],
              d[f"{name}_vert_gid"], d[f"{name}_tri_gid"], d[f"{name}_inv2a"],
              d[f"{name}_epsfac"], float(g[0]), float(g[1]), float(g[2]), float(g[3]),
              int(gn[0]), int(gn[1]), d[f"{name}_cell_off"], d[f"{name}_cell_items"], tol)


@pytest.mark.parametrize("name", ["sq", "disk"])
@pytest.mark.parametrize("tol", [1e-10, 0.0, 1e-6])
def test_oracle_locate_batch_bitwise(name, tol):
    """locate_batch restatement vs the reference's own outputs (_ext.pyx:88-152)."""
    d = golden("locate")
    got = _locate_case(d, name, tol, O.locate_batch)
    for k, a in zip(("found", "elem", "dim", "ent", "bary"), got):
        want = d[f"{name}_{tol:g}_{k}"]
        assert a.dtype == want.dtype
        assert np.array_equal(a, want, equal_nan=(k == "bary")), k


@pytest.mark.parametrize("name", ["sq", "disk"])
@pytest.mark.parametrize("loc", ["vertices", "centroids"])
@pytest.mark.parametrize("layers", [1, 2, 3])
def test_oracle_patch_supports_bitwise(name, loc, layers):
    """ElementPatch restatement vs the reference's own _PatchTopology.patch_dofs
    (pointwise.py:190-230) for every element as seed."""
    d = golden("patch")
    tris = d[f"{name}_tris"]
    seeds = np.arange(tris.shape[0])
    off, idx = O.patch_supports(seeds, d[f"{name}_edge_tris"], tris, layers, loc == "centroids")
    assert np.array_equal(off, d[f"{name}_{loc}_{layers}_off"])
    assert np.array_equal(idx, d[f"{name}_{loc}_{layers}_idx"])


def _golden_mesh(d, name):
    from types import SimpleNamespace

    keys = ("tris", "edge_tris", "tri_xy", "tri_edges", "vert_gid", "tri_gid", "inv2a", "epsfac",
            "diameters", "bbox")
    return SimpleNamespace(**{k: d[f"{name}_{k}"] for k in keys})


@pytest.mark.parametrize("name", ["sq", "disk"])
def test_element_grid_matches_reference_uniform_grid(name):
    """ElementGrid (tensor ops; run here on CPU tensors) == the reference's
    UniformGrid (locate.py:111-141): geometry and cell CSR bitwise."""
    import torch

    from paper_2510_18838_b200.locate import ElementGrid

    d = golden("patch")
    eg = ElementGrid(_golden_mesh(d, name), device=torch.device("cpu"))
    g, gn = d[f"{name}_grid"], d[f"{name}_grid_n"]
    assert (eg.nx, eg.ny) == (int(gn[0]), int(gn[1]))
    assert [eg.lo[0], eg.lo[1], eg.dx, eg.dy] == g.tolist()
    assert np.array_equal(eg.cell_offsets.numpy(), d[f"{name}_cell_off"])
    assert np.array_equal(eg.cell_items.numpy(), d[f"{name}_cell_items"])
