"""GPU parity: the B200 path against the reference's golden outputs and the
CPU oracle, through the package API and the C ABI.

Mirrors the reference's hot-path tests (pkg/tests/test_pointwise.py and
test_locate.py:128-141).  Bars (north_star): neighbour
sets and distances bit-exact; values within 1e-10 relative in fp64.
"""

import numpy as np
import pytest

from conftest import golden, sample_field
from oracle import oracle as O
from paper_2510_18838_b200 import _kernels as Kb
from paper_2510_18838_b200 import pointwise as P
from paper_2510_18838_b200 import synth

pytestmark = pytest.mark.gpu

VALUE_RTOL = 1e-10  # north_star: interpolated values within 1e-10 relative (fp64)
ALL_KINDS = list(P.RbfKind)


def _rel(a, b):
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


# ------------------------------------------------------------ rbf (a5)
def test_rbf_table():
    g = golden("rbf")
    for kind in range(8):
        got = Kb.rbf_weights(kind, 2.0, 0.7, g["r"])
        want = g[f"w{kind}"]
        if kind in (0, 6):  # exp / log: CUDA libm vs glibc, <= 2 ulp
            assert np.allclose(got, want, rtol=5e-16, atol=0), kind
        else:
            assert np.array_equal(got, want), kind


def test_eval_rbf_table_values():
    # reference test_pointwise.py:24-46
    assert P.eval_rbf(P.RadialBasisSpec(P.RbfKind.GAUSSIAN, r_c=1.0), 0.0) == 1.0
    assert P.eval_rbf(P.RadialBasisSpec(P.RbfKind.C4, r_c=1.0), 0.0) == 6.0
    got = P.eval_rbf(P.RadialBasisSpec(P.RbfKind.MULTIQUADRIC, a=2.0, r_c=0.7), 0.7)
    assert got == pytest.approx(np.sqrt(5.0), rel=1e-15)
    assert P.eval_rbf(P.RadialBasisSpec(P.RbfKind.THIN_PLATE_SPLINE, r_c=1.0), 0.0) == 0.0
    for kind in ALL_KINDS:
        w = P.eval_rbf(P.RadialBasisSpec(kind, r_c=0.4), 0.6)
        assert w == (1.0 if kind is P.RbfKind.IDENTITY else 0.0)
    spec = P.RadialBasisSpec(P.RbfKind.IDENTITY)
    assert np.array_equal(P.eval_rbf(spec, np.array([0.0, 5.0])), [1.0, 1.0])
    with pytest.raises(ValueError):
        Kb.rbf_weights(9, 2.0, 1.0, np.array([0.1]))


# ------------------------------------------------------ search (a1-a4)
def test_point_grid_radius_query_bitwise():
    # reference test_locate.py:128-141, through the drop-in seam
    g = golden("disk_small")
    pg = P.PointGrid(g["coords"])
    t = np.ascontiguousarray(g["centroids"][:50])
    off, idx, dist = Kb.fixed_radius_supports(t, pg.points, float(pg.lo[0]), float(pg.lo[1]),
                                              pg.dx, pg.dy, pg.nx, pg.ny, None, None, 0.3)
    assert off.dtype == np.int64 and idx.dtype == np.int64 and dist.dtype == np.float64
    assert np.array_equal(off, g["rq_off"])
    assert np.array_equal(idx, g["rq_idx"])
    assert np.array_equal(dist, g["rq_dist"])
    d_all = np.linalg.norm(g["coords"][None, :, :] - t[:, None, :], axis=2)
    for i in range(t.shape[0]):
        assert np.array_equal(idx[off[i]:off[i + 1]], np.nonzero(d_all[i] < 0.3)[0])


def test_point_grid_cells_match_reference():
    g = golden("disk_small")
    pg = P.PointGrid(g["coords"])
    assert np.array_equal(pg.cell_offsets, g["cell_offsets"])
    assert np.array_equal(pg.cell_items, g["cell_items"])


def _c1():
    m = synth.square(99)
    src = m.coords
    tg = np.random.RandomState(0).uniform(0, 1, (10000, 2))
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    return src, tg, vals, m.mean_edge_length


def test_c1_supports_bitwise():
    g = golden("c1")
    src, tg, vals, h = _c1()
    pg = P.PointGrid(src)
    off, idx, dist = Kb.fixed_radius_supports(tg, src, float(pg.lo[0]), float(pg.lo[1]), pg.dx,
                                              pg.dy, pg.nx, pg.ny, None, None, 2 * h)
    assert np.array_equal(np.diff(off), g["counts"].astype(np.int64))
    k = int(g["off1000"][-1])
    assert np.array_equal(idx[:k], g["idx1000"])
    assert np.array_equal(dist[:k], g["dist1000"])
    # the whole CSR against the oracle (bitwise)
    po = O.OraclePointGrid(src)
    want = O.supports_nd(tg, po, 2 * h)
    for a, b in zip((off, idx, dist), want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cells_per_point", [0.25, 1.0, 4.0])
def test_supports_independent_of_grid_resolution(cells_per_point):
    src, tg, _vals, h = _c1()
    from paper_2510_18838_b200 import device as D

    cloud = D.SourceCloud(src, cells_per_point)
    t = D.to_device(tg)
    sel = D.fixed(2.5 * h)
    cnt = D.count_supports(cloud, t, sel, cloud.target_order(t))
    idx, dist, _ = D.fill_supports(cloud, t, sel, cnt, None)
    want = O.supports_nd(tg, O.OraclePointGrid(src), 2.5 * h)
    assert np.array_equal(cnt.offsets.cpu().numpy(), want[0])
    assert np.array_equal(idx.cpu().numpy(), want[1])
    assert np.array_equal(dist.cpu().numpy(), want[2])


def test_adaptive_supports_bitwise():
    g = golden("adaptive")
    src = synth.disk_graded(1.0, 30, 0.6).coords
    tg = synth.disk(1.0, 30).coords
    h = float(g["mean_edge_length"])
    pg = P.PointGrid(src)
    got = Kb.adaptive_radius_supports(tg, src, float(pg.lo[0]), float(pg.lo[1]), pg.dx, pg.dy,
                                      pg.nx, pg.ny, None, None, 12, h, 1.5, float(g["r_max"]))
    for name, a in zip(("off", "idx", "dist", "radii", "status"), got):
        assert np.array_equal(a, g[name]), name


def test_lattice_targets_at_exact_spacing_multiples():
    # targets on the source lattice and half-way: exact ties d == r must be excluded
    src = synth.square(40).coords
    h = 1.0 / 40
    tg = np.vstack([src[::7], src[::11] + 0.5 * h])
    for r in (h, 2 * h, np.sqrt(2) * h, 3 * h):
        po = O.OraclePointGrid(src)
        want = O.supports_nd(tg, po, r)
        got = Kb.fixed_radius_supports(tg, src, po.lo[0], po.lo[1], po.dx, po.dy, po.nx, po.ny,
                                       None, None, r)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)


def test_select_support_single_coincident_source():
    src = np.array([[0.5, 0.5], [3.0, 3.0]])
    idx, w = P.select_support((0.5, 0.5), src, P.FixedRadius(0.1),
                              rbf=P.RadialBasisSpec(P.RbfKind.C4, r_c=0.1), fit_degree=0)
    assert list(idx) == [0]
    assert w[0] == 6.0


def test_fixed_radius_underdetermined():
    src = np.random.RandomState(0).uniform(0, 1, size=(4, 2))
    with pytest.raises(P.UnderdeterminedError):
        P.select_support((0.5, 0.5), src, P.FixedRadius(5.0),
                         rbf=P.RadialBasisSpec(P.RbfKind.CONST, r_c=5.0), fit_degree=2)


def test_adaptive_radius_matches_distance_sort_oracle():
    xs = np.linspace(0, 1, 11)
    src = np.array([(x, y) for x in xs for y in xs])
    target = np.array([0.52, 0.47])
    r0, growth, min_points = 1e-3, 1.5, 10
    idx, w = P.select_support(target, src, P.AdaptiveRadius(min_points, r0, growth),
                              rbf=P.RadialBasisSpec(P.RbfKind.CONST), fit_degree=1)
    d = np.linalg.norm(src - target, axis=1)
    r = r0
    while np.count_nonzero(d < r) < min_points:
        r *= growth
    assert np.array_equal(np.sort(idx), np.nonzero(d < r)[0])
    assert set(np.argsort(d)[:min_points]).issubset(set(idx))


def test_adaptive_radius_insufficient_sources():
    src = np.array([[0.0, 0.0], [1.0, 0.0]])
    with pytest.raises(P.InsufficientSourcesError):
        P.select_support((0.5, 0.5), src, P.AdaptiveRadius(5, 0.1, 2.0),
                         rbf=P.RadialBasisSpec(P.RbfKind.CONST), fit_degree=0)


# ----------------------------------------------------------- fit (a7)
def test_fit_local_cases():
    g = golden("fit_local")
    c = P.fit_local((0.1, -0.2), g["const_pts"], np.full(8, 7.0), g["const_w"], degree=2)
    assert c[0] == pytest.approx(7.0, rel=1e-13)
    assert np.abs(c[1:]).max() < 1e-12
    assert np.allclose(c, g["const_c"], rtol=1e-10, atol=1e-13)
    pts = np.array([[0.0, 0.0], [1.0, 0.1], [0.2, 1.0], [0.9, 0.8]])
    c = P.fit_local((0.4, 0.3), pts, 2 * pts[:, 0] + 3 * pts[:, 1], np.ones(4), degree=1)
    assert c[0] == pytest.approx(2 * 0.4 + 3 * 0.3, abs=1e-12)
    assert c[1] == pytest.approx(2.0, abs=1e-12) and c[2] == pytest.approx(3.0, abs=1e-12)
    norms = []
    for lam in (0.0, 1e2, 1e4, 1e6):
        c = P.fit_local((0.0, 0.0), g["ridge_pts"], g["ridge_vals"], np.ones(10), degree=1,
                        lam=lam)
        assert _rel(c, g[f"ridge_c_{lam:g}"]) < 1e-10
        norms.append(np.linalg.norm(c))
    assert all(a >= b for a, b in zip(norms, norms[1:]))
    assert norms[-1] < 1e-4 * norms[0]


def test_fit_local_singular_without_regularization():
    pts = np.array([[0.0, 0.0], [0.5, 0.5], [1.0, 1.0], [0.25, 0.25]])
    vals = np.array([0.0, 1.0, 2.0, 0.5])
    with pytest.raises(P.SingularFitError):
        P.fit_local((0.5, 0.5), pts, vals, np.ones(4), degree=1, lam=0.0)
    c = P.fit_local((0.5, 0.5), pts, vals, np.ones(4), degree=1, lam=1e-8)
    assert np.isfinite(c).all()
    assert _rel(c, golden("fit_local")["collinear_ridge_c"]) < 1e-8


def test_weight_scaling_invariance():
    rng = np.random.RandomState(3)
    pts = rng.uniform(-1, 1, size=(12, 2))
    vals = np.sin(pts[:, 0]) + pts[:, 1] ** 2
    w = rng.uniform(0.5, 1.5, size=12)
    c1 = P.fit_local((0.1, 0.2), pts, vals, w, degree=2)
    c2 = P.fit_local((0.1, 0.2), pts, vals, 37.5 * w, degree=2)
    assert np.allclose(c1, c2, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("deg", [0, 1, 2])
@pytest.mark.parametrize("lam", [0.0, 1e-6])
@pytest.mark.parametrize("cen", [True, False])
def test_fit_many_variants_vs_reference(deg, lam, cen):
    g = golden("c1")
    src, tg, vals, h = _c1()
    n = 600
    off = g["off1000"][:n + 1]
    idx = g["idx1000"][:off[-1]]
    w = np.abs(O.rbf_weights(O.RBF_C4, 2.0, 2 * h, g["dist1000"][:off[-1]]))
    v, c, st = Kb.fit_many(tg[:n], off, idx, w, src, vals, deg, lam, cen)
    key = f"d{deg}_l{'r' if lam else '0'}_{'c' if cen else 'u'}"
    assert np.array_equal(st, g["fit_s_" + key])
    assert _rel(v, g["fit_v_" + key]) < VALUE_RTOL
    # coefficients in the solver's scaled basis (c_j * s^deg_j, _ext.pyx:411-412):
    # both solvers are backward stable there, so they agree to ~eps*cond(A)
    want_c = g["fit_c_" + key]
    s = np.empty(n)
    for i in range(n):
        d = src[idx[off[i]:off[i + 1]]] - (tg[i] if cen else 0.0)
        s[i] = np.sqrt(np.max(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]))
    degs = np.array([0, 1, 1, 2, 2, 2])[:c.shape[1]]
    sp = s[:, None] ** degs[None, :]
    scale = np.abs(want_c * sp).max(axis=1, keepdims=True)
    # uncentered fits at C1 geometry have cond(A) up to ~4e8
    assert np.max(np.abs((c - want_c) * sp) / scale) < (1e-9 if cen else 1e-6)


def test_singular_status_outside_gray_zone():
    g = golden("singular")
    off = g["off"]
    n = len(g["degs"])
    gray = compared = 0
    for i in range(n):
        sl = slice(off[i], off[i + 1])
        m = off[i + 1] - off[i]
        v, _c, st = Kb.fit_many(g["tg"][i:i + 1], np.array([0, m]), np.arange(m), g["w"][sl],
                                g["pts"][sl], g["vals"][sl], int(g["degs"][i]), 0.0, True)
        cond = g["cond"][i]
        if 1e15 <= cond <= 1e17:
            gray += 1
            continue
        assert st[0] == g["status"][i], (i, cond)
        # value parity is meaningful only for well-posed fits: two backward
        # stable solvers differ by ~eps*cond(A) (SURVEY.md §7 "Rank / status parity")
        if st[0] == 0 and cond < 1e5:
            compared += 1
            assert abs(v[0] - g["values"][i]) <= VALUE_RTOL * abs(g["values"][i]) + 1e-13
    assert gray < n // 2 and compared >= 15


# ------------------------------------------------- transfers (a8, a9)
@pytest.mark.parametrize("kind", ALL_KINDS)
@pytest.mark.parametrize("degree", [0, 1, 2])
def test_polynomial_reproduction_small(disk_small, kind, degree):
    # reference test_pointwise.py:146-163 + values vs the reference's
    polys = {
        0: lambda x, y: np.full_like(x, 3.5),
        1: lambda x, y: 2 * x - y + 1,
        2: lambda x, y: x * x + 2 * x * y - y * y + x + 0.5,
    }
    f = sample_field(disk_small, polys[degree])
    h = disk_small.mean_edge_length
    spec = P.FitSpec(degree, P.RadialBasisSpec(kind, a=2.0),
                     P.AdaptiveRadius(max(6, 2 * P.n_monomials(degree)), 1.5 * h, 1.5), lam=0.0)
    got = P.transfer_pointwise(f, disk_small.centroids(), spec)
    c = disk_small.centroids()
    want = polys[degree](c[:, 0], c[:, 1])
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-10
    ref = golden("poly_repro")[f"{kind.value}_{degree}"]
    assert _rel(got, ref) < VALUE_RTOL


def test_cutoff_locality_bitwise(disk_small):
    h = disk_small.mean_edge_length
    r_c = 2.0 * h
    f = sample_field(disk_small, lambda x, y: np.sin(x) * np.cos(y) + 2)
    targets = disk_small.centroids()[:40]
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(r_c))
    base = P.transfer_pointwise(f, targets, spec)
    d = np.linalg.norm(disk_small.coords[None, :, :] - targets[:, None, :], axis=2).min(axis=0)
    far = int(np.argmax(d))
    assert d[far] > r_c
    values = f.values.copy()
    values[far] += 1e6
    assert np.array_equal(base, P.transfer_pointwise(f.with_values(values), targets, spec))


def test_transfer_against_dense_least_squares_oracle(disk_small):
    h = disk_small.mean_edge_length
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(2.0 * h))
    f = sample_field(disk_small, lambda x, y: np.sin(x) * np.cos(y) + 2)
    targets = disk_small.centroids()
    got = P.transfer_pointwise(f, targets, spec)
    src = disk_small.coords
    oracle = np.empty(targets.shape[0])
    for i, t in enumerate(targets):
        d = np.linalg.norm(src - t, axis=1)
        sel = np.nonzero(d < 2.0 * h)[0]
        w = O.rbf_weights(O.RBF_C4, 2.0, 2.0 * h, d[sel])
        A = np.column_stack([np.ones(sel.size), src[sel, 0] - t[0], src[sel, 1] - t[1]])
        cc, *_ = np.linalg.lstsq(A * w[:, None], w * f.values[sel], rcond=None)
        oracle[i] = cc[0]
    assert np.abs(got - oracle).max() < 1e-12
    assert _rel(got, golden("poly_repro")["fixed_c4_1"]) < VALUE_RTOL


def test_transfer_threads_identical(disk_small):
    h = disk_small.mean_edge_length
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(2.0 * h))
    f = sample_field(disk_small, lambda x, y: np.sin(3 * x) + y)
    one = P.transfer_pointwise(f, disk_small.centroids(), spec, threads=1)
    four = P.transfer_pointwise(f, disk_small.centroids(), spec, threads=4)
    assert np.array_equal(one, four)


def test_extrinsic_analytic_callback_exact(disk_small):
    h = disk_small.mean_edge_length
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.GAUSSIAN), P.FixedRadius(2.5 * h))
    got = P.transfer_extrinsic(lambda p: 4 * p[:, 0] - p[:, 1] + 2, disk_small.centroids(), spec,
                               disk_small.coords)
    c = disk_small.centroids()
    assert np.abs(got - (4 * c[:, 0] - c[:, 1] + 2)).max() < 1e-10


def test_extrinsic_matches_intrinsic_bitwise(disk_small):
    h = disk_small.mean_edge_length
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(2.0 * h))
    f = sample_field(disk_small, lambda x, y: np.sin(x) * np.cos(y) + 2)
    table = {(float(x), float(y)): float(v) for (x, y), v in zip(disk_small.coords, f.values)}
    calls = []

    def callback(pts):
        calls.append(len(pts))
        return np.array([table[(float(x), float(y))] for x, y in pts])

    intrinsic = P.transfer_pointwise(f, disk_small.centroids(), spec)
    extrinsic = P.transfer_extrinsic(callback, disk_small.centroids(), spec, disk_small.coords,
                                     batch_size=100)
    assert np.array_equal(intrinsic, extrinsic)
    assert len(calls) <= int(np.ceil(disk_small.nelems / 100))


def test_extrinsic_failure_names_batch(disk_small):
    h = disk_small.mean_edge_length
    spec = P.FitSpec(0, P.RadialBasisSpec(P.RbfKind.CONST), P.FixedRadius(2.0 * h))
    state = {"batch": 0}

    def flaky(pts):
        if state["batch"] == 3:
            raise RuntimeError("remote evaluation unavailable")
        state["batch"] += 1
        return np.zeros(len(pts))

    with pytest.raises(P.ExtrinsicEvaluationError) as exc:
        P.transfer_extrinsic(flaky, disk_small.centroids(), spec, disk_small.coords,
                             batch_size=50)
    assert exc.value.batch == 3 and "batch 3" in str(exc.value)


def test_source_equals_target_polynomial_consistency(disk_small):
    f = sample_field(disk_small, lambda x, y: x - 2 * y + 3)
    h = disk_small.mean_edge_length
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(2.5 * h))
    got = P.transfer_pointwise(f, disk_small.coords, spec)
    assert np.linalg.norm(got - f.values) / np.linalg.norm(f.values) < 1e-10


def test_c1_values_vs_reference():
    g = golden("c1")
    src, tg, vals, h = _c1()
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.FixedRadius(2 * h))
    got = P.fit_point_cloud(src, vals, tg, spec)
    assert _rel(got, g["values"]) < VALUE_RTOL


def test_prepared_transfer_adaptive_vs_reference():
    g = golden("adaptive")
    src = synth.disk_graded(1.0, 30, 0.6).coords
    tg = synth.disk(1.0, 30).coords
    h = float(g["mean_edge_length"])
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.AdaptiveRadius(12, h, 1.5))
    pt = P.PreparedTransfer(src, tg, spec)
    vals3 = synth.sincos_field(src, 3)
    Y = pt.apply(vals3)
    assert Y.shape == (tg.shape[0], 3)
    assert _rel(Y, g["values3"]) < VALUE_RTOL
    for c in range(3):
        assert _rel(pt.apply(vals3[:, c]), g["values3"][:, c]) < VALUE_RTOL
    off, idx, w = pt.support
    assert np.array_equal(off, g["off"]) and np.array_equal(idx, g["idx"])
    with pytest.raises(P.FieldError):
        pt.apply(np.ones(3))


def test_random_cloud_gaussian_multiquadric():
    g = golden("random_clouds")
    src, tg = g["src"], g["tg"]
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    for kind in (P.RbfKind.GAUSSIAN, P.RbfKind.MULTIQUADRIC):
        spec = P.FitSpec(2, P.RadialBasisSpec(kind, a=2.0),
                         P.AdaptiveRadius(12, 1.5 / np.sqrt(src.shape[0]), 1.5))
        assert _rel(P.fit_point_cloud(src, vals, tg, spec), g[kind.value]) < VALUE_RTOL


def test_singular_transfer_raises():
    # all sources on a line: a degree-1 fit is rank deficient everywhere
    x = np.linspace(0, 1, 50)
    src = np.column_stack([x, 0.5 * x])
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.CONST), P.FixedRadius(0.3))
    with pytest.raises(P.SingularFitError, match="rank-deficient degree-1"):
        P.fit_point_cloud(src, x, src[10:20], spec)
    pt = P.PreparedTransfer(src, src[10:20], spec)  # supports fine, fit fails at apply
    with pytest.raises(P.SingularFitError):
        pt.apply(x)


def test_empty_weight_support_raises_singular():
    # thin plate spline weight is 0 at r = 0: a lone coincident source has no weight
    src = np.array([[0.0, 0.0], [5.0, 5.0]])
    spec = P.FitSpec(0, P.RadialBasisSpec(P.RbfKind.THIN_PLATE_SPLINE), P.FixedRadius(0.5))
    with pytest.raises(P.SingularFitError, match="no support points with nonzero weight"):
        P.fit_point_cloud(src, np.ones(2), [(0.0, 0.0)], spec)


def test_empty_targets():
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(0.1))
    src = np.random.RandomState(0).uniform(0, 1, (100, 2))
    assert P.fit_point_cloud(src, np.ones(100), np.zeros((0, 2)), spec).shape == (0,)
    off, idx, dist = Kb.fixed_radius_supports(np.zeros((0, 2)), src, 0.0, 0.0, 0.1, 0.1, 10, 10,
                                              None, None, 0.1)
    assert off.tolist() == [0] and idx.size == 0


# ------------------------------------------------ extensions (oracle)
def test_extension_3d_degree3_vs_oracle():
    rng = np.random.RandomState(3)
    src = rng.uniform(0, 1, (6000, 3))
    tg = rng.uniform(0.1, 0.9, (500, 3))
    vals = np.cos(2 * src[:, 0]) + src[:, 1] * src[:, 2]
    spec = P.FitSpec(3, P.RadialBasisSpec(P.RbfKind.C4), P.AdaptiveRadius(40, 0.05, 1.5))
    got = P.fit_point_cloud(src, vals, tg, spec)
    want, st, sup = O.transfer(src, vals, tg, 3, O.RBF_C4, 2.0, ("adaptive", 40, 0.05, 1.5))
    assert (st == 0).all()
    assert _rel(got, want) < VALUE_RTOL


@pytest.mark.parametrize("dim,deg", [(1, 2), (3, 2), (4, 1), (5, 1), (5, 2)])
def test_extension_nd_vs_oracle(dim, deg):
    rng = np.random.RandomState(10 + dim)
    ns = {1: 500, 3: 8000, 4: 20000, 5: 30000}[dim]
    src = rng.uniform(0, 1, (ns, dim))
    tg = rng.uniform(0.2, 0.8, (300, dim))
    vals = np.sin(src.sum(axis=1)) + 2
    need = P.n_monomials(deg, dim)
    spec = P.FitSpec(deg, P.RadialBasisSpec(P.RbfKind.C4), P.AdaptiveRadius(2 * need, 0.02, 1.5))
    got = P.fit_point_cloud(src, vals, tg, spec)
    want, st, _ = O.transfer(src, vals, tg, deg, O.RBF_C4, 2.0, ("adaptive", 2 * need, 0.02, 1.5))
    assert (st == 0).all()
    assert _rel(got, want) < VALUE_RTOL


def test_extension_multicomponent_apply_equals_columns():
    src, tg, vals, h = _c1()
    V = synth.sincos_field(src, 8)
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(2 * h))
    pt = P.PreparedTransfer(src, tg, spec)
    Y = pt.apply(V)
    want, _c, st = O.fit_many_nd(tg, *O.supports_nd(tg, O.OraclePointGrid(src), 2 * h)[:2],
                                 np.abs(O.rbf_weights(O.RBF_C4, 2.0, 2 * h,
                                                      O.supports_nd(tg, O.OraclePointGrid(src),
                                                                    2 * h)[2])),
                                 src, V, 2, 0.0, True)
    assert _rel(Y, want) < VALUE_RTOL
    assert _rel(P.fit_point_cloud(src, V, tg, spec), want) < VALUE_RTOL


def _apply_direct(row_lens, ns, C, seed, local=True):
    """fm_apply on a synthetic CSR (rows in stored order, perm reversed)
    against a float64 numpy reference; exercises the tiled kernel's staged
    path (local columns), its fallbacks (tile streams > 2048 nonzeros, > 512
    distinct columns) and the direct kernels (C != 8)."""
    import torch

    from paper_2510_18838_b200 import _lib as L
    from paper_2510_18838_b200.device import _stream

    rng = np.random.default_rng(seed)
    nt = len(row_lens)
    off = np.zeros(nt + 1, np.int64)
    off[1:] = np.cumsum(row_lens)
    nnz = int(off[-1])
    if local:  # columns near the row's position (neighbouring rows share)
        base = (np.repeat(np.arange(nt), row_lens) * ns) // max(nt, 1)
        col = np.clip(base + rng.integers(-20, 21, nnz), 0, ns - 1).astype(np.int32)
    else:
        col = rng.integers(0, ns, nnz).astype(np.int32)
    val = rng.standard_normal(nnz)
    perm = np.arange(nt)[::-1].astype(np.int32).copy()
    X = rng.standard_normal((ns, C))
    want = np.zeros((nt, C))
    for k in range(nt):
        sl = slice(off[k], off[k + 1])
        want[perm[k]] = val[sl] @ X[col[sl]]
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    Y = torch.full((nt, C), np.nan, dtype=torch.float64, device="cuda")
    off_d, col_d, val_d, perm_d, X_d = d(off), d(col), d(val), d(perm), d(X)
    L.check(L.lib().fm_apply(nt, L.ptr(off_d), L.ptr(col_d), L.ptr(val_d), L.ptr(perm_d),
                             L.ptr(X_d), C, L.ptr(Y), _stream()), "fm_apply")
    got = Y.cpu().numpy()
    scale = (np.abs(val).max() if nnz else 1.0) * np.abs(X).max() * max(int(row_lens.max()), 1)
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want)) <= 1e-13 * scale


@pytest.mark.gpu
@pytest.mark.parametrize("C", [1, 2, 4, 8, 16, 3])
def test_apply_local_rows(C):
    rng = np.random.default_rng(5)
    _apply_direct(rng.integers(0, 40, 5000), 3000, C, 11)


@pytest.mark.gpu
def test_apply_tiled_fallbacks():
    rng = np.random.default_rng(6)
    lens = rng.integers(5, 30, 3000)
    lens[640:704] = 100          # one 64-row tile with 6400 nonzeros (> 2048 staged)
    lens[1000] = 5000            # a single very long row
    lens[2000:2010] = 0          # empty rows
    _apply_direct(lens, 100000, 8, 12, local=True)
    _apply_direct(rng.integers(20, 30, 3000), 100000, 8, 13, local=False)  # > 512 distinct/tile
    _apply_direct(np.array([3]), 10, 8, 14)       # one row, partial tile
    _apply_direct(np.zeros(70, np.int64), 10, 8, 15)  # all rows empty


@pytest.mark.gpu
def test_fit_point_cloud_tensor_paths():
    """torch inputs: pinned host tensors -> pinned host tensor, CUDA tensors
    -> CUDA tensor; same values as the numpy path (scalar and 8 components)."""
    import torch

    src, tg, vals, h = _c1()
    V = synth.sincos_field(src, 8)
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(2 * h))
    for field in (vals, V):
        want = P.fit_point_cloud(src, field, tg, spec)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        got_h = P.fit_point_cloud(pin(src), pin(field), pin(tg), spec)
        assert isinstance(got_h, torch.Tensor) and not got_h.is_cuda and got_h.is_pinned()
        assert np.array_equal(got_h.numpy(), want)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        got_d = P.fit_point_cloud(cu(src), cu(field), cu(tg), spec)
        assert got_d.is_cuda
        assert np.array_equal(got_d.cpu().numpy(), want)
    with pytest.raises(P.FieldError):
        P.fit_point_cloud(torch.from_numpy(src), torch.ones(3, dtype=torch.float64),
                          torch.from_numpy(tg), spec)
    empty = P.fit_point_cloud(torch.from_numpy(src), torch.from_numpy(V),
                              torch.zeros((0, 2), dtype=torch.float64), spec)
    assert tuple(empty.shape) == (0, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sq", "disk"])
@pytest.mark.parametrize("tol", [1e-10, 0.0, 1e-6])
def test_locate_batch_bitwise(name, tol):
    """fm_locate_batch vs the reference's own locate_batch outputs
    (_ext.pyx:88-152, golden fixture): found/elem/dim/ent/bary bitwise."""
    d = golden("locate")
    g, gn = d[f"{name}_grid"], d[f"{name}_grid_n"]
    got = Kb.locate_batch(d[f"{name}_pts"], d[f"{name}_tri_xy"], d[f"{name}_tris"],
                          d[f"{name}_tri_edges"], d[f"{name}_vert_gid"], d[f"{name}_tri_gid"],
                          d[f"{name}_inv2a"], d[f"{name}_epsfac"], float(g[0]), float(g[1]),
                          float(g[2]), float(g[3]), int(gn[0]), int(gn[1]),
                          d[f"{name}_cell_off"], d[f"{name}_cell_items"], tol)
    for k, a in zip(("found", "elem", "dim", "ent", "bary"), got):
        want = d[f"{name}_{tol:g}_{k}"]
        assert a.dtype == want.dtype and a.shape == want.shape, k
        assert np.array_equal(a, want, equal_nan=(k == "bary")), k


@pytest.mark.gpu
def test_locate_batch_large_vs_oracle():
    """100k random points (some outside) on the golden square mesh: GPU == C oracle."""
    d = golden("locate")
    sys_pts = np.random.default_rng(3).uniform(-0.05, 1.05, (100000, 2))
    g, gn = d["sq_grid"], d["sq_grid_n"]
    args = (d["sq_tri_xy"], d["sq_tris"], d["sq_tri_edges"], d["sq_vert_gid"], d["sq_tri_gid"],
            d["sq_inv2a"], d["sq_epsfac"], float(g[0]), float(g[1]), float(g[2]), float(g[3]),
            int(gn[0]), int(gn[1]), d["sq_cell_off"], d["sq_cell_items"], 1e-10)
    got = Kb.locate_batch(sys_pts, *args)
    want = O.locate_batch(sys_pts, *args)
    for a, b in zip(got, want):
        assert np.array_equal(a, b, equal_nan=True)


@pytest.mark.gpu
def test_prepared_transfer_all_size_buckets_and_overflow():
    """Clustered sources + a fixed radius: support sizes 6 .. 143, so the
    build runs one fit shape per size bucket (<= 8 ... > 128) and the
    supports beyond the 64-entry slots go through the overflow rescan; the
    operator applied to 3 components matches the CPU oracle per column."""
    rng = np.random.default_rng(21)
    bg = rng.uniform(0, 1, (6000, 2))
    cl = np.clip(0.5 + 0.03 * rng.standard_normal((250, 2)), 0, 1)
    src = np.concatenate([bg, cl])
    tg = rng.uniform(0.05, 0.95, (2000, 2))
    V = synth.sincos_field(src, 3)
    r = 0.035
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4), P.FixedRadius(r))
    pt = P.PreparedTransfer(src, tg, spec)
    Y = pt.apply(V)
    want, st, (off, idx, _d, w) = O.transfer(src, V, tg, 2, O.RBF_C4, 2.0, ("fixed", r))
    counts = np.diff(off)
    edges = [8, 16, 24, 32, 48, 64, 96, 128]
    assert counts.max() > 128 and counts.min() <= 8
    assert all(np.any((counts > lo) & (counts <= hi)) for lo, hi in zip(edges[:-1], edges[1:]))
    assert (st == 0).all()
    # values agree to ~eps*cond(A) (two backward-stable solvers): compare where
    # the scaled weighted Vandermonde is well conditioned
    cond = np.empty(len(tg))
    for i in range(len(tg)):
        sl = slice(off[i], off[i + 1])
        dx = src[idx[sl]] - tg[i]
        sc = np.sqrt((dx ** 2).sum(1).max())
        u, v = dx[:, 0] / sc, dx[:, 1] / sc
        A = w[sl, None] * np.stack([np.ones_like(u), u, v, u * u, u * v, v * v], 1)
        cond[i] = np.linalg.cond(A)
    ok = cond < 1e5
    assert ok.sum() > 0.9 * len(tg)
    err = np.abs(Y - want).max(1) / np.abs(want).max(1)
    for lo, hi in zip([0] + edges, edges + [10 ** 9]):
        b = ok & (counts > lo) & (counts <= hi)
        assert not b.any() or err[b].max() < VALUE_RTOL, (lo, hi, err[b].max())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sq", "disk"])
@pytest.mark.parametrize("loc", ["vertices", "centroids"])
@pytest.mark.parametrize("layers", [1, 2, 3])
def test_patch_supports_bitwise(name, loc, layers):
    """fm_patch_count/fill vs the reference's own _PatchTopology.patch_dofs
    (pointwise.py:190-230, golden fixture), every element as seed: the
    support CSR (offsets, ids) bitwise."""
    d = golden("patch")
    tris = d[f"{name}_tris"]
    seeds = np.arange(tris.shape[0])
    off, idx, _ = Kb.patch_supports(seeds, tris, d[f"{name}_edge_tris"], layers,
                                    loc == "centroids")
    assert off.dtype == np.int64 and idx.dtype == np.int64
    assert np.array_equal(off, d[f"{name}_{loc}_{layers}_off"])
    assert np.array_equal(idx, d[f"{name}_{loc}_{layers}_idx"])


@pytest.mark.gpu
def test_patch_supports_random_seeds_and_overflow():
    """20k random seeds (repeats, any order) at layers 1-4: GPU == oracle;
    patches beyond the per-thread bounds are computed exactly too."""
    d = golden("patch")
    tris, et = d["disk_tris"], d["disk_edge_tris"]
    seeds = np.random.default_rng(5).integers(0, tris.shape[0], 20000)
    for layers in (1, 4):
        for cen in (False, True):
            off, idx, _ = Kb.patch_supports(seeds, tris, et, layers, cen)
            w_off, w_idx = O.patch_supports(seeds, et, tris, layers, cen)
            assert np.array_equal(off, w_off) and np.array_equal(idx, w_idx)
    off, idx, _ = Kb.patch_supports(np.array([], np.int64), tris, et, 1, False)
    assert off.tolist() == [0] and idx.size == 0
    # patches beyond the per-thread bounds (128 elements / 256 dofs) take the
    # global-scratch path: no limit the reference does not have
    for cen in (True, False):
        off, idx, _ = Kb.patch_supports(seeds[:10], tris, et, 12, cen)
        w_off, w_idx = O.patch_supports(seeds[:10], et, tris, 12, cen)
        assert np.array_equal(off, w_off) and np.array_equal(idx, w_idx)
        if cen:  # more elements than the per-thread list holds
            assert np.diff(off).max() > 128
    # locate's not-found seed (-1) and out-of-range ids are rejected, not read
    for bad in (-1, tris.shape[0]):
        with pytest.raises(ValueError):
            Kb.patch_supports(np.array([3, bad, 5]), tris, et, 2, False)


@pytest.mark.gpu
def test_element_patch_locate_fit_chain():
    """The reference's ElementPatch flow (_select_batch 271-296 then
    _fit_batch 299-314) on device: locate_batch -> patch supports (unit
    weights) -> fit_many, vs the same chain on the CPU oracle."""
    d = golden("locate")
    p = golden("patch")
    rng = np.random.default_rng(11)
    t = rng.uniform(0.02, 0.98, (3000, 2))
    g, gn = d["sq_grid"], d["sq_grid_n"]
    args = (d["sq_tri_xy"], d["sq_tris"], d["sq_tri_edges"], d["sq_vert_gid"], d["sq_tri_gid"],
            d["sq_inv2a"], d["sq_epsfac"], float(g[0]), float(g[1]), float(g[2]), float(g[3]),
            int(gn[0]), int(gn[1]), d["sq_cell_off"], d["sq_cell_items"], 1e-10)
    found, elem, _, _, _ = Kb.locate_batch(t, *args)
    assert found.all()
    # vertex coordinates in vertex-id order, recovered from tri_xy / tris
    tris = p["sq_tris"]
    nv = int(tris.max()) + 1
    xy = np.empty((nv, 2))
    xy[tris.reshape(-1)] = d["sq_tri_xy"].reshape(-1, 2)
    f = np.sin(xy[:, 0]) * np.cos(xy[:, 1]) + 2
    off, idx, _ = Kb.patch_supports(elem, tris, p["sq_edge_tris"], 2, False)
    w = np.ones(idx.size)
    v, c, s = Kb.fit_many(t, off, idx, w, xy, f, 2, 0.0, True)
    w_off, w_idx = O.patch_supports(elem, p["sq_edge_tris"], tris, 2, False)
    assert np.array_equal(off, w_off) and np.array_equal(idx, w_idx)
    wv, wc, ws = O.fit_many(t, w_off, w_idx, w, xy, f, 2, 0.0, True)
    assert np.array_equal(s, ws)
    ok = s == 0
    assert ok.mean() > 0.99
    np.testing.assert_allclose(v[ok], wv[ok], rtol=1e-10, atol=0)


def _golden_mesh(d, name):
    from types import SimpleNamespace

    keys = ("tris", "edge_tris", "tri_xy", "tri_edges", "vert_gid", "tri_gid", "inv2a", "epsfac",
            "diameters", "bbox")
    return SimpleNamespace(**{k: d[f"{name}_{k}"] for k in keys})


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sq", "disk"])
@pytest.mark.parametrize("loc", ["vertices", "centroids"])
def test_fit_point_cloud_element_patch_vs_reference(name, loc):
    """fit_point_cloud with ElementPatch on a mesh (pointwise.py:271-296 +
    434-451) vs the reference's own outputs: values within 1e-10 rel;
    select_support bitwise; PreparedTransfer.apply (2 components, numpy and
    CUDA tensors) equal to the per-component values."""
    import torch

    d = golden("patch")
    mesh = _golden_mesh(d, name)
    src = d[f"{name}_coords"] if loc == "vertices" else d[f"{name}_centroids"]
    t = d[f"{name}_targets"]
    f = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    for deg, layers in ((1, 2), (2, 3)):
        spec = P.FitSpec(deg, P.RadialBasisSpec(P.RbfKind.CONST, r_c=None),
                         P.ElementPatch(layers))
        got = P.fit_point_cloud(src, f, t, spec, mesh=mesh, source_location=loc)
        want = d[f"{name}_{loc}_fit_{deg}_{layers}"]
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=0)
        pt = P.PreparedTransfer(src, t, spec, mesh=mesh, source_location=loc)
        two = np.stack([f, 2 * f + 1], axis=1)
        y = pt.apply(two)
        np.testing.assert_allclose(y[:, 0], want, rtol=1e-10, atol=0)
        np.testing.assert_allclose(y[:, 1], 2 * got + 1, rtol=1e-12, atol=1e-12)
        yt = P.fit_point_cloud(torch.from_numpy(src).cuda(), torch.from_numpy(f).cuda(),
                               torch.from_numpy(t).cuda(), spec, mesh=mesh, source_location=loc)
        assert yt.is_cuda and np.array_equal(yt.cpu().numpy(), got)
    idx, w = P.select_support(t[0], src, P.ElementPatch(2), fit_degree=2, mesh=mesh,
                              source_location=loc)
    assert np.array_equal(idx, d[f"{name}_{loc}_sel_idx"])
    assert np.array_equal(w, d[f"{name}_{loc}_sel_w"])


@pytest.mark.gpu
def test_element_patch_errors_match_reference():
    """The reference's ElementPatch errors: too few patch dofs ->
    UnderdeterminedError naming the first target (message measured on the
    reference: 'target 86 at (0.00984544, 0.994239) (index 86) patch has 2
    dofs; a degree-1 fit needs at least 3'); a target outside the mesh ->
    InsufficientSourcesError; no mesh -> FieldError."""
    from paper_2510_18838_b200.errors import (FieldError, InsufficientSourcesError,
                                              UnderdeterminedError)

    d = golden("patch")
    mesh = _golden_mesh(d, "sq")
    src, t = d["sq_centroids"], d["sq_targets"]
    f = np.ones(src.shape[0])
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.CONST, r_c=None), P.ElementPatch(1))
    with pytest.raises(UnderdeterminedError) as e:
        P.fit_point_cloud(src, f, t, spec, mesh=mesh, source_location="centroids")
    assert str(e.value) == ("target 86 at (0.00984544, 0.994239) (index 86) patch has 2 dofs; "
                            "a degree-1 fit needs at least 3")
    spec2 = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.CONST, r_c=None), P.ElementPatch(2))
    with pytest.raises(InsufficientSourcesError):
        P.fit_point_cloud(src, f, np.array([[0.5, 0.5], [1.5, 0.5]]), spec2, mesh=mesh,
                          source_location="centroids")
    with pytest.raises(FieldError):
        P.fit_point_cloud(src, f, t, spec2)


def _golden_cycle_mesh(d, name):
    from types import SimpleNamespace

    keys = ("coords", "tris", "edge_tris", "tri_xy", "tri_edges", "vert_gid", "tri_gid", "inv2a",
            "epsfac", "diameters", "bbox")
    ns = SimpleNamespace(**{k: d[f"{name}_{k}"] for k in keys})
    cen = d[f"{name}_centroids"]
    ns.centroids = lambda: cen
    return ns


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["adaptive", "patch"])
def test_pointwise_cycle_vs_reference(key):
    """PointwiseCycle vs the reference's metrics._PointwiseCycle
    (metrics.py:127-148): one mesh (vertices -> centroids -> vertices) after
    1 and 3 cycles, two meshes after 2 cycles; within 1e-10 rel.  `iterate`
    (field resident on the device) equals repeated `cycle`."""
    import torch

    from paper_2510_18838_b200 import PointwiseCycle

    d = golden("cycle")
    a, b = _golden_cycle_mesh(d, "a"), _golden_cycle_mesh(d, "b")
    if key == "adaptive":
        spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0),
                         P.AdaptiveRadius(12, float(d["mean_edge_length"]), 1.5))
    else:
        spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.CONST, r_c=None), P.ElementPatch(2))
    cyc = PointwiseCycle(a, spec)
    v = d["f0"]
    for it in range(1, 4):
        v = cyc.cycle(v)
        if it in (1, 3):
            np.testing.assert_allclose(v, d[f"{key}_one_{it}"], rtol=1e-10, atol=0)
    fin, hist = cyc.iterate(d["f0"], 3, keep_history=True)
    np.testing.assert_allclose(fin, d[f"{key}_one_3"], rtol=1e-10, atol=0)
    assert hist.shape == (3,) + d["f0"].shape
    dv = cyc.iterate(torch.from_numpy(d["f0"]).cuda(), 3)
    assert dv.is_cuda and np.array_equal(dv.cpu().numpy(), fin)
    cyc2 = PointwiseCycle(a, spec, target_mesh=b)
    np.testing.assert_allclose(cyc2.iterate(d["f0"], 2), d[f"{key}_two_2"], rtol=1e-10, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("loc", ["vertices", "centroids"])
def test_transfer_extrinsic_element_patch(loc):
    """transfer_extrinsic with ElementPatch (pointwise.py:467-510): a callback
    returning the field's own dof values reproduces the intrinsic path
    bitwise (reference test_pointwise.py:254-271) and the reference's values;
    one callback per batch."""
    d = golden("patch")
    mesh = _golden_mesh(d, "sq")
    src = d["sq_coords"] if loc == "vertices" else d["sq_centroids"]
    t = d["sq_targets"]
    f = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.CONST, r_c=None), P.ElementPatch(3))
    calls = []

    def cb(pts):
        calls.append(pts.shape[0])
        key = {tuple(p): i for i, p in enumerate(src)}
        return f[[key[tuple(p)] for p in pts]]

    got = P.transfer_extrinsic(cb, t, spec, src, batch_size=128, mesh=mesh,
                               source_location=loc)
    intr = P.fit_point_cloud(src, f, t, spec, mesh=mesh, source_location=loc)
    assert len(calls) == -(-t.shape[0] // 128)
    assert np.array_equal(got, intr)
    np.testing.assert_allclose(got, d[f"sq_{loc}_fit_2_3"], rtol=1e-10, atol=0)


@pytest.mark.gpu
def test_map_gathered_blocks_equal_one_shot():
    """distributed.map_gathered (blocks of targets, all-gather pipelined on a
    side stream) on a one-rank NCCL group: bitwise the one-shot transfer."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2510_18838_b200 import distributed as Dist
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200 import synth

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        m = synth.disk_graded(1.0, 60, 0.6)
        src = m.coords
        tgt = synth.disk(1.0, 50).coords
        X = synth.sincos_field(src, 8)
        h = m.mean_edge_length
        spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.AdaptiveRadius(12, h, 1.5))
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        want = P.fit_point_cloud(d(src), d(X), d(tgt), spec)
        for nb in (1, 3, 7):
            got = Dist.map_gathered(d(src), d(tgt), d(X), spec, nblocks=nb)
            assert torch.equal(got, want), nb
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_per_axis_metric_5d_vs_oracle():
    """Extension (SURVEY §7 decision 6): fit_point_cloud(metric=...) equals
    the oracle run on the per-axis scaled coordinates (5-D tensor grid, degree
    1, adaptive), bitwise supports through PreparedTransfer.support."""
    import torch

    from oracle import oracle as O
    from paper_2510_18838_b200 import pointwise as P

    axes = [np.linspace(0, 1, k) for k in (9, 9, 5, 5, 5)]
    g = np.meshgrid(*axes, indexing="ij")
    src = np.ascontiguousarray(np.stack([a.reshape(-1) for a in g], axis=1))
    tgt = np.random.RandomState(4).uniform(0, 1, (3000, 5))
    metric = [1.0, 1.0, 0.5, 0.5, 0.5]
    f = np.exp(-np.sum((src[:, 2:] - 0.5) ** 2, axis=1) * 4) * (1 + 0.1 * np.sin(3 * src[:, 0]))
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.AdaptiveRadius(12, 0.125, 1.5))
    got = P.fit_point_cloud(src, f, tgt, spec, metric=metric)
    ss, ts = src * np.asarray(metric), tgt * np.asarray(metric)
    want, st, (off, idx, dist, w) = O.transfer(ss, f, ts, 1, O.RBF_C4, 2.0,
                                               ("adaptive", 12, 0.125, 1.5))
    assert (st == 0).all()
    assert np.max(np.abs(got - want) / np.abs(want)) < 1e-10
    pt = P.PreparedTransfer(src, tgt, spec, metric=metric)
    off2, idx2, _w = pt.support
    assert np.array_equal(off2, off) and np.array_equal(idx2, idx)
    # device tensors in: same values
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    got_t = P.fit_point_cloud(d(src), d(f), d(tgt), spec, metric=metric).cpu().numpy()
    assert np.array_equal(got_t, got)


@pytest.mark.gpu
def test_map_chunked_equals_one_shot():
    """device.map_chunked (bounded scratch for C4/C5-size target sets) gives
    bitwise the one-shot operator's values, for 3-D degree 3 (k = 20)."""
    import torch

    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200 import pointwise as P

    src = np.random.RandomState(1).uniform(0, 1, (20000, 3))
    tgt = np.random.RandomState(5).uniform(0, 1, (7000, 3))
    f = (np.sin(3 * src[:, 0]) * np.cos(2 * src[:, 1]) * np.exp(src[:, 2]) + 2.0)[:, None]
    spec = P.FitSpec(3, P.RadialBasisSpec(P.RbfKind.C4, a=2.0),
                     P.AdaptiveRadius(40, 20000 ** (-1 / 3), 1.5))
    want = P.fit_point_cloud(src, f, tgt, spec)
    src_d, tgt_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(f)
    bs, bt = D.device_bboxes([src_d, tgt_d])
    cloud = D.SourceCloud(src_d, bbox=bs)
    sel = spec.selection
    dsel = D.adaptive(sel.min_points, sel.r0, sel.growth, P._r_max_device(cloud, tgt_d, bt))
    Y = torch.empty((7000, 1), dtype=torch.float64, device="cuda")
    ops, checks = D.map_chunked(cloud, tgt_d, dsel, P._rbf_pair(spec.rbf), 3, 0.0, True, X_d, Y,
                                2500, keep=True)
    assert len(ops) == 3 and all(int(st[0].item()) == 0 for _, _, st in checks)
    assert np.array_equal(Y.cpu().numpy(), want)


@pytest.mark.gpu
@pytest.mark.parametrize("lam", [0.0, 1e-6])
def test_supports_beyond_256_rows_vs_oracle(lam):
    """No support-size limit (the reference sizes its workspace from the
    largest support, _ext.pyx:305-312): ~400-point supports go through the
    warp-per-target fit (fm_big.cuh) -- one-shot, prepared, 3 components,
    and the fit_many seam -- and match the oracle."""
    from oracle import oracle as O
    from paper_2510_18838_b200 import _kernels as Kb
    from paper_2510_18838_b200 import pointwise as P

    side = np.linspace(0, 1, 120)
    xx, yy = np.meshgrid(side, side)
    src = np.ascontiguousarray(np.column_stack([xx.ravel(), yy.ravel()]))
    tgt = np.random.RandomState(3).uniform(0.2, 0.8, (300, 2))
    X = np.column_stack([np.sin((c + 1) * src[:, 0]) * np.cos(src[:, 1]) + 2 for c in range(3)])
    r = 0.095  # ~400 lattice points inside
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.FixedRadius(r), lam=lam)
    want, st, (off, idx, dist, w) = O.transfer(src, X, tgt, 2, O.RBF_C4, 2.0, ("fixed", r),
                                               lam=lam)
    assert (st == 0).all() and np.diff(off).min() > 256
    got1 = P.fit_point_cloud(src, X[:, 0], tgt, spec)
    assert np.max(np.abs(got1 - want[:, 0]) / np.abs(want[:, 0])) < 1e-10
    got = P.PreparedTransfer(src, tgt, spec).apply(X)
    assert np.max(np.abs(got - want) / np.abs(want)) < 1e-10
    v, c, s2 = Kb.fit_many(tgt, off, idx, w, src, X[:, 1], 2, lam, True)
    vw, cw, sw = O.fit_many(tgt, off, idx, w, src, X[:, 1], 2, lam, True)
    assert np.array_equal(s2, sw)
    assert np.max(np.abs(v - vw) / np.abs(vw)) < 1e-10
    assert np.max(np.abs(c - cw) / np.maximum(np.abs(cw), 1e-300)) < 1e-6


@pytest.mark.gpu
def test_graphed_transfer_equals_eager():
    """device.GraphedTransfer (the whole path replayed as one CUDA graph)
    gives bitwise the eager operator's result, reports validity, follows
    coordinates written into its tensors (same geometry: replay; new
    geometry: recapture), and flags an overflowing support as invalid."""
    import torch

    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200 import pointwise as P
    from paper_2510_18838_b200 import synth

    m = synth.disk_graded(1.0, 80, 0.6)
    src = m.coords
    tgt = synth.disk(1.0, 70).coords
    X = synth.sincos_field(src, 4)
    spec = P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0),
                     P.AdaptiveRadius(12, m.mean_edge_length, 1.5))
    s_d, t_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)
    gt = D.GraphedTransfer(s_d, t_d, X_d, spec)
    for _ in range(2):
        Y = gt.run().clone()
        assert gt.check()["valid"]
        assert np.array_equal(Y.cpu().numpy(), P.fit_point_cloud(src, X, tgt, spec))
    # new target coordinates in place (same bbox -> replay of the same graph)
    rot = tgt[::-1].copy()
    t_d.copy_(torch.from_numpy(rot))
    Y = gt.run()
    assert np.array_equal(Y.cpu().numpy(), P.fit_point_cloud(src, X, rot, spec))
    # new source geometry (different bbox -> recapture)
    src2 = src * 1.001 + 0.001
    s_d.copy_(torch.from_numpy(src2))
    Y = gt.run()
    assert gt.check()["valid"]
    assert np.array_equal(Y.cpu().numpy(), P.fit_point_cloud(src2, X, rot, spec))
    # a slot too small for the supports: the replay reports itself invalid
    gt2 = D.GraphedTransfer(s_d, t_d, X_d, spec, slot_cap=8)
    gt2.run()
    chk = gt2.check()
    assert chk["overflow"] > 0 and not chk["valid"]


@pytest.mark.gpu
def test_scan_tiles_and_edges():
    """The single-pass look-back scan (fm_scan.cuh) through fm_offsets_from_counts:
    exact int64 offsets for empty, one-element, partial-tile, exact multiples of
    the 8192-element tile (vector stores + the closing total), misaligned
    inputs (scalar path) and a 3M-element input with large counts."""
    import torch

    from paper_2510_18838_b200 import _lib
    from paper_2510_18838_b200.device import _stream

    L = _lib.lib()
    rs = np.random.RandomState(7)
    for n in (0, 1, 5, 8191, 8192, 8193, 16384, 3 * 8192 + 17, 3_000_000):
        for shift in ((0, 1) if n else (0,)):
            c = rs.randint(0, 1000 if n < 10**6 else 2000, n + shift).astype(np.int32)
            cd = torch.from_numpy(c).cuda()[shift:]  # shift 1: a 4-byte misaligned input
            off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            ws_bytes = L.fm_scan_workspace(n)
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
            _lib.check(L.fm_offsets_from_counts(_lib.ptr(cd) if n else None, n, _lib.ptr(off),
                                                _lib.ptr(ws), ws_bytes, _stream()),
                       "fm_offsets_from_counts")
            want = np.concatenate([[0], np.cumsum(c[shift:].astype(np.int64))])
            assert np.array_equal(off.cpu().numpy(), want), (n, shift)


@pytest.mark.gpu
def test_grid_binning_crowded_and_coincident_cells():
    """fm_grid_build's cell CSR (counting sort + in-cell id order) against a
    numpy restatement of the same cell formula (trunc(fl(p - lo) * inv_d),
    clamped; ids ascending per cell, the lexsort order of locate.py:79), at
    the default density, at the reference's 1 cell per point, and at 0.01
    cells per point (~100 points per cell: the heapsort path for cells of
    more than 64 points), with 3000 coincident duplicates in one cell."""
    from paper_2510_18838_b200 import device as D

    rs = np.random.RandomState(11)
    src = np.concatenate([rs.uniform(0, 1, (20000, 2)),
                          np.tile([[0.3, 0.7]], (3000, 1)),
                          rs.normal(0.6, 1e-3, (2000, 2))])
    src = src[rs.permutation(src.shape[0])]
    for cpp in (None, 1.0, 0.01):
        cloud = D.SourceCloud(src, cells_per_point=cpp)
        g = cloud.grid
        cells = np.zeros(src.shape[0], dtype=np.int64)
        stride = 1
        for a in range(2):
            ia = np.trunc((src[:, a] - g.lo[a]) * g.inv_d[a]).astype(np.int64)
            cells += np.clip(ia, 0, g.n[a] - 1) * stride
            stride *= g.n[a]
        ids = np.arange(src.shape[0])
        order = np.lexsort((ids, cells))
        start = np.zeros(g.ncell + 1, dtype=np.int64)
        np.add.at(start, cells + 1, 1)
        np.cumsum(start, out=start)
        assert np.array_equal(cloud.cell_start.cpu().numpy(), start), cpp
        assert np.array_equal(cloud.sorted_ids.cpu().numpy(), ids[order]), cpp
        assert np.array_equal(cloud.sorted_pts.cpu().numpy(), src[order]), cpp


@pytest.mark.gpu
def test_graphed_transfer_flags_unbuilt_bucket():
    """GraphedTransfer captures only the size buckets its first geometry
    fills; a replay whose supports land in another bucket (same capture key:
    fixed radius, same sources) must report itself invalid, and a fresh
    transfer of that input gives the oracle's values."""
    from paper_2510_18838_b200 import device as D
    from paper_2510_18838_b200 import pointwise as P

    rs = np.random.RandomState(5)
    dense = rs.uniform(0.0, 0.5, (2000, 2)) * [1, 2]  # ~2x the density: m ~ 31
    sparse = rs.uniform(0.5, 1.0, (1000, 2)) * [1, 2]
    src = np.concatenate([dense, sparse])
    X = np.stack([np.sin(3 * src[:, 0]), np.cos(2 * src[:, 1])], 1)
    spec = P.FitSpec(1, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.FixedRadius(0.05))
    t_sparse = rs.uniform(0.6, 0.9, (500, 2)) * [1, 2]
    t_dense = rs.uniform(0.1, 0.4, (500, 2)) * [1, 2]
    tgt_d = D.to_device(t_sparse)
    gt = D.GraphedTransfer(D.to_device(src), tgt_d, D.to_device(X), spec)
    Y = gt.run()
    c = gt.check()
    assert c["valid"], c
    assert np.allclose(Y.cpu().numpy(), P.fit_point_cloud(src, X, t_sparse, spec), rtol=1e-12,
                       atol=0)
    tgt_d.copy_(D.to_device(t_dense))  # ~2x the points per support: other buckets
    gt.run()
    c = gt.check()
    assert c["unbuilt_bucket"] and not c["valid"], c
