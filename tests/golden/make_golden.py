"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only in the build container, where /root/reference exists: it imports
the reference package `fieldbridge` with its compiled Cython backend
(oracle/_ref, built by `make -C oracle ref` from the reference's own
_ext.pyx) and records inputs + outputs of the hot-path calls as small .npz
files.  The GPU box never needs the reference: tests read these files.

    python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

fb = ref.import_reference_package()
K = fb._kernels
from fieldbridge.pointwise import PreparedTransfer  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{path}: {os.path.getsize(path) / 1024:.1f} KiB")


def rbf_table():
    r = np.concatenate([[0.0], np.linspace(0.0, 0.7, 71)[1:], [0.7000000001, 0.9]])
    out = {"r": r}
    for kind in range(8):
        out[f"w{kind}"] = K.rbf_weights(kind, 2.0, 0.7, r)
    save("rbf", **out)


def disk_small():
    m = fb.disk(1.0, 8)
    t = np.ascontiguousarray(m.centroids()[:50])
    pg = fb.build_point_grid(m.coords)
    off, idx, dist = K.fixed_radius_supports(t, pg.points, float(pg.lo[0]), float(pg.lo[1]),
                                             pg.dx, pg.dy, pg.nx, pg.ny, pg.cell_offsets,
                                             pg.cell_items, 0.3)
    save("disk_small", coords=m.coords, tris=m.tris, centroids=m.centroids(),
         mean_edge_length=m.mean_edge_length, grid_lo=pg.lo, grid_n=np.array([pg.nx, pg.ny]),
         grid_d=np.array([pg.dx, pg.dy]), cell_offsets=pg.cell_offsets,
         cell_items=pg.cell_items, rq_off=off, rq_idx=idx, rq_dist=dist)


def c1():
    m = fb.square(99)
    src = m.coords
    tg = np.random.RandomState(0).uniform(0, 1, (10000, 2))
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    h = m.mean_edge_length
    pg = fb.build_point_grid(src)
    off, idx, dist = K.fixed_radius_supports(tg, pg.points, float(pg.lo[0]), float(pg.lo[1]),
                                             pg.dx, pg.dy, pg.nx, pg.ny, pg.cell_offsets,
                                             pg.cell_items, 2 * h)
    spec = fb.FitSpec(2, fb.RadialBasisSpec(fb.RbfKind.C4, a=2.0), fb.FixedRadius(2 * h))
    values = fb.fit_point_cloud(src, vals, tg, spec)
    w = np.abs(K.rbf_weights(K.RBF_C4, 2.0, 2 * h, dist))
    # fit_many variants on the first 600 targets (all degrees, ridge, centering)
    n = 600
    fits = {}
    for deg in (0, 1, 2):
        for lam in (0.0, 1e-6):
            for cen in (True, False):
                v, c, st = K.fit_many(tg[:n], off[:n + 1], idx, w, src, vals, deg, lam, cen)
                key = f"d{deg}_l{'r' if lam else '0'}_{'c' if cen else 'u'}"
                fits["fit_v_" + key] = v
                fits["fit_c_" + key] = c
                fits["fit_s_" + key] = st
    keep = off[1000]
    save("c1", mean_edge_length=h, values=values, counts=np.diff(off).astype(np.int16),
         off1000=off[:1001], idx1000=idx[:keep], dist1000=dist[:keep], nnz=off[-1], **fits)


def adaptive():
    srcm = fb.disk_graded(1.0, 30, 0.6)
    tgm = fb.disk(1.0, 30)
    src, tg = srcm.coords, tgm.coords
    h = srcm.mean_edge_length
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    pg = fb.build_point_grid(src)
    span = np.vstack([src, tg])
    lo, hi = span.min(axis=0), span.max(axis=0)
    r_max = 1.0000001 * float(np.hypot(hi[0] - lo[0], hi[1] - lo[1])) + 1e-300
    off, idx, dist, radii, status = K.adaptive_radius_supports(
        tg, pg.points, float(pg.lo[0]), float(pg.lo[1]), pg.dx, pg.dy, pg.nx, pg.ny,
        pg.cell_offsets, pg.cell_items, 12, h, 1.5, r_max)
    spec = fb.FitSpec(2, fb.RadialBasisSpec(fb.RbfKind.C4, a=2.0), fb.AdaptiveRadius(12, h, 1.5))
    pt = PreparedTransfer(src, tg, spec)
    vals8 = np.stack([np.sin((c + 1) * src[:, 0]) * np.cos(src[:, 1]) + 2 for c in range(3)], 1)
    applied = np.stack([pt.apply(vals8[:, c]) for c in range(3)], 1)
    save("adaptive", src_n_rings=30, mean_edge_length=h, r_max=r_max, off=off, idx=idx,
         dist=dist, radii=radii, status=status, values3=applied)


def poly_repro():
    m = fb.disk(1.0, 8)
    polys = {
        0: lambda x, y: np.full_like(x, 3.5),
        1: lambda x, y: 2 * x - y + 1,
        2: lambda x, y: x * x + 2 * x * y - y * y + x + 0.5,
    }
    out = {}
    h = m.mean_edge_length
    for kind in fb.RbfKind:
        for deg in (0, 1, 2):
            f = fb.sample_field(m, polys[deg], "vertices", 1)
            spec = fb.FitSpec(deg, fb.RadialBasisSpec(kind, a=2.0),
                              fb.AdaptiveRadius(max(6, 2 * fb.pointwise.n_monomials(deg)),
                                                1.5 * h, 1.5), lam=0.0)
            out[f"{kind.value}_{deg}"] = fb.transfer_pointwise(f, m.centroids(), spec)
    # fixed-radius C4 degree 1 (dense-LS oracle test) and Gaussian 2.5h
    f = fb.sample_field(m, lambda x, y: np.sin(x) * np.cos(y) + 2, "vertices", 1)
    out["fixed_c4_1"] = fb.transfer_pointwise(
        f, m.centroids(), fb.FitSpec(1, fb.RadialBasisSpec(fb.RbfKind.C4), fb.FixedRadius(2 * h)))
    save("poly_repro", **out)


def random_clouds():
    rs1, rs2 = np.random.RandomState(1), np.random.RandomState(2)
    src = rs1.uniform(0, 1, (20000, 2))
    tg = rs2.uniform(0, 1, (4000, 2))
    vals = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
    out = {"src": src, "tg": tg}
    for kind in (fb.RbfKind.GAUSSIAN, fb.RbfKind.MULTIQUADRIC):
        spec = fb.FitSpec(2, fb.RadialBasisSpec(kind, a=2.0),
                          fb.AdaptiveRadius(12, 1.5 / np.sqrt(src.shape[0]), 1.5))
        out[kind.value] = fb.fit_point_cloud(src, vals, tg, spec)
    save("random_clouds", **out)


def singular_cases():
    rng = np.random.RandomState(7)
    pts_l, vals_l, w_l, off = [], [], [], [0]
    tg = []
    degs = []
    for trial in range(400):
        deg = 1 + trial % 2
        k = (deg + 1) * (deg + 2) // 2
        m = rng.randint(k, 20)
        x = rng.uniform(-1, 1, m)
        delta = 10.0 ** rng.uniform(-19, -4)
        y = (0.3 * x if deg == 1 else 0.3 * x * x) + delta * rng.randn(m)
        pts_l.append(np.column_stack([x, y]))
        vals_l.append(rng.randn(m))
        w_l.append(rng.uniform(0.5, 2, m))
        off.append(off[-1] + m)
        tg.append([0.01, 0.02])
        degs.append(deg)
    pts = np.vstack(pts_l)
    vals = np.concatenate(vals_l)
    w = np.concatenate(w_l)
    off = np.array(off)
    tg = np.array(tg)
    degs = np.array(degs)
    st = np.zeros(len(degs), np.uint8)
    v = np.zeros(len(degs))
    cond = np.zeros(len(degs))
    for i in range(len(degs)):
        sl = slice(off[i], off[i + 1])
        vi, _c, si = K.fit_many(tg[i:i + 1], np.array([0, off[i + 1] - off[i]]),
                                np.arange(off[i + 1] - off[i]), w[sl], pts[sl], vals[sl],
                                int(degs[i]), 0.0, True)
        st[i], v[i] = si[0], vi[0]
        d = pts[sl] - tg[i]
        s = np.sqrt(np.max(d[:, 0] ** 2 + d[:, 1] ** 2))
        u, vv = d[:, 0] / s, d[:, 1] / s
        cols = [np.ones_like(u), u, vv, u * u, u * vv, vv * vv][:(degs[i] + 1) * (degs[i] + 2) // 2]
        cond[i] = np.linalg.cond(np.stack(cols, 1) * w[sl][:, None])
    save("singular", pts=pts, vals=vals, w=w, off=off, tg=tg, degs=degs, status=st, values=v,
         cond=cond)


def fit_local_cases():
    out = {}
    rng = np.random.RandomState(1)
    pts = rng.uniform(-1, 1, size=(8, 2))
    w = rng.uniform(0.1, 2.0, size=8)
    out["const_pts"], out["const_w"] = pts, w
    out["const_c"] = fb.fit_local((0.1, -0.2), pts, np.full(8, 7.0), w, degree=2)
    rng = np.random.RandomState(2)
    pts = rng.uniform(-1, 1, size=(10, 2))
    vals = rng.randn(10)
    out["ridge_pts"], out["ridge_vals"] = pts, vals
    for lam in (0.0, 1e2, 1e4, 1e6):
        out[f"ridge_c_{lam:g}"] = fb.fit_local((0.0, 0.0), pts, vals, np.ones(10), degree=1,
                                               lam=lam)
    pts = np.array([[0.0, 0.0], [0.5, 0.5], [1.0, 1.0], [0.25, 0.25]])
    out["collinear_ridge_c"] = fb.fit_local((0.5, 0.5), pts, np.array([0.0, 1.0, 2.0, 0.5]),
                                            np.ones(4), degree=1, lam=1e-8)
    save("fit_local", **out)


def locate_cases():
    """locate_batch (_ext.pyx:88-152) on two meshes with the reference's own
    UniformGrid: interior points, vertices (dim 0), edge midpoints (dim 1),
    centroids (dim 2), points just outside (tol halo) and far outside."""
    out = {}
    for name, m in (("sq", fb.square(12)), ("disk", fb.disk(1.0, 6))):
        g = fb.build_grid(m)
        rng = np.random.RandomState(7)
        lo, hi = m.bbox[0], m.bbox[1]
        span = hi - lo
        e = m.edges
        mids = 0.5 * (m.coords[e[:, 0]] + m.coords[e[:, 1]])
        pts = np.concatenate([
            rng.uniform(lo - 0.1 * span, hi + 0.1 * span, (400, 2)),
            m.coords, mids, m.centroids(),
            m.coords + 1e-12 * rng.standard_normal(m.coords.shape),
            mids + 3e-11 * rng.standard_normal(mids.shape),
        ])
        pts = np.ascontiguousarray(pts)
        for tol in (1e-10, 0.0, 1e-6):
            res = K.locate_batch(pts, m.tri_xy, m.tris, m.tri_edges, m.vert_gid, m.tri_gid,
                                 m.inv2a, m.epsfac, float(g.lo[0]), float(g.lo[1]), g.dx, g.dy,
                                 g.nx, g.ny, g.cell_offsets, g.cell_items, tol)
            for k, a in zip(("found", "elem", "dim", "ent", "bary"), res):
                out[f"{name}_{tol:g}_{k}"] = a
        out.update({f"{name}_pts": pts, f"{name}_tri_xy": m.tri_xy, f"{name}_tris": m.tris,
                    f"{name}_tri_edges": m.tri_edges, f"{name}_vert_gid": m.vert_gid,
                    f"{name}_tri_gid": m.tri_gid, f"{name}_inv2a": m.inv2a,
                    f"{name}_epsfac": m.epsfac,
                    f"{name}_grid": np.array([g.lo[0], g.lo[1], g.dx, g.dy]),
                    f"{name}_grid_n": np.array([g.nx, g.ny]),
                    f"{name}_cell_off": g.cell_offsets, f"{name}_cell_items": g.cell_items})
    save("locate", **out)


def patch_cases():
    """ElementPatch supports: the reference's own _PatchTopology.patch_dofs
    (pointwise.py:190-230) for every element of two meshes as seed, layers
    1-3, vertex and centroid dofs."""
    from fieldbridge.pointwise import _PatchTopology

    out = {}
    for name, m in (("sq", fb.square(12)), ("disk", fb.disk(1.0, 6))):
        out[f"{name}_tris"] = m.tris
        out[f"{name}_edge_tris"] = m.edge_tris
        seeds = np.arange(m.tris.shape[0], dtype=np.int64)
        for loc in ("vertices", "centroids"):
            topo = _PatchTopology(m, loc)
            for layers in (1, 2, 3):
                parts = [topo.patch_dofs(int(s), layers) for s in seeds]
                off = np.concatenate([[0], np.cumsum([p.size for p in parts])]).astype(np.int64)
                out[f"{name}_{loc}_{layers}_off"] = off
                out[f"{name}_{loc}_{layers}_idx"] = np.concatenate(parts).astype(np.int64)
    # the public API on ElementPatch (pointwise.py:434-451, 317-336):
    # fit_point_cloud values and select_support, with the mesh arrays the
    # device path needs (tests rebuild a mesh-like namespace from them)
    from fieldbridge.pointwise import (ElementPatch, FitSpec, RadialBasisSpec, RbfKind,
                                       fit_point_cloud, select_support)

    for name, m in (("sq", fb.square(12)), ("disk", fb.disk(1.0, 6))):
        for k in ("coords", "tri_xy", "tri_edges", "vert_gid", "tri_gid", "inv2a", "epsfac",
                  "diameters", "bbox"):
            out[f"{name}_{k}"] = getattr(m, k)
        g = fb.build_grid(m)
        out[f"{name}_grid"] = np.array([g.lo[0], g.lo[1], g.dx, g.dy])
        out[f"{name}_grid_n"] = np.array([g.nx, g.ny])
        out[f"{name}_cell_off"] = g.cell_offsets
        out[f"{name}_cell_items"] = g.cell_items
        rng = np.random.RandomState(13)
        if name == "sq":
            t = rng.uniform(0.0, 1.0, (500, 2))
        else:
            r = 0.95 * np.sqrt(rng.uniform(0, 1, 500))
            a = rng.uniform(0, 2 * np.pi, 500)
            t = np.stack([r * np.cos(a), r * np.sin(a)], axis=1)
        out[f"{name}_targets"] = t
        cen = m.centroids()
        out[f"{name}_centroids"] = cen
        for loc, src in (("vertices", m.coords), ("centroids", cen)):
            f = np.sin(src[:, 0]) * np.cos(src[:, 1]) + 2
            for deg, layers in ((1, 2), (2, 3)):
                spec = FitSpec(deg, RadialBasisSpec(RbfKind.CONST, r_c=None),
                               ElementPatch(layers))
                out[f"{name}_{loc}_fit_{deg}_{layers}"] = fit_point_cloud(
                    src, f, t, spec, mesh=m, source_location=loc)
            idx, w = select_support(t[0], src, ElementPatch(2), fit_degree=2, mesh=m,
                                    source_location=loc)
            out[f"{name}_{loc}_sel_idx"] = idx
            out[f"{name}_{loc}_sel_w"] = w
    save("patch", **out)


def cycle_cases():
    """metrics._PointwiseCycle (metrics.py:127-148): fields after 1 and 3
    vertex -> centroid -> vertex cycles on one mesh, and after 2 cycles
    between two meshes, for a radius selection and an element patch."""
    from fieldbridge.metrics import _PointwiseCycle
    from fieldbridge.pointwise import (AdaptiveRadius, ElementPatch, FitSpec, RadialBasisSpec,
                                       RbfKind)

    m, m2 = fb.square(12), fb.square(9)
    out = {}
    for name, mm in (("a", m), ("b", m2)):
        for k in ("coords", "tris", "edge_tris", "tri_xy", "tri_edges", "vert_gid", "tri_gid",
                  "inv2a", "epsfac", "diameters", "bbox"):
            out[f"{name}_{k}"] = getattr(mm, k)
        out[f"{name}_centroids"] = mm.centroids()
    f0 = np.sin(m.coords[:, 0]) * np.cos(m.coords[:, 1]) + 2
    out["f0"] = f0
    out["mean_edge_length"] = np.float64(m.mean_edge_length)
    specs = {
        "adaptive": FitSpec(2, RadialBasisSpec(RbfKind.C4, a=2.0),
                            AdaptiveRadius(12, m.mean_edge_length, 1.5)),
        "patch": FitSpec(1, RadialBasisSpec(RbfKind.CONST, r_c=None), ElementPatch(2)),
    }
    for key, spec in specs.items():
        cyc = _PointwiseCycle(m, spec, None)
        v = f0
        for it in range(1, 4):
            v = cyc.cycle(v)
            if it in (1, 3):
                out[f"{key}_one_{it}"] = v
        cyc2 = _PointwiseCycle(m, spec, m2)
        v = f0
        for it in range(2):
            v = cyc2.cycle(v)
        out[f"{key}_two_2"] = v
    save("cycle", **out)


def rendezvous_cases():
    """coupled_transfer's pointwise branch (rendezvous.py:452-495, 601-629):
    two square meshes partitioned by rcb, a rendezvous grid, the coupled
    field and the MessageStats table, for several rank counts."""
    from fieldbridge.rendezvous import build_rdv_partition, coupled_transfer, rcb_partition
    from fieldbridge.pointwise import FitSpec, FixedRadius, RadialBasisSpec, RbfKind

    ma, mb = fb.square(30), fb.square(22)
    f = np.sin(ma.coords[:, 0]) * np.cos(ma.coords[:, 1]) + 2
    field = fb.Field(ma, "vertices", 1, f)
    lo = np.minimum(ma.bbox[0], mb.bbox[0])
    hi = np.maximum(ma.bbox[1], mb.bbox[1])
    r_c = 2.0 * ma.mean_edge_length
    spec = FitSpec(2, RadialBasisSpec(RbfKind.C4, a=2.0), FixedRadius(r_c))
    out = {"coords_a": ma.coords, "values_a": f, "coords_b": mb.coords, "lo": lo, "hi": hi,
           "r_c": r_c}
    for na, nb, nr, grid in ((4, 2, 3, (6, 5)), (2, 4, 4, (7, 7)), (1, 1, 1, (3, 3))):
        rdv = build_rdv_partition((lo, hi), grid[0], grid[1], nr)
        pa, pb = rcb_partition(ma, na), rcb_partition(mb, nb)
        res, stats = coupled_transfer(field, pa, mb, pb, rdv, spec)
        key = f"{na}_{nb}_{nr}"
        out[f"own_a_{key}"] = pa.dof_owner("vertices")
        out[f"own_b_{key}"] = pb.dof_owner("vertices")
        out[f"grid_{key}"] = np.array(grid)
        out[f"values_{key}"] = res.values
        out[f"stats_{key}"] = np.array([row[2:] for row in stats.table()], dtype=np.int64)
        out[f"stats_roles_{key}"] = np.array([f"{row[0]}:{row[1]}" for row in stats.table()])
    save("rendezvous", **out)


if __name__ == "__main__":
    rendezvous_cases()
    cycle_cases()
    patch_cases()
    locate_cases()
    rbf_table()
    disk_small()
    c1()
    adaptive()
    poly_repro()
    random_clouds()
    singular_cases()
    fit_local_cases()
