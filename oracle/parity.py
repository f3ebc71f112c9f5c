"""Full-scale parity check of a device transfer against the CPU oracle
(TEST INFRASTRUCTURE ONLY).

Only tests/ and bench.py (outside its timed region, as the checker of the
benchmarked workload) call this; the product package never imports it.

`check_transfer` runs the whole reference path on the host cores with the
oracle restatement of _ext.pyx (oracle/fb_oracle.c, OpenMP across targets;
the restatement is pinned bitwise against the reference in
tests/test_oracle.py):

  PointGrid (locate.py:144-161)  -> adaptive/fixed radius supports
  (_ext.pyx:203-288)             -> rbf weights at the selection radius
  (pointwise.py:250, 266-269)    -> |w| (pointwise.py:301)
  -> fit_many per component (_ext.pyx:291-426, LAPACK dgelsy)

and compares the device outputs with it:
  * the neighbour CSR (offsets, ids, distances), the adaptive radii and the
    selection status: bitwise (np.array_equal on the raw doubles);
  * the fit status: equal;
  * the values: max |y - y_ref| / |y_ref| over every target and component,
    against `rtol` (the north-star 1e-10).  Targets above it are counted and
    their cond(A) reported (two backward-stable least-squares solvers differ
    by ~eps * cond(A)^2 * |r| / |b|).
"""

import os
import time

import numpy as np

from . import oracle as O
from .pointgrid import OraclePointGrid


def cond_of_fit(src, target, idx, w, degree, centering=True):
    """cond_2 of the weighted scaled Vandermonde the reference factors
    (_ext.pyx:353-394) for one target."""
    src = np.asarray(src, dtype=np.float64)
    dim = src.shape[1]
    parent, var, _deg = O.monomial_table(dim, degree)
    dx = src[idx] - target if centering else src[idx].copy()
    s = np.sqrt(np.max(np.sum(dx * dx, axis=1))) or 1.0
    u = dx / s
    k = parent.shape[0]
    A = np.empty((idx.shape[0], k))
    A[:, 0] = 1.0
    for c in range(1, k):
        A[:, c] = u[:, var[c]] if parent[c] == 0 else A[:, parent[c]] * u[:, var[c]]
    A *= np.asarray(w)[:, None]
    return float(np.linalg.cond(A))


def oracle_transfer(src, X, tgt, degree, kind, a, selection, lam=0.0, centering=True,
                    nthreads=None, r_max=None):
    """The reference path on the host (see module docstring).  Returns a dict
    with off/idx/dist[/radii/status], w, values (nt, C), fit_status."""
    nthreads = nthreads or os.cpu_count() or 1
    src = np.ascontiguousarray(src, dtype=np.float64)
    tgt = np.ascontiguousarray(tgt, dtype=np.float64).reshape(-1, src.shape[1])
    t0 = time.perf_counter()
    grid = OraclePointGrid(src)
    out = {}
    if selection[0] == "fixed":
        off, idx, dist = O.supports_nd(tgt, grid, float(selection[1]), nthreads)
        radius = float(selection[1])
    else:
        _, min_pts, r0, growth = selection
        rm = O.r_max_for(src, tgt) if r_max is None else float(r_max)
        off, idx, dist, radii, st = O.supports_nd(
            tgt, grid, (int(min_pts), float(r0), float(growth), rm), nthreads)
        out.update(radii=radii, status=st)
        radius = radii
    w = np.abs(O.rbf_for_supports(kind, a, off, dist, radius))
    values, _c, fst = O.fit_many_nd(tgt, off, idx, w, src, X, degree, lam, centering, nthreads)
    out.update(off=off, idx=idx, dist=dist, w=w, values=values, fit_status=fst,
               seconds=time.perf_counter() - t0, threads=nthreads)
    return out


def check_transfer(src, X, tgt, degree, kind, a, selection, dev, lam=0.0, centering=True,
                   rtol=1e-10, nthreads=None, ref=None):
    """Compare device results `dev` (dict with numpy off, idx, dist, values
    and optionally radii, status, fit_status) with the oracle.  Returns a
    JSON-able summary; `ref` may pass a precomputed oracle_transfer()."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    tgt = np.ascontiguousarray(tgt, dtype=np.float64).reshape(-1, src.shape[1])
    X2 = np.asarray(X, dtype=np.float64).reshape(src.shape[0], -1)
    if ref is None:
        ref = oracle_transfer(src, X2, tgt, degree, kind, a, selection, lam, centering,
                              nthreads)
    r = {"targets": int(tgt.shape[0]), "components": int(X2.shape[1]),
         "nnz": int(ref["off"][-1]), "oracle": "oracle/fb_oracle.c (restated _ext.pyx, "
         "pinned bitwise to the reference), OpenMP", "oracle_threads": ref["threads"],
         "oracle_seconds": round(ref["seconds"], 2)}
    r["supports_bitwise"] = bool(
        np.array_equal(np.asarray(dev["off"], np.int64), ref["off"])
        and np.array_equal(np.asarray(dev["idx"], np.int64), ref["idx"])
        and np.array_equal(np.asarray(dev["dist"]).view(np.int64), ref["dist"].view(np.int64)))
    if "radii" in ref:
        r["radii_bitwise"] = bool(np.array_equal(np.asarray(dev["radii"]).view(np.int64),
                                                 ref["radii"].view(np.int64)))
        r["select_status_equal"] = bool(np.array_equal(np.asarray(dev["status"]),
                                                       ref["status"]))
    if dev.get("fit_status") is not None:
        r["fit_status_equal"] = bool(np.array_equal(np.asarray(dev["fit_status"]),
                                                    ref["fit_status"]))
        r["fit_failures"] = int(np.count_nonzero(ref["fit_status"]))
    y = np.asarray(dev["values"], dtype=np.float64).reshape(tgt.shape[0], -1)
    yr = ref["values"].reshape(tgt.shape[0], -1)
    ok = ref["fit_status"] == 0
    rel = np.abs(y[ok] - yr[ok]) / np.maximum(np.abs(yr[ok]), np.finfo(float).tiny)
    per_t = rel.max(axis=1) if rel.size else np.zeros(0)
    r["max_rel"] = float(per_t.max()) if per_t.size else 0.0
    r["median_rel"] = float(np.median(per_t)) if per_t.size else 0.0
    r["rtol"] = rtol
    bad = np.flatnonzero(ok)[per_t > rtol] if per_t.size else np.zeros(0, np.int64)
    r["n_above_rtol"] = int(bad.size)
    if bad.size:
        worst = bad[np.argsort(-per_t[per_t > rtol])[:5]]
        off = ref["off"]
        r["worst"] = [{"target": int(i), "rel": float(np.max(
            np.abs(y[i] - yr[i]) / np.abs(yr[i]))), "cond_A": cond_of_fit(
                src, tgt[i], ref["idx"][off[i]:off[i + 1]], ref["w"][off[i]:off[i + 1]],
                degree, centering)} for i in worst]
    r["values_within_rtol"] = r["n_above_rtol"] == 0
    return r
