"""Measure ElementPatch selection at scale.

    python scripts/bench_patch.py [--n 1000] [--layers 2] [--targets 1000000]

Synthetic structured triangle mesh of the unit square: (n+1)^2 vertices,
2n^2 triangles (each lattice cell split along its diagonal), edge_tris built
with numpy.  Seeds are uniformly random elements.  Times fm_patch_count +
fm_patch_fill (CUDA events, best of 5 after warm-up, inputs resident) and the
patch fit (degree 2, unit weights) of a scalar field, and the oracle's
plain-Python BFS (the reference's algorithm, pointwise.py:212-230) on a
bounded sample on one host core.  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18838_b200 import device as D  # noqa: E402


def square_mesh(n):
    xs = np.linspace(0.0, 1.0, n + 1)
    X, Y = np.meshgrid(xs, xs)
    coords = np.stack([X.ravel(), Y.ravel()], axis=1)
    i, j = np.meshgrid(np.arange(n), np.arange(n))
    v0 = (j * (n + 1) + i).ravel()
    v1, v2, v3 = v0 + 1, v0 + n + 2, v0 + n + 1
    tris = np.concatenate([np.stack([v0, v1, v2], 1), np.stack([v0, v2, v3], 1)])
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
    e.sort(axis=1)
    owner = np.tile(np.arange(tris.shape[0]), 3)
    _, inv = np.unique(e[:, 0] * (coords.shape[0] + 1) + e[:, 1], return_inverse=True)
    order = np.argsort(inv, kind="stable")
    inv_s, own_s = inv[order], owner[order]
    nedge = int(inv.max()) + 1
    edge_tris = np.full((nedge, 2), -1, dtype=np.int64)
    first = np.ones(inv_s.size, dtype=bool)
    first[1:] = inv_s[1:] != inv_s[:-1]
    edge_tris[inv_s[first], 0] = own_s[first]
    edge_tris[inv_s[~first], 1] = own_s[~first]
    return coords, tris.astype(np.int64), edge_tris


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--targets", type=int, default=1_000_000)
    ap.add_argument("--cpu-sample", type=int, default=20000)
    a = ap.parse_args()
    coords, tris, edge_tris = square_mesh(a.n)
    rng = np.random.default_rng(0)
    seeds = rng.integers(0, tris.shape[0], a.targets)
    topo = D.PatchTopology.from_mesh_arrays(tris, edge_tris)
    seed_d = D.to_device(seeds, torch.int64)
    res = {"workload": f"square mesh n={a.n} ({tris.shape[0]} triangles), {a.targets} random "
                       f"seed elements, layers={a.layers}, vertex dofs"}
    for cen in (False, True):
        ms, (off, idx, counts) = timed(lambda: D.patch_supports(topo, seed_d, a.layers, cen))
        key = "centroids" if cen else "vertices"
        res[f"patch_{key}_ms"] = ms
        res[f"patch_{key}_targets_per_s"] = a.targets / (ms * 1e-3)
        res[f"nnz_{key}"] = int(off[-1])
        if not cen:
            off_v, idx_v = off, idx
            ms_u, _ = timed(lambda: D.patch_supports(topo, seed_d, a.layers, cen,
                                                     sort_by_seed=False))
            res["patch_vertices_unsorted_ms"] = ms_u
            res["seed_argsort_ms"], _ = timed(lambda: torch.argsort(seed_d.to(torch.int32)))
    # patch fit, degree 2, unit weights, scalar field (fm_fit_many)
    src = D.to_device(coords)
    f = D.to_device(np.sin(coords[:, 0]) * np.cos(coords[:, 1]) + 2)
    t = src[D.to_device(tris[seeds, 0], torch.int64)] * 0.5 + src[
        D.to_device(tris[seeds, 1], torch.int64)] * 0.25 + src[
        D.to_device(tris[seeds, 2], torch.int64)] * 0.25
    w = torch.ones(idx_v.shape[0], dtype=torch.float64, device=src.device)
    max_m = int((off_v[1:] - off_v[:-1]).max())
    ms_fit, (vals, _, status, _) = timed(lambda: D.fit_many(t.contiguous(), off_v, idx_v, w, src,
                                                            f, 2, 0.0, True, max_m))
    res["fit_ms"] = ms_fit
    res["patch_plus_fit_targets_per_s"] = a.targets / ((res["patch_vertices_ms"] + ms_fit) * 1e-3)
    tx, ty = t[:, 0].cpu().numpy(), t[:, 1].cpu().numpy()
    ok = status.cpu().numpy() == 0
    res["fit_ok_frac"] = float(ok.mean())
    res["max_abs_err_vs_field"] = float(np.abs(vals.cpu().numpy()[ok] -
                                               (np.sin(tx) * np.cos(ty) + 2)[ok]).max())
    # parity on a sample + the reference algorithm on one host core
    from oracle import oracle as O

    s = min(a.cpu_sample, a.targets)
    t0 = time.perf_counter()
    w_off, w_idx = O.patch_supports(seeds[:s], edge_tris, tris, a.layers, False)
    cpu_s = time.perf_counter() - t0
    off_h = off_v[:s + 1].cpu().numpy()
    res["parity_sample_bitwise"] = bool(np.array_equal(off_h, w_off) and np.array_equal(
        idx_v[:int(off_h[-1])].cpu().numpy(), w_idx))
    res["cpu_baseline"] = {"value": s / cpu_s, "unit": "targets/s", "cores": 1, "kind": "port",
                           "sample": f"first {s} seeds, plain-Python BFS (oracle.patch_supports; "
                                     "the reference's patch_dofs algorithm, adjacency prebuilt)"}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
