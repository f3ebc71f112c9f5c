"""Device-resident hot path: torch tensors in HBM, compute in libfieldmap.so.

PyTorch only provides memory, streams and host<->device copies here; every
arithmetic step of the path is one of the library's sm_100a kernels:

  SourceCloud          a1  source binning (fm_grid_build)       locate.py:144-161
  count_supports       a3/a4 count / radius growth              _ext.pyx:203-288
  fill_supports        a3/a4 fill + a5 weights                  _ext.pyx:225-287
  fit_many             a7  fit_many                             _ext.pyx:291-426
  transfer_values      a9  one-shot fused transfer              pointwise.py:434-451
  Operator / build     a8  explicit transfer operator           pointwise.py:399-431
  Operator.apply       a13 CSR SpMM over field components

All launches go on torch's current CUDA stream.
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import FM_MAX_DIM, FmFit, FmGrid, FmLists, FmRbf, FmSelect, check, ptr

INT32_MAX = 2 ** 31 - 1
# capacities of the global-scratch patch path (targets beyond FM_PATCH_MAX_*)
PATCH_BIG_ELEMS = 16384
PATCH_BIG_DOFS = 32768


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def to_device(a, dtype=torch.float64):
    """numpy / torch -> contiguous CUDA tensor (no copy if already there)."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            return a.to(dtype=dtype).contiguous()
        # host tensor: pinned memory makes this an async H2D copy on the stream
        return a.to(dtype=dtype).contiguous().to(_dev(), non_blocking=a.is_pinned())
    arr = np.ascontiguousarray(a, dtype=np.float64 if dtype == torch.float64 else None)
    if not arr.flags.writeable:  # torch.from_numpy wants a writable buffer
        arr = arr.copy()
    return torch.from_numpy(arr).to(_dev(), non_blocking=False)


def _empty(shape, dtype, device):
    return torch.empty(shape, dtype=dtype, device=device)


def _workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ a1
# Source grid density (cells per source point).  The search grid is ours:
# the supports and radii do not depend on it (§3), only the discovery order
# of a support's points -- the fit's row order, i.e. its rounding -- does.
# 1-D/2-D (thread-per-target select): 0.35 cells per point, measured fastest
# on C2 (select 0.417 -> 0.356 ms: fewer, longer window rows); dim >= 3: 1.
# Env FM_CELLS_PER_POINT overrides (A/B).
_CELLS_PER_POINT_ENV = os.environ.get("FM_CELLS_PER_POINT")


def default_cells_per_point(dim):
    if _CELLS_PER_POINT_ENV:
        return float(_CELLS_PER_POINT_ENV)
    return 0.35 if dim <= 2 else 1.0


class SourceCloud:
    """Source points resident in HBM and binned into a uniform grid.

    `points` (n, dim) fp64, dim 1..5.  The grid geometry follows the
    reference's PointGrid rules (locate.py:144-161: padded bbox, ~cells_per_point
    cells per point; at 1.0 and dim 2 the very same nx, ny, lo, dx, dy) at
    `default_cells_per_point(dim)`.  Supports and radii do not depend on the
    geometry."""

    def __init__(self, points, cells_per_point=None, bbox=None, geom=None):
        if cells_per_point is None:
            cells_per_point = default_cells_per_point(
                points.shape[1] if getattr(points, "ndim", 1) == 2 else 2)
        host = None if isinstance(points, torch.Tensor) else np.ascontiguousarray(points,
                                                                                  dtype=np.float64)
        self.pts = to_device(points if host is None else host)
        if self.pts.ndim != 2 or not 1 <= self.pts.shape[1] <= 5 or self.pts.shape[0] == 0:
            raise ValueError("points must be a nonempty (n, d) array with 1 <= d <= 5")
        self.n, self.dim = self.pts.shape
        L = _lib.lib()
        if geom is None:
            if bbox is None:
                if host is not None:
                    bbox = (host.min(axis=0), host.max(axis=0))
                else:
                    bbox = device_bbox(self.pts)
            # the PointGrid geometry (locate.grid_geometry) computed in C
            self.grid = FmGrid()
            lo = np.ascontiguousarray(bbox[0], dtype=np.float64)
            hi = np.ascontiguousarray(bbox[1], dtype=np.float64)
            check(L.fm_grid_geometry(self.dim, lo.ctypes.data, hi.ctypes.data, self.n,
                                     float(cells_per_point), ctypes.byref(self.grid), None, None),
                  "fm_grid_geometry")
        else:
            self.grid = geom.to_ctypes()
        self.bbox = bbox  # exact (unpadded) source bbox on the host, or None
        self.geom = geom
        ncell = int(self.grid.ncell)
        dev = self.pts.device
        self.cell_start = _empty(ncell + 1, torch.int32, dev)
        self.sorted_ids = _empty(self.n, torch.int32, dev)
        self.sorted_pts = _empty((self.n, self.dim), torch.float64, dev)
        ws_bytes = L.fm_grid_workspace(self.n, ncell)
        ws = _workspace(ws_bytes, dev)
        check(L.fm_grid_build(ctypes.byref(self.grid), ptr(self.pts), self.n,
                              ptr(self.cell_start), ptr(self.sorted_ids), ptr(self.sorted_pts),
                              ptr(ws), ws_bytes, _stream()), "fm_grid_build")
        self._ws = ws  # keep alive until the stream has consumed it

    def target_order(self, targets, nblocks=1):
        """Cell order of `targets` (device int32 perm) for locality.  With
        nblocks > 1 the targets of index block b = [nt*b/nblocks,
        nt*(b+1)/nblocks) occupy exactly those processing positions."""
        L = _lib.lib()
        nt = targets.shape[0]
        perm = _empty(nt, torch.int32, targets.device)
        ws_bytes = L.fm_order_workspace_blocked(nt, ctypes.byref(self.grid), int(nblocks))
        ws = _workspace(ws_bytes, targets.device)
        check(L.fm_target_order_blocked(ctypes.byref(self.grid), ptr(targets), nt, int(nblocks),
                                        ptr(perm), ptr(ws), ws_bytes, _stream()),
              "fm_target_order_blocked")
        self._ws_order = ws
        return perm


def device_bbox(pts):
    return device_bboxes([pts])[0]


_BBOX_WS = {}


def device_bboxes(arrays):
    """Bounding boxes of one or two device point arrays: one launch and ONE
    device->host round trip (fm_bbox_pair)."""
    dim = arrays[0].shape[1]
    if len(arrays) > 2:
        return device_bboxes(arrays[:2]) + device_bboxes(arrays[2:])
    dev = arrays[0].device
    ws = _BBOX_WS.get(dev)
    if ws is None:
        ws = _BBOX_WS[dev] = torch.empty(64 * FM_MAX_DIM, dtype=torch.uint8, device=dev)
    h = np.empty(4 * dim, dtype=np.float64)
    a = arrays[0]
    b = arrays[1] if len(arrays) > 1 else None
    check(_lib.lib().fm_bbox_pair(dim, ptr(a), a.shape[0], ptr(b), 0 if b is None else b.shape[0],
                                  h.ctypes.data, ptr(ws), _stream()), "fm_bbox_pair")
    out = [(h[:dim].copy(), h[dim:2 * dim].copy())]
    if b is not None:
        out.append((h[2 * dim:3 * dim].copy(), h[3 * dim:].copy()))
    return out


# ------------------------------------------------------- selection spec
@dataclass(frozen=True)
class Select:
    """fixed radius r_c, or adaptive (min_pts, r0, growth, r_max)."""

    adaptive: bool
    r_c: float = 0.0
    min_pts: int = 0
    r0: float = 0.0
    growth: float = 0.0
    r_max: float = 0.0

    def to_ctypes(self):
        return FmSelect(1 if self.adaptive else 0, int(self.min_pts), float(self.r_c),
                        float(self.r0), float(self.growth), float(self.r_max))


def fixed(r_c):
    return Select(False, r_c=float(r_c))


def adaptive(min_pts, r0, growth, r_max):
    return Select(True, min_pts=int(min_pts), r0=float(r0), growth=float(growth),
                  r_max=float(r_max))


@dataclass
class Counts:
    counts: torch.Tensor  # int32 (nt,)
    radii: torch.Tensor   # f64 (nt,) final radius (fixed: None)
    status: torch.Tensor  # u8 (nt,) adaptive status (fixed: None)
    stats: np.ndarray     # int32[6] host (see fieldmap.h)
    offsets: torch.Tensor = None  # int64 (nt+1,)
    nnz: int = 0

    @property
    def max_count(self):
        return int(self.stats[0])


def count_supports(cloud, targets, sel, perm=None, min_required=0, with_offsets=True):
    """Count pass (+ exclusive scan).  One device->host sync for the stats."""
    L = _lib.lib()
    dev = targets.device
    nt = targets.shape[0]
    counts = _empty(nt, torch.int32, dev)
    radii = _empty(nt, torch.float64, dev) if sel.adaptive else None
    status = _empty(nt, torch.uint8, dev) if sel.adaptive else None
    stats_d = _empty(6, torch.int32, dev)
    csel = sel.to_ctypes()
    check(L.fm_support_count(ctypes.byref(cloud.grid), ptr(cloud.cell_start),
                             ptr(cloud.sorted_pts), ptr(targets), nt, ptr(perm),
                             ctypes.byref(csel), int(min_required), ptr(counts), ptr(radii),
                             ptr(status), ptr(stats_d), _stream()), "fm_support_count")
    offsets = None
    if with_offsets:
        offsets = _empty(nt + 1, torch.int64, dev)
        ws_bytes = L.fm_scan_workspace(nt)
        ws = _workspace(ws_bytes, dev)
        check(L.fm_offsets_from_counts(ptr(counts), nt, ptr(offsets), ptr(ws), ws_bytes,
                                       _stream()), "fm_offsets_from_counts")
        summary = torch.cat([stats_d.to(torch.int64), offsets[nt:nt + 1]]).cpu().numpy()
        stats = summary[:6].astype(np.int32)
        nnz = int(summary[6])
    else:
        stats = stats_d.cpu().numpy()
        nnz = 0
    if nt == 0:
        stats[0] = 0
    return Counts(counts, radii, status, stats, offsets, nnz)


def fill_supports(cloud, targets, sel, cnt, perm=None, rbf=None):
    """Fill pass: (idx int64, dist f64[, raw weights f64]) CSR at cnt.offsets."""
    L = _lib.lib()
    dev = targets.device
    idx = _empty(cnt.nnz, torch.int64, dev)
    dist = _empty(cnt.nnz, torch.float64, dev)
    w = _empty(cnt.nnz, torch.float64, dev) if rbf is not None else None
    crbf = FmRbf(int(rbf[0]), 0, float(rbf[1])) if rbf is not None else None
    csel = sel.to_ctypes()
    check(L.fm_support_fill(ctypes.byref(cloud.grid), ptr(cloud.cell_start),
                            ptr(cloud.sorted_pts), ptr(cloud.sorted_ids), ptr(targets),
                            targets.shape[0], ptr(perm), ctypes.byref(csel), ptr(cnt.radii),
                            ptr(cnt.offsets), max(cnt.max_count, 1), ptr(idx), ptr(dist),
                            ctypes.byref(crbf) if crbf is not None else None, ptr(w), _stream()),
          "fm_support_fill")
    return idx, dist, w


def rbf_weights(kind, a, r_c, r):
    out = torch.empty_like(r)
    check(_lib.lib().fm_rbf_weights(int(kind), float(a), float(r_c), ptr(r), r.numel(), ptr(out),
                                    _stream()), "fm_rbf_weights")
    return out


def _fit_struct(dim, degree, lam, centering):
    return FmFit(int(dim), int(degree), float(lam), 1 if centering else 0, 0)


def fit_many(targets, sup_off, sup_idx, sup_w, src, src_val, degree, lam, centering, max_m):
    """fit_many on device CSR supports -> (values, coeffs, status, stats)."""
    L = _lib.lib()
    dev = targets.device
    nt, dim = targets.shape
    k = L.fm_n_monomials(dim, degree)
    values = _empty(nt, torch.float64, dev)
    coeffs = _empty((nt, k), torch.float64, dev)
    status = _empty(nt, torch.uint8, dev)
    stats = _empty(2, torch.int32, dev)
    f = _fit_struct(dim, degree, lam, centering)
    check(L.fm_fit_many(ctypes.byref(f), ptr(targets), nt, ptr(sup_off), ptr(sup_idx), ptr(sup_w),
                        int(max_m), ptr(src), ptr(src_val), ptr(values), ptr(coeffs), ptr(status),
                        ptr(stats), _stream()), "fm_fit_many")
    return values, coeffs, status, stats


def slot_capacity(dim, sel):
    """Per-target slot size of the select pass (overflowing supports are
    re-gathered by the build, so this is a speed knob, not a limit)."""
    if dim <= 2:
        return 48  # the thread-per-target select's list (k_select_t): 8 CTAs per SM
    base = 128 if dim == 3 else 256
    if sel.adaptive:
        est = int(np.ceil(sel.min_pts * sel.growth ** dim * 1.25))
        base = max(base, min(256, -(-est // 32) * 32))
    return base


@dataclass
class Selection:
    """Output of the select pass: supports of every target in HBM."""

    sel: Select
    counts: torch.Tensor    # int32 (nt,) by target
    radii: torch.Tensor     # f64 (nt,) final radius (adaptive) or None
    status: torch.Tensor    # u8 (nt,) adaptive status or None
    slot_id: torch.Tensor   # int32 (nt * slot_cap,) by processing position, or None
    slot_pos: torch.Tensor
    slot_cap: int
    overflow: torch.Tensor  # int32 positions whose support did not fit a slot
    stats: np.ndarray       # int32[8] host (fieldmap.h fm_select)
    offsets: torch.Tensor   # int64 (nt+1,) row offsets in processing order
    nnz: int
    perm: torch.Tensor
    pos_info: torch.Tensor = None  # 16 B per position (target, support size, radius)
    pos_t: torch.Tensor = None     # (nt, dim) targets in processing order
    bucket_list: torch.Tensor = None  # int32 (FM_NBUCKETS * nt) positions by support size
    bucket_count: np.ndarray = None   # int32[FM_NBUCKETS] host

    @property
    def max_count(self):
        return int(self.stats[0])

    @property
    def n_overflow(self):
        return int(self.stats[6])

    def lists(self):
        nb = _lib.FM_NBUCKETS
        buckets = self.bucket_list is not None and self.bucket_count is not None
        return FmLists(self.counts.data_ptr(),
                       self.slot_id.data_ptr() if self.slot_id is not None else None,
                       self.slot_pos.data_ptr(),
                       int(self.slot_cap), self.n_overflow, self.overflow.data_ptr(),
                       self.pos_info.data_ptr() if self.pos_info is not None else None,
                       self.pos_t.data_ptr() if self.pos_t is not None else None,
                       self.bucket_list.data_ptr() if buckets else None,
                       self.counts.shape[0] if buckets else 0,
                       (ctypes.c_int32 * nb)(*(self.bucket_count if buckets else [0] * nb)))


def select(cloud, targets, sel, perm=None, min_required=0, slot_cap=None):
    """Select pass + row offsets in processing order.  One device->host
    sync (the stats and nnz)."""
    L = _lib.lib()
    dev = targets.device
    nt = targets.shape[0]
    cap = int(slot_cap or slot_capacity(cloud.dim, sel))
    counts = _empty(nt, torch.int32, dev)
    radii = _empty(nt, torch.float64, dev) if sel.adaptive else None
    status = _empty(nt, torch.uint8, dev) if sel.adaptive else None
    slot_id = None  # the build reads ids as sorted_ids[slot_pos]
    slot_pos = _empty(max(nt * cap, 1), torch.int32, dev)
    overflow = _empty(max(nt, 1), torch.int32, dev)
    pos_info = _empty(max(nt, 1) * 2, torch.float64, dev)  # 16 B records
    pos_t = _empty((max(nt, 1), cloud.dim), torch.float64, dev)
    nb = _lib.FM_NBUCKETS
    stats_d = _empty(8 + nb, torch.int32, dev)  # select stats + bucket sizes
    blist = _empty(max(nt, 1) * nb, torch.int32, dev)
    csel = sel.to_ctypes()
    check(L.fm_select_supports(ctypes.byref(cloud.grid), ptr(cloud.cell_start), ptr(cloud.sorted_pts),
                      ptr(cloud.sorted_ids), ptr(targets), nt, ptr(perm), ctypes.byref(csel),
                      int(min_required), ptr(counts), ptr(radii), ptr(status), ptr(slot_id),
                      ptr(slot_pos), cap, ptr(overflow), ptr(stats_d), ptr(pos_info),
                      ptr(pos_t), _stream()), "fm_select_supports")
    offsets = _empty(nt + 1, torch.int64, dev)
    ws_bytes = L.fm_offsets_ordered_workspace(nt)
    ws = _workspace(ws_bytes, dev)
    check(L.fm_offsets_ordered(ptr(counts), ptr(perm), nt, cap, ptr(offsets), ptr(blist),
                               ptr(stats_d[8:]), ptr(ws), ws_bytes, _stream()),
          "fm_offsets_ordered")
    host = torch.empty(8 + nb + 2, dtype=torch.int32, pin_memory=True)
    host[:8 + nb].copy_(stats_d, non_blocking=True)
    host[8 + nb:].copy_(offsets[nt:nt + 1].view(torch.int32), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    h = host.numpy()
    stats = h[:8].copy()
    nnz = int(h[8 + nb:].view(np.int64)[0])
    if nt == 0:
        stats[0] = 0
    return Selection(sel, counts, radii, status, slot_id, slot_pos, cap, overflow, stats,
                     offsets, nnz, perm, pos_info, pos_t, blist, h[8:8 + nb].copy())


def support_csr(cloud, targets, sl, rbf=None):
    """The reference's support CSR (offsets in target order, ids ascending,
    distances, raw weights) for a Selection: what _select_batch returns."""
    L = _lib.lib()
    nt = targets.shape[0]
    offsets = _empty(nt + 1, torch.int64, targets.device)
    ws_bytes = L.fm_scan_workspace(nt)
    ws = _workspace(ws_bytes, targets.device)
    check(L.fm_offsets_from_counts(ptr(sl.counts), nt, ptr(offsets), ptr(ws), ws_bytes,
                                   _stream()), "fm_offsets_from_counts")
    cnt = Counts(sl.counts, sl.radii, sl.status, sl.stats[:6], offsets, sl.nnz)
    idx, dist, w = fill_supports(cloud, targets, sl.sel, cnt, sl.perm, rbf)
    return offsets, idx, dist, w


def transfer_values(cloud, targets, sl, src_val, rbf, degree, lam, centering):
    """Weights + fit for one scalar field from a Selection (no operator kept)."""
    L = _lib.lib()
    dev = targets.device
    nt = targets.shape[0]
    values = _empty(nt, torch.float64, dev)
    status = _empty(nt, torch.uint8, dev)
    stats = _empty(2, torch.int32, dev)
    csel = sl.sel.to_ctypes()
    crbf = FmRbf(int(rbf[0]), 0, float(rbf[1]))
    f = _fit_struct(cloud.dim, degree, lam, centering)
    lists = sl.lists()
    check(L.fm_transfer_values(ctypes.byref(cloud.grid), ptr(cloud.cell_start),
                               ptr(cloud.sorted_pts), ptr(cloud.sorted_ids), ptr(targets), nt,
                               ptr(sl.perm), ctypes.byref(csel), ptr(sl.radii),
                               ctypes.byref(lists), max(sl.max_count, 1), ctypes.byref(crbf),
                               ctypes.byref(f), ptr(src_val), ptr(values), ptr(status), ptr(stats),
                               _stream()), "fm_transfer_values")
    return values, status, stats


# ----------------------------------------------------------- operator
class Operator:
    """Explicit transfer operator W (nt x ns), resident in HBM.

    Stored row k is target perm[k] (processing = cell order, so the apply
    streams the CSR and gathers neighbouring source rows); each row holds
    the weights with which the reference's fit combines the support values
    (fit_many is linear in src_val), so W @ f == fit_many(..., f).values for
    every field f."""

    def __init__(self, offsets, col, val, status, perm, ns):
        self.offsets = offsets
        self.col = col
        self.val = val
        self.status = status
        self.perm = perm
        self.nt = offsets.shape[0] - 1
        self.ns = ns

    @property
    def nnz(self):
        return int(self.col.shape[0])

    def apply(self, X, out=None):
        """Y = W X for X (ns,) or (ns, C) fp64 on the device."""
        squeeze = X.ndim == 1
        X2 = X.reshape(X.shape[0], -1)
        if X2.shape[0] != self.ns:
            raise ValueError(f"field has {X2.shape[0]} rows, operator expects {self.ns}")
        X2 = X2.contiguous()
        C = X2.shape[1]
        Y = out if out is not None else torch.empty((self.nt, C), dtype=torch.float64,
                                                     device=X2.device)
        check(_lib.lib().fm_apply(self.nt, ptr(self.offsets), ptr(self.col), ptr(self.val),
                                  ptr(self.perm), ptr(X2), C, ptr(Y), _stream()), "fm_apply")
        return Y[:, 0] if squeeze else Y

    def algorithmic_bytes(self, C):
        """nnz*(4+8) + nt*4 + ns*C*8 + nt*C*8."""
        return self.nnz * 12 + self.nt * 4 + self.ns * C * 8 + self.nt * C * 8


def build_operator(cloud, targets, sl, rbf, degree, lam, centering):
    """Weights + fit from a Selection -> Operator (plus the fit stats, device)."""
    L = _lib.lib()
    dev = targets.device
    nt = targets.shape[0]
    col = _empty(max(sl.nnz, 1), torch.int32, dev)[:sl.nnz]
    val = _empty(max(sl.nnz, 1), torch.float64, dev)[:sl.nnz]
    status = _empty(nt, torch.uint8, dev)
    stats = _empty(2, torch.int32, dev)
    csel = sl.sel.to_ctypes()
    crbf = FmRbf(int(rbf[0]), 0, float(rbf[1]))
    f = _fit_struct(cloud.dim, degree, lam, centering)
    lists = sl.lists()
    check(L.fm_build_operator(ctypes.byref(cloud.grid), ptr(cloud.cell_start),
                              ptr(cloud.sorted_pts), ptr(cloud.sorted_ids), ptr(targets), nt,
                              ptr(sl.perm), ctypes.byref(csel), ptr(sl.radii), ctypes.byref(lists),
                              ptr(sl.offsets), max(sl.max_count, 1), ctypes.byref(crbf),
                              ctypes.byref(f), ptr(col), ptr(val), ptr(status), ptr(stats),
                              _stream()), "fm_build_operator")
    return Operator(sl.offsets, col, val, status, sl.perm, cloud.n), stats


def scale_points(pts, scale):
    """Per-axis metric: pts * scale (fm_scale_points, device in/out)."""
    sc = np.ascontiguousarray(scale, dtype=np.float64)
    if sc.shape != (pts.shape[1],):
        raise ValueError(f"metric needs {pts.shape[1]} per-axis scales, got {sc.shape}")
    out = torch.empty_like(pts)
    check(_lib.lib().fm_scale_points(ptr(pts), pts.shape[0], pts.shape[1], sc.ctypes.data,
                                     ptr(out), _stream()), "fm_scale_points")
    return out


def map_chunked(cloud, targets, sel, rbf, degree, lam, centering, X, Y, chunk, keep=False,
                min_required=0, on_chunk=None):
    """The whole path for `targets` in chunks of `chunk` (bounded scratch:
    slots and records exist for one chunk at a time): per chunk, target order,
    select, operator build, apply of X (ns, C) into Y[c0:c1].  Returns the
    chunks' operators when `keep` (repeated applies), and the per-chunk
    (select stats, fit stats) for error reporting."""
    nt = int(targets.shape[0])
    X2 = X.reshape(X.shape[0], -1)
    ops, checks = [], []
    for c0 in range(0, nt, max(1, int(chunk))):
        c1 = min(nt, c0 + int(chunk))
        tb = targets[c0:c1]
        perm = cloud.target_order(tb)
        sl = select(cloud, tb, sel, perm, min_required)
        op, st = build_operator(cloud, tb, sl, rbf, degree, lam, centering)
        op.apply(X2, out=Y[c0:c1])
        checks.append((c0, sl.stats.copy(), st))
        if keep:
            ops.append((c0, c1, op))
        if on_chunk is not None:
            on_chunk(c0, c1, sl, op)
        del sl
    return ops, checks


def fp64_probe(blocks=148 * 8, threads=256, iters=4096):
    """Measured FP64 FMA peak in TFLOP/s (CUDA events, best of 5)."""
    sink = torch.zeros(1, dtype=torch.float64, device=_dev())
    L = _lib.lib()
    check(L.fm_fp64_probe(blocks, threads, 64, ptr(sink), _stream()), "fm_fp64_probe")
    best = None
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        check(L.fm_fp64_probe(blocks, threads, iters, ptr(sink), _stream()), "fm_fp64_probe")
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    flops = 2.0 * 8 * iters * blocks * threads
    return flops / (best * 1e-3) / 1e12


@dataclass
class PatchTopology:
    """Device element adjacency for ElementPatch selection
    (_PatchTopology.__init__, pointwise.py:193-200): each interior edge of
    edge_tris links its two elements in both directions, as a CSR over
    elements.  Neighbour order inside a row does not affect the patch."""

    adj_off: torch.Tensor  # int32 (ne + 1)
    adj: torch.Tensor  # int32
    tris: torch.Tensor  # int32 (ne, 3)
    ne: int

    @classmethod
    def from_mesh_arrays(cls, tris, edge_tris):
        i64 = lambda a: to_device(  # noqa: E731
            a if isinstance(a, torch.Tensor) else np.array(a, dtype=np.int64), torch.int64)
        tris = i64(tris).reshape(-1, 3)
        et = i64(edge_tris).reshape(-1, 2)
        ne = int(tris.shape[0])
        et = et[et[:, 1] >= 0]
        src = torch.cat([et[:, 0], et[:, 1]])
        dst = torch.cat([et[:, 1], et[:, 0]])
        order = torch.argsort(src, stable=True)
        counts = torch.bincount(src, minlength=ne)
        adj_off = torch.zeros(ne + 1, dtype=torch.int64, device=tris.device)
        torch.cumsum(counts, 0, out=adj_off[1:])
        # int32 on the device: half the footprint, so the topology stays in L2
        return cls(adj_off.to(torch.int32), dst[order].to(torch.int32).contiguous(),
                   tris.to(torch.int32).contiguous(), ne)


def patch_supports(topo, seed, layers, centroids, sort_by_seed=None):
    """ElementPatch support CSR on the device (fm_patch_count / fm_patch_fill;
    pointwise.py:212-230): (offsets int64 (nt+1), idx int64, counts int64 (nt),
    -1 where a patch exceeds FM_PATCH_MAX_ELEMS / FM_PATCH_MAX_DOFS).
    Vertex-dof patches process targets in seed order (neighbouring threads
    walk neighbouring elements; measured 0.58 -> 0.50 ms at 1M random seeds
    including the sort); centroid patches are cheap enough that the sort does
    not pay (sort_by_seed=None picks this).  Results do not depend on it."""
    L = _lib.lib()
    seed = to_device(seed if isinstance(seed, torch.Tensor) else np.asarray(seed, np.int64),
                     torch.int64)
    nt = int(seed.shape[0])
    counts = torch.empty(nt, dtype=torch.int64, device=seed.device)
    if sort_by_seed is None:
        sort_by_seed = not centroids
    order = torch.argsort(seed.to(torch.int32)) if (sort_by_seed and nt > 1) else None
    args = (ptr(seed), nt, ptr(order), ptr(topo.adj_off), ptr(topo.adj), ptr(topo.tris), topo.ne,
            int(layers), int(bool(centroids)))
    check(L.fm_patch_count(*args, ptr(counts), _stream()), "fm_patch_count")
    # patches beyond the per-thread bounds: again, with the element / dof lists
    # in global scratch (no size limit the reference does not have)
    big = torch.nonzero(counts == -1).reshape(-1) if nt else counts[:0]
    nbig = int(big.shape[0])
    bargs = None
    if nbig:
        ws_bytes = L.fm_patch_big_workspace(nbig, PATCH_BIG_ELEMS, PATCH_BIG_DOFS)
        ws = _workspace(ws_bytes, seed.device)
        bargs = (ptr(seed), ptr(big), nbig, ptr(topo.adj_off), ptr(topo.adj), ptr(topo.tris),
                 topo.ne, int(layers), int(bool(centroids)), PATCH_BIG_ELEMS, PATCH_BIG_DOFS,
                 ptr(ws), ws_bytes)
        check(L.fm_patch_count_big(*bargs, ptr(counts), _stream()), "fm_patch_count_big")
    offsets = torch.zeros(nt + 1, dtype=torch.int64, device=seed.device)
    torch.cumsum(counts.clamp_min(0), 0, out=offsets[1:])
    nnz = int(offsets[-1]) if nt else 0
    idx = torch.empty(nnz, dtype=torch.int64, device=seed.device)
    check(L.fm_patch_fill(*args, ptr(offsets), ptr(idx), _stream()), "fm_patch_fill")
    if nbig:
        check(L.fm_patch_fill_big(*bargs, ptr(offsets), ptr(idx), _stream()), "fm_patch_fill_big")
    return offsets, idx, counts


class MeshDevice:
    """A triangle mesh's arrays resident in HBM, uploaded once per mesh: what
    fm_locate_batch reads (tri_xy, tris, tri_edges, vert_gid, tri_gid, inv2a,
    epsfac), the element grid, and the patch adjacency (PatchTopology) --
    reused by every batch of transfer_extrinsic and every apply."""

    def __init__(self, mesh):
        f64 = lambda a: to_device(a, torch.float64)  # noqa: E731
        i64 = lambda a: to_device(  # noqa: E731
            a if isinstance(a, torch.Tensor) else np.array(a, dtype=np.int64), torch.int64)
        self.arrays = [f64(mesh.tri_xy), i64(mesh.tris), i64(mesh.tri_edges),
                       i64(mesh.vert_gid), i64(mesh.tri_gid), f64(mesh.inv2a), f64(mesh.epsfac)]
        self._grid = None
        self._topo = None
        self.mesh = mesh

    def grid(self):
        if self._grid is None:
            from .locate import ElementGrid

            self._grid = ElementGrid(self.mesh)
        return self._grid

    def topology(self):
        if self._topo is None:
            self._topo = PatchTopology.from_mesh_arrays(self.mesh.tris, self.mesh.edge_tris)
        return self._topo


_MESHES = {}


def mesh_device(mesh):
    """The MeshDevice of `mesh`, cached on the mesh object (or, when it takes
    no attributes, in a small per-process table that keeps the mesh alive)."""
    md = getattr(mesh, "_fm_device", None)
    if isinstance(md, MeshDevice) and md.mesh is mesh:
        return md
    md = MeshDevice(mesh)
    try:
        mesh._fm_device = md
    except (AttributeError, TypeError):
        if len(_MESHES) >= 8:
            _MESHES.pop(next(iter(_MESHES)))
        _MESHES[id(mesh)] = md
        md = _MESHES[id(mesh)]
    return md


def locate_elements(eg, mesh, pts, tol=1e-10, md=None):
    """fm_locate_batch on device points over an element grid (the caller's
    locate_arrays, locate.py:175-186, DEFAULT_TOL 1e-10 at locate.py:28):
    (found u8, elem int64) device tensors.  The mesh arrays come from its
    MeshDevice (uploaded once)."""
    L = _lib.lib()
    n = int(pts.shape[0])
    dev = pts.device
    md = md or mesh_device(mesh)
    arrs = md.arrays
    i64 = lambda a: to_device(  # noqa: E731
        a if isinstance(a, torch.Tensor) else np.array(a, dtype=np.int64), torch.int64)
    if getattr(eg, "_dev_csr", None) is None:
        eg._dev_csr = (i64(eg.cell_offsets), i64(eg.cell_items))
    cell_off, cell_items = eg._dev_csr
    found = _empty(n, torch.uint8, dev)
    elem = _empty(n, torch.int64, dev)
    dim = _empty(n, torch.int64, dev)
    ent = _empty(n, torch.int64, dev)
    bary = _empty((n, 3), torch.float64, dev)
    check(L.fm_locate_batch(ptr(pts), n, *[ptr(a) for a in arrs], float(eg.lo[0]),
                            float(eg.lo[1]), float(eg.dx), float(eg.dy), int(eg.nx), int(eg.ny),
                            ptr(cell_off), ptr(cell_items), float(tol), ptr(found), ptr(elem),
                            ptr(dim), ptr(ent), ptr(bary), _stream()), "fm_locate_batch")
    return found.bool(), elem


class GraphedTransfer:
    """The whole path -- grid, target order, select, operator build, apply --
    for fixed point counts as ONE CUDA graph, replayed per call.

    Geometry-dependent sizes are the only host knowledge the path needs: each
    run() computes the sources' and targets' bboxes (one launch, one D2H), the
    grid geometry (C) and r_max; the graph captured for that geometry is then
    replayed -- no further host syncs, no per-kernel launch cost (the select's
    statistics, the size-bucket counts and the row offsets stay on the device:
    fm_lists.bucket_count_dev).  A geometry change recaptures.  The points and
    the field are read from the tensors given at construction, so a caller
    with moving geometry copies new coordinates into them and calls run().

    Capacities: operator storage for slot_cap entries per target.  A replay is
    valid when no support overflows its slot and no selection / fit fails;
    check() reads the on-device statistics back (one small D2H) and reports
    it -- the eager path (select + build_operator) handles the other cases."""

    def __init__(self, src_d, tgt_d, X_d, fitspec, slot_cap=None, out=None):
        self.src, self.tgt = src_d, tgt_d
        self.X = X_d.reshape(X_d.shape[0], -1)
        self.spec = fitspec
        self.ns, self.dim = src_d.shape
        self.nt = int(tgt_d.shape[0])
        self.C = self.X.shape[1]
        self.key = None
        self.graph = None
        self._fork = None
        self._keys_h = None
        self.slot_cap = slot_cap
        self.Y = out if out is not None else torch.empty((self.nt, self.C), dtype=torch.float64,
                                                          device=src_d.device)
        if tuple(self.Y.shape) != (self.nt, self.C) or not self.Y.is_contiguous():
            raise ValueError("out must be a contiguous (nt, C) tensor")

    def _select_spec(self, bs, bt):
        s = self.spec.selection
        if hasattr(s, "min_points"):
            lo, hi = np.minimum(bs[0], bt[0]), np.maximum(bs[1], bt[1])
            ext = float(np.hypot(hi[0] - lo[0], hi[1] - lo[1])) if lo.size == 2 else \
                float(np.sqrt(np.sum((hi - lo) ** 2)))
            return adaptive(s.min_points, s.r0, s.growth, 1.0000001 * ext + 1e-300)
        return fixed(s.r_c)

    def _allocate(self, grid):
        dev = self.src.device
        L = _lib.lib()
        nt, ns = self.nt, self.ns
        self.grid = grid
        ncell = int(grid.ncell)
        self.cap = int(self.slot_cap or slot_capacity(self.dim, self.sel))
        e = lambda n, t: _empty(max(int(n), 1), t, dev)  # noqa: E731
        self.cell_start, self.sorted_ids = e(ncell + 1, torch.int32), e(ns, torch.int32)
        self.sorted_pts = _empty((ns, self.dim), torch.float64, dev)
        self.gws_bytes = L.fm_grid_workspace(ns, ncell)
        self.gws = _workspace(self.gws_bytes, dev)
        self.perm = e(nt, torch.int32)
        self.ows_bytes = L.fm_order_workspace(nt, ctypes.byref(grid))
        self.ows = _workspace(self.ows_bytes, dev)
        self.counts = e(nt, torch.int32)
        self.radii = e(nt, torch.float64) if self.sel.adaptive else None
        self.status = e(nt, torch.uint8) if self.sel.adaptive else None
        self.slot_pos = e(nt * self.cap, torch.int32)
        self.overflow = e(nt, torch.int32)
        self.pos_info = e(2 * nt, torch.float64)
        self.pos_t = _empty((max(nt, 1), self.dim), torch.float64, dev)
        nb = _lib.FM_NBUCKETS
        self.stats = e(8 + nb + 2, torch.int32)  # select stats, bucket sizes, fit stats
        self.blist = e(nt * nb, torch.int32)
        self.offsets = e(nt + 1, torch.int64)
        self.pos_counts = e(nt, torch.int32)
        self.sws_bytes = L.fm_scan_workspace(nt)
        self.sws = _workspace(self.sws_bytes, dev)
        # zero-filled once: a row the graph does not build (a support in a
        # size bucket the capture left out, flagged by check()) then holds
        # in-range column ids -- stale or 0 -- and the apply stays in bounds
        self.col = torch.zeros(nt * self.cap, dtype=torch.int32, device=dev)
        self.val = e(nt * self.cap, torch.float64)
        self.fstatus = e(nt, torch.uint8)
        edges = _lib.FM_BUCKET_EDGES
        # every bucket a slotted support can fall in (sizes read on the device)
        self.mask = sum(1 << b for b in range(nb) if b == 0 or edges[b - 1] < self.cap)

    def _launch(self):
        L = _lib.lib()
        st = _stream()
        g, nt, ns = self.grid, self.nt, self.ns
        # the target order needs only the grid geometry: it runs on a forked
        # stream beside the source binning (a graph branch once captured)
        main = torch.cuda.current_stream()
        if self._fork is None:
            self._fork = torch.cuda.Stream()
        self._fork.wait_stream(main)
        with torch.cuda.stream(self._fork):
            check(L.fm_target_order(ctypes.byref(g), ptr(self.tgt), nt, ptr(self.perm),
                                    ptr(self.ows), self.ows_bytes, _stream()), "fm_target_order")
        check(L.fm_grid_build(ctypes.byref(g), ptr(self.src), ns, ptr(self.cell_start),
                              ptr(self.sorted_ids), ptr(self.sorted_pts), ptr(self.gws),
                              self.gws_bytes, st), "fm_grid_build")
        main.wait_stream(self._fork)
        csel = self.sel.to_ctypes()
        need = 0 if self.sel.adaptive else _n_monomials(self.dim, self.spec.degree)
        # the select also writes the row lengths by position (capped: 0 for a
        # support beyond the slot, so the offsets stay within nt * cap) and
        # the size buckets; then one scan for the row offsets
        check(L.fm_select_supports_bucketed(
            ctypes.byref(g), ptr(self.cell_start), ptr(self.sorted_pts), ptr(self.sorted_ids),
            ptr(self.tgt), nt, ptr(self.perm), ctypes.byref(csel), need, ptr(self.counts),
            ptr(self.radii), ptr(self.status), None, ptr(self.slot_pos), self.cap,
            ptr(self.overflow), ptr(self.stats), ptr(self.pos_info), ptr(self.pos_t), 1,
            ptr(self.pos_counts), ptr(self.blist), ptr(self.stats[8:]), st),
            "fm_select_supports_bucketed")
        check(L.fm_offsets_from_counts(ptr(self.pos_counts), nt, ptr(self.offsets), ptr(self.sws),
                                       self.sws_bytes, st), "fm_offsets_from_counts")
        nb = _lib.FM_NBUCKETS
        lists = FmLists(self.counts.data_ptr(), None, self.slot_pos.data_ptr(), self.cap, 0,
                        self.overflow.data_ptr(), self.pos_info.data_ptr(),
                        self.pos_t.data_ptr(), self.blist.data_ptr(), nt,
                        (ctypes.c_int32 * nb)(*([0] * nb)), self.stats[8:].data_ptr(), self.mask,
                        1)
        rbf = self.spec.rbf
        from .pointwise import _rbf_pair

        kind, a = _rbf_pair(rbf)
        crbf = FmRbf(int(kind), 0, float(a))
        cfit = _fit_struct(self.dim, self.spec.degree, self.spec.lam, self.spec.centering)
        check(L.fm_build_operator(ctypes.byref(g), ptr(self.cell_start), ptr(self.sorted_pts),
                                  ptr(self.sorted_ids), ptr(self.tgt), nt, ptr(self.perm),
                                  ctypes.byref(csel), ptr(self.radii), ctypes.byref(lists),
                                  ptr(self.offsets), self.cap, ctypes.byref(crbf),
                                  ctypes.byref(cfit), ptr(self.col), ptr(self.val),
                                  ptr(self.fstatus), ptr(self.stats[8 + nb:]), st),
              "fm_build_operator")
        check(L.fm_apply(nt, ptr(self.offsets), ptr(self.col), ptr(self.val), ptr(self.perm),
                         ptr(self.X), self.C, ptr(self.Y), st), "fm_apply")

    def _bboxes_async(self):
        """Queue the bbox pair and its D2H into pinned memory on a side
        stream (ordered after the caller's prior work, concurrent with the
        replay that follows); returns the event after which the keys are
        readable."""
        if self._keys_h is None:
            self._keys_h = torch.empty(4 * self.dim, dtype=torch.int64, pin_memory=True)
            self._bbox_ws = torch.empty(64 * FM_MAX_DIM, dtype=torch.uint8,
                                        device=self.src.device)
            self._bbox_ev = torch.cuda.Event()
            self._bbox_st = torch.cuda.Stream()
        self._bbox_st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self._bbox_st):
            check(_lib.lib().fm_bbox_pair_async(self.dim, ptr(self.src), self.ns, ptr(self.tgt),
                                                self.nt, self._keys_h.data_ptr(),
                                                ptr(self._bbox_ws), _stream()),
                  "fm_bbox_pair_async")
            self._bbox_ev.record()
        return self._bbox_ev

    def _decode_bboxes(self):
        h = np.empty(4 * self.dim, dtype=np.float64)
        check(_lib.lib().fm_bbox_decode(self.dim, self._keys_h.data_ptr(), h.ctypes.data),
              "fm_bbox_decode")
        d = self.dim
        return (h[:d].copy(), h[d:2 * d].copy()), (h[2 * d:3 * d].copy(), h[3 * d:].copy())

    def run(self):
        """Map the current sources/targets/field; returns Y (nt, C) on the
        device (valid when check() says so).

        Once a graph exists the step is replayed optimistically: the bbox
        reduction, its copy to pinned host memory and the graph are queued
        back to back, and only then does the host wait -- for the bbox copy,
        not the graph -- and check that the grid geometry and selection are
        the captured ones.  If not, the replay (memory-safe with a stale
        geometry: every cell index is clamped to the grid) is discarded and
        the step re-captured and replayed.  So the GPU never idles on the
        host's geometry check in the steady state."""
        if self.graph is not None:
            ev = self._bboxes_async()
            self.graph.replay()
            ev.synchronize()
            bs, bt = self._decode_bboxes()
            if self._key_for(bs, bt)[0] == self.key:
                return self.Y
            torch.cuda.current_stream().synchronize()  # stale replay: discard
        else:
            bs, bt = device_bboxes([self.src, self.tgt])
        key, grid = self._key_for(bs, bt)
        if key != self.key:
            self._allocate(grid)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # eager pass: lazy attributes/streams outside capture
                self._launch()
            torch.cuda.current_stream().wait_stream(side)
            # the graph launches only the size buckets this geometry fills (an
            # empty bucket's persistent launch still costs its slot in the
            # step); check() flags a later replay that fills another one
            counts = self.stats[8:8 + _lib.FM_NBUCKETS].cpu().numpy()
            used = sum(1 << b for b in range(_lib.FM_NBUCKETS) if counts[b] > 0)
            self.mask = (self.mask & used) or self.mask
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._launch()
            self.key = key
        self.graph.replay()
        return self.Y

    def _key_for(self, bs, bt):
        """(capture key, grid) of the step for these bboxes; sets self.sel."""
        grid = FmGrid()
        lo = np.ascontiguousarray(bs[0])
        hi = np.ascontiguousarray(bs[1])
        check(_lib.lib().fm_grid_geometry(self.dim, lo.ctypes.data, hi.ctypes.data, self.ns,
                                          default_cells_per_point(self.dim), ctypes.byref(grid),
                                          None,
                                          None), "fm_grid_geometry")
        self.sel = self._select_spec(bs, bt)
        return (bytes(grid), self.sel), grid

    def check(self):
        """On-device statistics of the last run (one small D2H): dict with
        the select stats (fieldmap.h fm_select_supports), fit failures and
        `valid` (no overflow, no selection or fit failure)."""
        h = self.stats.cpu().numpy()
        nb = _lib.FM_NBUCKETS
        out = {"max_count": int(h[0]), "short": int(h[2]), "status_fail": int(h[4]),
               "overflow": int(h[6]), "fit_fail": int(h[8 + nb]),
               "buckets": h[8:8 + nb].tolist(), "nnz": int(self.offsets[self.nt].item())}
        out["unbuilt_bucket"] = any(c > 0 and not (self.mask >> b) & 1
                                    for b, c in enumerate(out["buckets"]))
        out["valid"] = (out["overflow"] == 0 and out["short"] == 0 and out["status_fail"] == 0
                        and out["fit_fail"] == 0 and not out["unbuilt_bucket"])
        return out


def _n_monomials(dim, degree):
    return int(_lib.lib().fm_n_monomials(int(dim), int(degree)))
