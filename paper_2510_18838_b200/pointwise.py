"""Pointwise (MLS/RBF) field transfer -- the reference API on the B200.

Mirror of the reference's public pointwise API
(/root/reference/pkg/src/fieldbridge/pointwise.py): same names, argument
meaning, defaults, return layout and exceptions, so code written against
`fieldbridge` switches by changing the import.  Underneath, selection,
weights and fits run as sm_100a kernels (device.py / libfieldmap.so) and
`PreparedTransfer` holds an explicit transfer operator in HBM so `apply`
is one SpMM instead of one least-squares solve per target.

Extensions (beyond the reference): points of dimension 1..5
(targets reshape to (-1, dim of the sources)), polynomial degree 3, and
fields with several components ((n, C) values -> (nt, C) results).

Differences that are not extensions:
  * `threads` is accepted and ignored (the GPU path has no host chunking;
    results are the reference's threads=1 results).
  * ElementPatch selection runs on the device:
    element grid, fm_locate_batch, fm_patch_count/fill, fm_fit_many; a patch
    beyond FM_PATCH_MAX_ELEMS / FM_PATCH_MAX_DOFS raises FieldmapError.
"""

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _kernels
from . import device as D
from .errors import (
    ExtrinsicEvaluationError,
    FieldError,
    InsufficientSourcesError,
    SingularFitError,
    UnderdeterminedError,
)
from .locate import PointGrid

__all__ = [
    "RbfKind",
    "RadialBasisSpec",
    "FixedRadius",
    "AdaptiveRadius",
    "ElementPatch",
    "FitSpec",
    "n_monomials",
    "eval_rbf",
    "select_support",
    "fit_local",
    "transfer_pointwise",
    "transfer_extrinsic",
    "fit_point_cloud",
    "PreparedTransfer",
]

MONOMIALS = ("1", "x", "y", "x^2", "xy", "y^2", "x^3", "x^2y", "xy^2", "y^3")
MAX_DEGREE = 3


class RbfKind(enum.Enum):
    """pointwise.py:47-55."""

    GAUSSIAN = "gaussian"
    C4 = "c4"
    CONST = "const"
    IDENTITY = "identity"
    MULTIQUADRIC = "multiquadric"
    INVERSE_MULTIQUADRIC = "inverse_multiquadric"
    THIN_PLATE_SPLINE = "thin_plate_spline"
    CUBIC_SPLINE = "cubic_spline"


_KIND_CODE = {
    RbfKind.GAUSSIAN: _kernels.RBF_GAUSSIAN,
    RbfKind.C4: _kernels.RBF_C4,
    RbfKind.CONST: _kernels.RBF_CONST,
    RbfKind.IDENTITY: _kernels.RBF_IDENTITY,
    RbfKind.MULTIQUADRIC: _kernels.RBF_MULTIQUADRIC,
    RbfKind.INVERSE_MULTIQUADRIC: _kernels.RBF_INVERSE_MULTIQUADRIC,
    RbfKind.THIN_PLATE_SPLINE: _kernels.RBF_THIN_PLATE_SPLINE,
    RbfKind.CUBIC_SPLINE: _kernels.RBF_CUBIC_SPLINE,
}


def n_monomials(degree, dim=2):
    """Monomial count of a polynomial basis of given degree (pointwise.py:70-72;
    `dim` generalises the bivariate count)."""
    num, den = 1, 1
    for i in range(1, degree + 1):
        num *= dim + i
        den *= i
    return num // den


@dataclass(frozen=True)
class RadialBasisSpec:
    """pointwise.py:75-91."""

    kind: RbfKind
    a: float = 2.0
    r_c: float | None = None

    def __post_init__(self):
        if self.a <= 0:
            raise ValueError("shape parameter a must be > 0")
        if self.r_c is not None and self.r_c <= 0:
            raise ValueError("cutoff radius r_c must be > 0")


@dataclass(frozen=True)
class FixedRadius:
    """All sources with distance < r_c (pointwise.py:94-102)."""

    r_c: float

    def __post_init__(self):
        if self.r_c <= 0:
            raise ValueError("r_c must be > 0")


@dataclass(frozen=True)
class AdaptiveRadius:
    """Radius grown geometrically from r0 until min_points sources fit
    (pointwise.py:105-119)."""

    min_points: int
    r0: float
    growth: float = 1.5

    def __post_init__(self):
        if self.min_points < 1:
            raise ValueError("min_points must be >= 1")
        if self.r0 <= 0:
            raise ValueError("r0 must be > 0")
        if self.growth <= 1:
            raise ValueError("growth must be > 1")


@dataclass(frozen=True)
class ElementPatch:
    """pointwise.py:122-131."""

    layers: int = 1

    def __post_init__(self):
        if self.layers < 1:
            raise ValueError("layers must be >= 1")


@dataclass(frozen=True)
class FitSpec:
    """Degree, radial weight, selection rule, and regularization of a fit
    (pointwise.py:134-161; degree 3 is an extension)."""

    degree: int
    rbf: RadialBasisSpec
    selection: object
    lam: float = 0.0
    centering: bool = True

    def __post_init__(self):
        if self.degree not in (0, 1, 2, 3):
            raise ValueError(f"fit degree must be 0, 1, 2 or 3, got {self.degree}")
        if self.lam < 0:
            raise ValueError("lambda must be >= 0")
        if not isinstance(self.selection, (FixedRadius, AdaptiveRadius, ElementPatch)):
            raise TypeError(f"unknown selection rule {self.selection!r}")
        if isinstance(self.selection, AdaptiveRadius):
            need = n_monomials(self.degree)
            if self.selection.min_points < need:
                raise ValueError(
                    f"min_points {self.selection.min_points} below monomial "
                    f"count {need} for degree {self.degree}")


def eval_rbf(spec, r):
    """Radial weight at distance r (pointwise.py:164-176)."""
    r_arr = np.atleast_1d(np.asarray(r, dtype=np.float64))
    if (r_arr < 0).any():
        raise ValueError("distance must be >= 0")
    if spec.kind is RbfKind.IDENTITY:
        w = np.ones_like(r_arr)
    else:
        if spec.r_c is None:
            raise ValueError(f"{spec.kind.value} requires a cutoff radius r_c")
        w = _kernels.rbf_weights(_KIND_CODE[spec.kind], spec.a, spec.r_c, r_arr)
    return w if np.ndim(r) else float(w[0])


def _point_label(points, i):
    """pointwise.py:186-187 (all coordinates for dim != 2)."""
    coords = ", ".join(f"{float(c):.6g}" for c in points[i])
    return f"target {i} at ({coords})"


def _rbf_pair(rbf):
    return (_KIND_CODE[rbf.kind], float(rbf.a))


def _r_max(src_xy, targets):
    """pointwise.py:253-255."""
    span = np.vstack([src_xy, targets])
    lo, hi = span.min(axis=0), span.max(axis=0)
    if span.shape[1] == 2:
        ext = float(np.hypot(hi[0] - lo[0], hi[1] - lo[1]))
    else:
        ext = float(np.sqrt(np.sum((hi - lo) ** 2)))
    return 1.0000001 * ext + 1e-300


_COPY_STREAMS = {}


def _copy_stream():
    """Side stream for host->device copies that overlap device work."""
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[dev]


def _r_max_device(cloud, targets, tbbox=None):
    """_r_max on device-resident points (bboxes by fm_bbox, one small D2H;
    the source bbox is the one the grid was built from)."""
    lo_s, hi_s = cloud.bbox if cloud.bbox is not None else D.device_bbox(cloud.pts)
    if tbbox is not None:
        lo_t, hi_t = tbbox
    else:
        lo_t, hi_t = D.device_bbox(targets) if targets.shape[0] else (lo_s, hi_s)
    lo, hi = np.minimum(lo_s, lo_t), np.maximum(hi_s, hi_t)
    if lo.size == 2:
        ext = float(np.hypot(hi[0] - lo[0], hi[1] - lo[1]))
    else:
        ext = float(np.sqrt(np.sum((hi - lo) ** 2)))
    return 1.0000001 * ext + 1e-300


def _check_patch(fitspec, mesh):
    """True when the selection is ElementPatch on mesh-backed sources (the
    patch path); FieldError for ElementPatch on a bare point cloud
    (pointwise.py:272-275)."""
    if isinstance(fitspec.selection, ElementPatch):
        if mesh is None:
            raise FieldError(
                "element-patch selection needs mesh-backed source dofs, not "
                "a bare point cloud")
        return True
    return False


class _PatchSupports:
    """_select_batch's ElementPatch branch (pointwise.py:271-296) on the
    device: the element grid (the caller's reference UniformGrid for this
    mesh, else the same grid built on the device, locate.py:111-141,
    164-168), fm_locate_batch for each target's element, fm_patch_count/fill
    for the patch dofs (pointwise.py:212-230), unit weights.  Errors are the
    reference's, naming the first failing target."""

    def __init__(self, targets, fitspec, mesh, source_location, grid=None, base_index=0):
        if targets.shape[1] != 2:
            raise FieldError("element-patch selection is 2-D (triangle meshes)")
        md = D.mesh_device(mesh)  # mesh arrays, element grid, adjacency: uploaded once
        if grid is not None and hasattr(grid, "cell_items") and not isinstance(grid, PointGrid):
            if getattr(grid, "mesh", None) is not mesh:
                raise ValueError("grid was built for a different mesh")  # locate.py:177-178
            eg = grid
        else:
            eg = md.grid()
        t = D.to_device(targets)
        found, elem = D.locate_elements(eg, mesh, t, md=md)
        found_h = found.cpu().numpy()
        if not found_h.all():
            i = int(np.argmax(~found_h))
            raise InsufficientSourcesError(
                f"{_point_label(targets, i)} (index {base_index + i}) lies "
                "outside the source mesh; element-patch selection needs a "
                "containing element")
        topo = md.topology()
        self.offsets, self.idx, counts = D.patch_supports(
            topo, elem, fitspec.selection.layers, source_location == "centroids")
        counts_h = counts.cpu().numpy()
        need = n_monomials(fitspec.degree)
        bad = (counts_h < 0) | (counts_h < need)
        if bad.any():
            # the first failing target in index order, as the reference's
            # per-target loop raises (pointwise.py:276-296)
            i = int(np.argmax(bad))
            if counts_h[i] == -2:  # seed is not an element (not located)
                raise InsufficientSourcesError(
                    f"{_point_label(targets, i)} (index {base_index + i}) lies outside the "
                    "source mesh; element-patch selection needs a containing element")
            if counts_h[i] < 0:
                from ._lib import FieldmapError

                raise FieldmapError(
                    f"{_point_label(targets, i)} (index {base_index + i}): element patch "
                    "exceeds the kernel's per-target bound (FM_PATCH_MAX_ELEMS / "
                    "FM_PATCH_MAX_DOFS)")
            raise UnderdeterminedError(
                f"{_point_label(targets, i)} (index {base_index + i}) patch "
                f"has {counts_h[i]} dofs; a degree-{fitspec.degree} fit needs "
                f"at least {need}")
        self.targets = targets
        self.t = t
        self.fitspec = fitspec
        self.base_index = base_index
        self.max_m = int(counts_h.max()) if counts_h.size else 0
        self.w = torch.ones(self.idx.shape[0], dtype=torch.float64, device=t.device)

    def host(self):
        return (self.offsets.cpu().numpy(), self.idx.cpu().numpy(), self.w.cpu().numpy())

    def values(self, src_xy, src_vals):
        """_fit_batch (pointwise.py:299-314) per component on the patch CSR.
        The source coordinates stay on the device between calls (same array)."""
        if getattr(self, "_src_key", None) is not src_xy:
            self._src_d = D.to_device(src_xy)
            self._src_key = src_xy
        src = self._src_d
        vals = D.to_device(src_vals)
        cols = vals.reshape(vals.shape[0], -1)
        out = []
        for c in range(cols.shape[1]):
            v, _, status, _ = D.fit_many(self.t, self.offsets, self.idx, self.w, src,
                                         cols[:, c].contiguous(), self.fitspec.degree,
                                         float(self.fitspec.lam), bool(self.fitspec.centering),
                                         self.max_m)
            _raise_status(status.cpu().numpy(), self.targets, self.fitspec, self.base_index)
            out.append(v)
        y = torch.stack(out, dim=1) if vals.ndim > 1 else out[0]
        return y.reshape((self.t.shape[0],) + tuple(vals.shape[1:]))


class _Plan:
    """Device state of one (sources, targets, selection): grid, processing
    order and the count pass (with the reference's selection errors)."""

    def __init__(self, src_xy, targets, fitspec, grid=None, base_index=0):
        # src_xy / targets: host numpy arrays, or CUDA tensors (device-resident
        # path: nothing but error labels ever comes back to the host)
        self.src_xy = src_xy
        self.targets = targets
        self.fitspec = fitspec
        self.base_index = base_index
        self.t = D.to_device(targets)
        nt = self.t.shape[0]
        self._tbbox = None
        if isinstance(grid, PointGrid) and grid.points.shape[1] == src_xy.shape[1]:
            self.cloud = grid.cloud()
        elif isinstance(src_xy, torch.Tensor) and nt:
            # device-resident inputs: both bounding boxes with one sync
            src_d = D.to_device(src_xy)
            bs, self._tbbox = D.device_bboxes([src_d, self.t])
            self.cloud = D.SourceCloud(src_d, bbox=bs)
        else:
            self.cloud = D.SourceCloud(src_xy)
        self.perm = self.cloud.target_order(self.t) if nt else None
        sel = fitspec.selection
        need = n_monomials(fitspec.degree, self.cloud.dim)
        if isinstance(sel, FixedRadius):
            self.sel = D.fixed(sel.r_c)
            self.sl = D.select(self.cloud, self.t, self.sel, self.perm, need)
            if self.sl.stats[2] > 0:
                i = int(self.sl.stats[3])
                c = int(self.sl.counts[i].item())
                raise UnderdeterminedError(
                    f"{self.label(i)} (index {base_index + i}) has "
                    f"{c} support points inside radius {sel.r_c:g}; a "
                    f"degree-{fitspec.degree} fit needs at least {need}")
        else:
            if isinstance(src_xy, np.ndarray) and isinstance(targets, np.ndarray):
                r_max = _r_max(src_xy, targets)
            else:
                r_max = _r_max_device(self.cloud, self.t, self._tbbox)
            self.sel = D.adaptive(sel.min_points, sel.r0, sel.growth, r_max)
            self.sl = D.select(self.cloud, self.t, self.sel, self.perm, 0)
            if self.sl.stats[4] > 0:
                i = int(self.sl.stats[5])
                c = int(self.sl.counts[i].item())
                raise InsufficientSourcesError(
                    f"{self.label(i)} (index {base_index + i}): only "
                    f"{c} sources in the whole domain, "
                    f"min_points is {sel.min_points}")

    def label(self, i):
        if isinstance(self.targets, np.ndarray):
            return _point_label(self.targets, i)
        return _point_label({i: self.t[i].cpu().numpy()}, i)

    def supports(self, raw_weights=True):
        """(offsets, idx, w_raw) numpy, the reference's _select_batch output."""
        rbf = self.fitspec.rbf
        off, idx, _dist, w = D.support_csr(self.cloud, self.t, self.sl,
                                           rbf=_rbf_pair(rbf) if raw_weights else None)
        return off.cpu().numpy(), idx.cpu().numpy(), w.cpu().numpy()

    def raise_fit_error(self, status, base_index=0):
        """pointwise.py:305-313 for the first failing target."""
        st = status.cpu().numpy() if isinstance(status, torch.Tensor) else status
        bad = st != _kernels.FIT_OK
        if not bad.any():
            return
        i = int(np.argmax(bad))
        if st[i] == _kernels.FIT_EMPTY:
            raise SingularFitError(
                f"{self.label(i)} (index {base_index + i}) has no "
                "support points with nonzero weight")
        raise SingularFitError(
            f"{self.label(i)} (index {base_index + i}): "
            f"rank-deficient degree-{self.fitspec.degree} fit with lambda=0")

    def build_operator(self):
        fs = self.fitspec
        op, stats = D.build_operator(self.cloud, self.t, self.sl, _rbf_pair(fs.rbf), fs.degree,
                                     fs.lam, fs.centering)
        return op, stats

    def transfer_scalar(self, vals_d):
        fs = self.fitspec
        return D.transfer_values(self.cloud, self.t, self.sl, vals_d, _rbf_pair(fs.rbf),
                                 fs.degree, fs.lam, fs.centering)


def _apply_metric(points, metric):
    """Per-axis metric (extension, SURVEY.md §7 decision 6): coordinates
    scaled by `metric` (one factor per axis) -- numpy on the host, tensors on
    the device (fm_scale_points); the same IEEE products either way."""
    if metric is None:
        return points
    if isinstance(points, torch.Tensor):
        pts = D.to_device(points)
        return D.scale_points(pts.reshape(pts.shape[0], -1), metric)
    pts = np.ascontiguousarray(points, dtype=np.float64)
    sc = np.asarray(metric, dtype=np.float64)
    if pts.ndim != 2 or sc.shape != (pts.shape[1],):
        raise ValueError(f"metric needs one scale per axis ({pts.shape[-1]}), got {sc.shape}")
    return np.ascontiguousarray(pts * sc)


def _as_points(a, dim=None):
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if dim is not None:
        arr = arr.reshape(-1, dim)
    return arr


def select_support(target, source_points, selection, rbf=None, grid=None, fit_degree=0,
                   mesh=None, source_location="vertices"):
    """Support indices and raw radial weights for one target point
    (pointwise.py:317-336)."""
    src = _as_points(source_points)
    if src.shape[0] == 0:
        raise InsufficientSourcesError("no source points")
    t = np.asarray(tuple(target), dtype=np.float64)[None, :]
    rbf = rbf if rbf is not None else RadialBasisSpec(RbfKind.CONST, r_c=None)
    spec = FitSpec(fit_degree, rbf, selection)
    if _check_patch(spec, mesh):
        off, idx, w = _PatchSupports(t, spec, mesh, source_location, grid).host()
    else:
        off, idx, w = _Plan(src, t, spec, grid).supports()
    return idx[off[0]:off[1]], w[off[0]:off[1]]


def fit_local(target, support_points, support_values, weights, degree, lam=0.0,
              centering=True):
    """Weighted ridge polynomial fit at one target point (pointwise.py:339-357)."""
    pts = _as_points(support_points)
    vals = np.ascontiguousarray(support_values, dtype=np.float64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if pts.shape[0] < 1:
        raise SingularFitError("empty support")
    t = np.asarray(tuple(target), dtype=np.float64)[None, :]
    spec = FitSpec(degree, RadialBasisSpec(RbfKind.CONST, r_c=None), FixedRadius(1.0), lam=lam,
                   centering=centering)
    off = np.array([0, pts.shape[0]], dtype=np.int64)
    idx = np.arange(pts.shape[0], dtype=np.int64)
    values, coeffs, status = _kernels.fit_many(t, off, idx, np.abs(w), pts, vals, spec.degree,
                                               float(spec.lam), bool(spec.centering))
    _raise_status(status, t, spec)
    return coeffs[0]


def _raise_status(status, targets, fitspec, base_index=0):
    bad = status != _kernels.FIT_OK
    if not bad.any():
        return
    i = int(np.argmax(bad))
    if status[i] == _kernels.FIT_EMPTY:
        raise SingularFitError(
            f"{_point_label(targets, i)} (index {base_index + i}) has no "
            "support points with nonzero weight")
    raise SingularFitError(
        f"{_point_label(targets, i)} (index {base_index + i}): "
        f"rank-deficient degree-{fitspec.degree} fit with lambda=0")


class PreparedTransfer:
    """Transfer operator frozen for fixed source/target geometry
    (pointwise.py:399-431).

    The reference caches only the supports and re-solves every target on each
    `apply`; here construction builds the explicit operator W (CSR in HBM,
    one fused kernel) and `apply` is W @ f for any number of components.
    Fit failures are reported by `apply`, like the reference's."""

    def __init__(self, source_points, target_points, fitspec, grid=None, mesh=None,
                 source_location="vertices", metric=None):
        if metric is not None:  # extension: anisotropic (per-axis) metric
            dim = (source_points.shape[1] if getattr(source_points, "ndim", 1) == 2 else 2)
            source_points = _apply_metric(source_points, metric)
            target_points = _apply_metric(
                target_points.reshape(-1, dim) if isinstance(target_points, torch.Tensor)
                else np.asarray(target_points, dtype=np.float64).reshape(-1, dim), metric)
        if isinstance(source_points, torch.Tensor):
            # device-resident inputs: CUDA tensors in, nothing copied to the host
            self.src_xy = D.to_device(source_points)
            self.targets = D.to_device(target_points).reshape(-1, self.src_xy.shape[1])
        else:
            self.src_xy = _as_points(source_points)
            self.targets = _as_points(target_points, self.src_xy.shape[1])
        self.fitspec = fitspec
        self._support = None
        self._patch = None
        if _check_patch(fitspec, mesh):
            # ElementPatch: the patch CSR stays on the device; apply re-solves
            # per component like the reference (pointwise.py:416, 422-431)
            self._patch = _PatchSupports(self.targets, fitspec, mesh, source_location, grid)
            return
        self._plan = _Plan(self.src_xy, self.targets, fitspec, grid)
        self.operator, self._stats = self._plan.build_operator()

    @property
    def support(self):
        """(offsets, idx, raw weights), as the reference's PreparedTransfer.support."""
        if self._support is None:
            self._support = (self._patch.host() if self._patch is not None else
                             self._plan.supports())
        return self._support

    def _check_fit(self):
        if int(self._stats[0].item()) > 0:
            self._plan.raise_fit_error(self.operator.status)

    def apply(self, source_values, threads=1):
        """Transfer values (ns,) or (ns, C).  numpy in -> numpy out; CUDA
        tensor in -> CUDA tensor out (no host round trip); host tensor in
        (pinned: async copies) -> pinned host tensor out."""
        if self._patch is not None:
            if source_values.shape[0] != self.src_xy.shape[0]:
                raise FieldError("source values disagree with prepared points")
            y = self._patch.values(self.src_xy, source_values)
            if isinstance(source_values, torch.Tensor):
                return y if source_values.is_cuda else y.cpu()
            return y.cpu().numpy()
        if isinstance(source_values, torch.Tensor):
            if source_values.shape[0] != self.src_xy.shape[0]:
                raise FieldError("source values disagree with prepared points")
            if source_values.is_cuda:
                self._check_fit()
                return self.operator.apply(source_values.to(torch.float64))
            # host field: its H2D copy runs on a side stream while the operator
            # build may still be executing; the fit check waits for the build
            # only after the apply is queued
            main = torch.cuda.current_stream()
            side = _copy_stream()
            with torch.cuda.stream(side):
                X = D.to_device(source_values)
            main.wait_stream(side)
            X.record_stream(main)
            Y = self.operator.apply(X)
            out = torch.empty(Y.shape, dtype=Y.dtype, pin_memory=True)
            out.copy_(Y, non_blocking=True)
            self._check_fit()
            main.synchronize()
            return out
        vals = np.ascontiguousarray(source_values, dtype=np.float64)
        if vals.shape[0] != self.src_xy.shape[0]:
            raise FieldError("source values disagree with prepared points")
        self._check_fit()
        return self.operator.apply(D.to_device(vals)).cpu().numpy()


def fit_point_cloud(source_points, source_values, target_points, fitspec, grid=None, mesh=None,
                    source_location="vertices", threads=1, metric=None):
    """Fit a value at each target from a scattered source point cloud
    (pointwise.py:434-451).  numpy in -> numpy out.  torch tensors in: CUDA
    tensors -> CUDA tensor out (nothing copied to the host); host tensors
    (pinned: asynchronous copies) -> pinned host tensor out, with the field's
    host->device copy on a side stream overlapping the whole selection and
    operator build.  `metric` (extension): per-axis coordinate scales of an
    anisotropic metric, applied to sources and targets before the search."""
    if metric is not None:
        dim = source_points.shape[1] if getattr(source_points, "ndim", 1) == 2 else 2
        source_points = _apply_metric(source_points, metric)
        target_points = _apply_metric(
            target_points.reshape(-1, dim) if isinstance(target_points, torch.Tensor)
            else np.asarray(target_points, dtype=np.float64).reshape(-1, dim), metric)
    if any(isinstance(a, torch.Tensor) for a in (source_points, source_values, target_points)):
        return _fit_point_cloud_tensors(source_points, source_values, target_points, fitspec,
                                        grid, mesh, source_location)
    src_xy = _as_points(source_points)
    src_vals = np.ascontiguousarray(source_values, dtype=np.float64)
    if src_xy.shape[0] == 0:
        raise InsufficientSourcesError("no source points")
    if src_xy.shape[0] != src_vals.shape[0]:
        raise FieldError("source points and values disagree in length")
    targets = _as_points(target_points, src_xy.shape[1])
    patch = _check_patch(fitspec, mesh)
    if targets.shape[0] == 0:
        return np.empty((0,) + src_vals.shape[1:], dtype=np.float64)
    if patch:
        ps = _PatchSupports(targets, fitspec, mesh, source_location, grid)
        return ps.values(src_xy, src_vals).cpu().numpy()
    plan = _Plan(src_xy, targets, fitspec, grid)
    if src_vals.ndim == 1:
        values, status, stats = plan.transfer_scalar(D.to_device(src_vals))
        if int(stats[0].item()) > 0:
            plan.raise_fit_error(status)
        return values.cpu().numpy()
    op, stats = plan.build_operator()
    if int(stats[0].item()) > 0:
        plan.raise_fit_error(op.status)
    return op.apply(D.to_device(src_vals)).cpu().numpy()


def _fit_point_cloud_tensors(source_points, source_values, target_points, fitspec, grid, mesh,
                             source_location="vertices"):
    as_t = lambda a: a if isinstance(a, torch.Tensor) else torch.from_numpy(  # noqa: E731
        np.ascontiguousarray(a, dtype=np.float64))
    sp, sv, tp = as_t(source_points), as_t(source_values), as_t(target_points)
    host_out = not sv.is_cuda
    if sp.shape[0] == 0:
        raise InsufficientSourcesError("no source points")
    if sp.shape[0] != sv.shape[0]:
        raise FieldError("source points and values disagree in length")
    if _check_patch(fitspec, mesh):
        ps = _PatchSupports(tp.reshape(-1, 2), fitspec, mesh, source_location, grid)
        y = ps.values(sp, sv)
        return y.cpu() if host_out else y
    main = torch.cuda.current_stream()
    # the geometry goes first (the pipeline starts on it); the field's copy
    # follows on a side stream and overlaps the selection and build
    src_d = D.to_device(sp)
    tgt_d = D.to_device(tp).reshape(-1, src_d.shape[1])
    side = _copy_stream()
    side.wait_stream(main)
    with torch.cuda.stream(side):
        X = D.to_device(sv)  # async when pinned
    if tgt_d.shape[0] == 0:
        main.wait_stream(side)
        Y = torch.empty((0,) + tuple(sv.shape[1:]), dtype=torch.float64, device=src_d.device)
    else:
        plan = _Plan(src_d, tgt_d, fitspec, grid)
        if sv.ndim == 1:
            main.wait_stream(side)
            X.record_stream(main)
            Y, status, stats = plan.transfer_scalar(X)
            bad = stats
        else:
            op, bad = plan.build_operator()
            status = op.status
            main.wait_stream(side)
            X.record_stream(main)
            Y = op.apply(X)
    if host_out:
        out = torch.empty(Y.shape, dtype=Y.dtype, pin_memory=True)
        out.copy_(Y, non_blocking=True)
    else:
        out = Y
    if tgt_d.shape[0] and int(bad[0].item()) > 0:
        plan.raise_fit_error(status)
    if host_out:
        main.synchronize()
    return out


def transfer_pointwise(source_field, target_points, fitspec, grid=None, threads=1):
    """Transfer a discrete field to arbitrary target points (pointwise.py:454-464)."""
    return fit_point_cloud(source_field.dof_points(), source_field.values, target_points, fitspec,
                           grid=grid, mesh=getattr(source_field, "mesh", None),
                           source_location=getattr(source_field, "location", "vertices"),
                           threads=threads)


def transfer_extrinsic(evaluate_callback, target_points, fitspec, source_points, batch_size=1024,
                       mesh=None, source_location="vertices"):
    """Transfer through remote evaluation of the source field
    (pointwise.py:467-510): per batch, select on the device, ask the callback
    for the values of the needed sources only, fit on the device."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    src_xy = _as_points(source_points)
    if src_xy.shape[0] == 0:
        raise InsufficientSourcesError("no source points")
    targets = _as_points(target_points, src_xy.shape[1])
    nt = targets.shape[0]
    if _check_patch(fitspec, mesh):
        return _transfer_extrinsic_patch(evaluate_callback, targets, fitspec, src_xy,
                                         batch_size, mesh, source_location)
    cloud = D.SourceCloud(src_xy)
    grid = _GridHandle(cloud)
    out = np.empty(nt, dtype=np.float64)
    values_cache = np.full(src_xy.shape[0], np.nan, dtype=np.float64)
    for bi, b0 in enumerate(range(0, nt, batch_size)):
        b1 = min(b0 + batch_size, nt)
        chunk = targets[b0:b1]
        plan = _Plan(src_xy, chunk, fitspec, grid, base_index=b0)
        off, idx, w = plan.supports()
        needed = np.unique(idx)
        try:
            got = np.asarray(evaluate_callback(src_xy[needed]), dtype=np.float64)
        except Exception as exc:
            raise ExtrinsicEvaluationError(
                f"evaluation callback failed on batch {bi} "
                f"(targets {b0}..{b1 - 1}): {exc}", batch=bi) from exc
        if got.shape != (needed.size,):
            raise ExtrinsicEvaluationError(
                f"callback returned {got.shape} values for {needed.size} "
                f"points on batch {bi}", batch=bi)
        values_cache[needed] = got
        # the same select + fit kernels as the intrinsic path, so a callback
        # returning the field's own values reproduces it bitwise
        # (reference test_pointwise.py:254-271)
        vals, status, stats = plan.transfer_scalar(D.to_device(values_cache))
        if int(stats[0].item()) > 0:
            plan.raise_fit_error(status, b0)
        out[b0:b1] = vals.cpu().numpy()
    return out


def _transfer_extrinsic_patch(evaluate_callback, targets, fitspec, src_xy, batch_size, mesh,
                              source_location):
    """transfer_extrinsic's batch loop (pointwise.py:488-510) with ElementPatch
    selection: per batch, locate + patch supports on the device, one callback
    for the batch's distinct dofs, the fit on the device."""

    nt = targets.shape[0]
    eg = D.mesh_device(mesh).grid()  # built once, reused by every batch
    out = np.empty(nt, dtype=np.float64)
    values_cache = np.full(src_xy.shape[0], np.nan, dtype=np.float64)
    for bi, b0 in enumerate(range(0, nt, batch_size)):
        b1 = min(b0 + batch_size, nt)
        chunk = targets[b0:b1]
        ps = _PatchSupports(chunk, fitspec, mesh, source_location, eg, base_index=b0)
        needed = torch.unique(ps.idx).cpu().numpy()
        try:
            got = np.asarray(evaluate_callback(src_xy[needed]), dtype=np.float64)
        except Exception as exc:
            raise ExtrinsicEvaluationError(
                f"evaluation callback failed on batch {bi} "
                f"(targets {b0}..{b1 - 1}): {exc}", batch=bi) from exc
        if got.shape != (needed.size,):
            raise ExtrinsicEvaluationError(
                f"callback returned {got.shape} values for {needed.size} "
                f"points on batch {bi}", batch=bi)
        values_cache[needed] = got
        out[b0:b1] = ps.values(src_xy, values_cache).cpu().numpy()
    return out


class _GridHandle(PointGrid):
    """A PointGrid view of an already-built SourceCloud (reused per batch)."""

    def __init__(self, cloud):
        self._cloud = cloud
        self.points = cloud.pts  # only .shape is read by _Plan

    def cloud(self):
        return self._cloud
