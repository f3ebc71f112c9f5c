/*
 * fieldmap.h -- C ABI of the B200 field-mapping library (libfieldmap.so).
 *
 * Drop-in boundary for the hot path of the reference package `fieldbridge`
 * (/root/reference/pkg/src/fieldbridge).  The reference's kernel seam is the
 * module `fieldbridge._kernels` (_kernels/__init__.py:9-42), which binds
 * either the Cython extension (_kernels/_ext.pyx) or the numpy fallback
 * (_kernels/_pure.py).  Every entry point below replaces one function of
 * that seam (or the Python code directly around it) and cites it.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (CUDA global memory) unless the
 *     parameter name ends in `_host`.  Struct arguments are host pointers to
 *     plain-old-data descriptors.
 *   - Every call is enqueued on `stream` and returns immediately; outputs are
 *     valid once the stream reaches that point.  No call allocates device
 *     memory: scratch is caller-owned, sized by the matching *_workspace()
 *     query.
 *   - Return value: FM_OK (0) or a negative FM_ERR_* code.  Numerical
 *     failures are never errors: they are reported per target in `status`
 *     arrays exactly like the reference (FIT_OK/SINGULAR/EMPTY, _ext.pyx:27-29;
 *     adaptive status, _ext.pyx:266).
 *   - Reentrant: no global mutable state; calls on different streams may
 *     overlap.
 *   - Layouts: points are row-major (n, dim) fp64; fields are row-major
 *     (n, ncomp) fp64 (component c of point p at p*ncomp + c).
 */
#ifndef FIELDMAP_H
#define FIELDMAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *fm_stream_t; /* == cudaStream_t */

#define FM_OK 0
#define FM_ERR_ARG (-1)         /* invalid argument / shape */
#define FM_ERR_CUDA (-2)        /* a CUDA launch or runtime call failed */
#define FM_ERR_UNSUPPORTED (-3) /* dimension / degree / size not compiled */
#define FM_ERR_WORKSPACE (-4)   /* caller scratch too small */

#define FM_MAX_DIM 5

/* RBF kind codes: identical to _ext.pyx:18-25 / _pure.py:13-20. */
#define FM_RBF_GAUSSIAN 0
#define FM_RBF_C4 1
#define FM_RBF_CONST 2
#define FM_RBF_IDENTITY 3
#define FM_RBF_MULTIQUADRIC 4
#define FM_RBF_INVERSE_MULTIQUADRIC 5
#define FM_RBF_THIN_PLATE_SPLINE 6
#define FM_RBF_CUBIC_SPLINE 7

/* fit status codes: _ext.pyx:27-29. */
#define FM_FIT_OK 0
#define FM_FIT_SINGULAR 1
#define FM_FIT_EMPTY 2

/* Uniform bucket grid over the source cloud (locate.py:65-99, 144-161).
 * A point's cell along axis a is clamp(trunc((v - lo[a]) * inv_d[a]), 0,
 * n[a]-1) (_ext.pyx:78-85); cells are linearised with axis 0 fastest
 * (the reference's `iy * nx + ix`, _ext.pyx:189). */
typedef struct fm_grid {
    int32_t dim;
    int32_t reserved;
    int64_t n[FM_MAX_DIM];
    double lo[FM_MAX_DIM];
    double inv_d[FM_MAX_DIM];
    int64_t ncell;
} fm_grid;

/* Support selection (pointwise.py:94-119): fixed radius (r_c) or adaptive
 * radius (min_pts, r0, growth, r_max with r_max from pointwise.py:253-255). */
typedef struct fm_select {
    int32_t adaptive;
    int32_t min_pts;
    double r_c;
    double r0;
    double growth;
    double r_max;
} fm_select;

/* Radial weight (pointwise.py:75-91): kind code and shape parameter a; the
 * cutoff is the selection radius (fixed: r_c, pointwise.py:250; adaptive:
 * the per-target final radius, pointwise.py:266-269).  The |w| of
 * _fit_batch (pointwise.py:301) is applied where weights feed a fit. */
typedef struct fm_rbf {
    int32_t kind;
    int32_t reserved;
    double a;
} fm_rbf;

/* Local polynomial fit (pointwise.py:134-161; _ext.pyx:291-293).  degree
 * 0..3, dim 1..5 with n_monomials(dim, degree) <= 21. */
typedef struct fm_fit {
    int32_t dim;
    int32_t degree;
    double lam;
    int32_t centering;
    int32_t reserved;
} fm_fit;

/* ------------------------------------------------------------------ info */
int fm_version(void);
const char *fm_error_string(int code);
/* n_monomials (pointwise.py:70-72, generalised to `dim` axes). */
int fm_n_monomials(int dim, int degree);

/* --------------------------------------------------- a1: source binning
 * Replaces PointGrid/_CsrGrid construction (locate.py:144-161, 65-87):
 * counting (radix) sort of the sources by cell key.  Outputs the CSR
 * cell_start[ncell+1] and the sources in cell order (ids ascending inside a
 * cell) as sorted_ids[n] / sorted_pts[n*dim]. */
size_t fm_grid_workspace(int64_t n, int64_t ncell);
int fm_grid_build(const fm_grid *grid, const double *pts, int64_t n, int32_t *cell_start,
                  int32_t *sorted_ids, double *sorted_pts, void *workspace,
                  size_t workspace_bytes, fm_stream_t stream);

/* Bounding box of n points: lohi[0..dim) = min, lohi[dim..2dim) = max
 * (device).  The `bbox` of locate.py:151. */
int fm_bbox(int dim, const double *pts, int64_t n, double *lohi, fm_stream_t stream);

/* Bounding boxes of two point arrays (b may be NULL with nb = 0) in one
 * launch, returned to HOST memory (the call synchronises `stream`):
 * lohi_host = [a.lo(dim), a.hi(dim), b.lo(dim), b.hi(dim)].  workspace:
 * >= 32*dim bytes of device memory.  The bboxes of locate.py:151 and of
 * pointwise.py:253-255 (r_max) with one device->host round trip. */
int fm_bbox_pair(int dim, const double *a, int64_t na, const double *b, int64_t nb,
                 double *lohi_host, void *workspace, fm_stream_t stream);

/* fm_bbox_pair without the host round trip: enqueues the reduction and an
 * asynchronous copy of 4*dim order-preserving keys into keys_host (pinned
 * host memory; valid once the stream has passed this point -- record an
 * event); fm_bbox_decode (host only) turns them into fm_bbox_pair's lohi.
 * Lets a caller queue work behind the bbox before knowing it (the graphed
 * step replays optimistically and checks the geometry afterwards). */
int fm_bbox_pair_async(int dim, const double *a, int64_t na, const double *b, int64_t nb,
                       unsigned long long *keys_host, void *workspace, fm_stream_t stream);
int fm_bbox_decode(int dim, const unsigned long long *keys_host, double *lohi_host);

/* Host-only: the PointGrid geometry for a source bbox -- _pad_bbox
 * (locate.py:50-62) and _grid_shape (locate.py:34-47) for dim 2, cells of
 * equal side for other dims -- as an fm_grid (lo/hi_out: padded box, may be
 * NULL).  No device work. */
int fm_grid_geometry(int dim, const double *bbox_lo, const double *bbox_hi, int64_t n_points,
                     double cells_per_point, fm_grid *out, double *lo_out, double *hi_out);

/* Processing order of targets for locality: the source grid's cells in
 * blocks of 8x8 (2-D), 4x4x4 (3-D) or 2^dim cells, block-major.  Results
 * never depend on it; perm[k] = target processed k-th. */
size_t fm_order_workspace(int64_t nt, const fm_grid *grid);
/* Same with the targets in nblocks index blocks [nt*b/nblocks,
 * nt*(b+1)/nblocks), block-major: the processing positions of block b are
 * exactly that index range (each block in cell-block order). */
size_t fm_order_workspace_blocked(int64_t nt, const fm_grid *grid, int32_t nblocks);
int fm_target_order_blocked(const fm_grid *grid, const double *targets, int64_t nt,
                            int32_t nblocks, int32_t *perm, void *workspace,
                            size_t workspace_bytes, fm_stream_t stream);
int fm_target_order(const fm_grid *grid, const double *targets, int64_t nt, int32_t *perm,
                    void *workspace, size_t workspace_bytes, fm_stream_t stream);

/* --------------------------------------------- a3/a4: radius search
 * Count pass of fixed_radius_supports (_ext.pyx:215-220) and the radius
 * growth loop of adaptive_radius_supports (_ext.pyx:256-272).  counts[t] is
 * the number of sources with fl(sqrt(sum dx^2)) < r (strict).  For adaptive
 * selection radii[t] / status[t] are the reference's `radii` / `status`
 * (status 1: r_max reached with fewer than min_pts sources); radii/status may
 * be NULL for a fixed radius.  perm may be NULL (identity order).
 * stats (device int32[6], may be NULL; written by the call) receives
 *   [0] max count  [1] min count
 *   [2] #targets with count < min_required  [3] first such target (INT32_MAX if none)
 *   [4] #targets with status != 0           [5] first such target
 * which is what pointwise.py:243-249 / 260-265 need to raise
 * UnderdeterminedError / InsufficientSourcesError naming the first target. */
int fm_support_count(const fm_grid *grid, const int32_t *cell_start,
                     const double *sorted_pts, const double *targets, int64_t nt,
                     const int32_t *perm, const fm_select *sel, int32_t min_required,
                     int32_t *counts, double *radii, uint8_t *status, int32_t *stats,
                     fm_stream_t stream);

/* offsets[0] = 0, offsets[i+1] = offsets[i] + counts[i] (np.cumsum of
 * _ext.pyx:220/272). */
size_t fm_scan_workspace(int64_t n);
int fm_offsets_from_counts(const int32_t *counts, int64_t n, int64_t *offsets,
                           void *workspace, size_t workspace_bytes, fm_stream_t stream);

/* Fill pass (_ext.pyx:225-234, 277-287): per target the source ids with
 * d < r in ascending id order, and d, written at offsets[t].  When rbf and
 * w are non-NULL also writes the raw radial weights (rbf_weights at the
 * selection radius; pointwise.py:250, 266-269), fused.  max_count must be
 * >= every counts[t] (as returned by fm_support_count). */
int fm_support_fill(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                    const int32_t *sorted_ids, const double *targets, int64_t nt,
                    const int32_t *perm, const fm_select *sel, const double *radii,
                    const int64_t *offsets, int32_t max_count, int64_t *idx, double *dist,
                    const fm_rbf *rbf, double *w, fm_stream_t stream);

/* Per-axis metric (an extension; the reference is isotropic): out[i, a] =
 * pts[i, a] * scale_host[a], (n, dim) row-major, device in/out.  Scaling
 * sources and targets alike turns the isotropic radius search and fit into
 * the anisotropic metric diag(scale) (e.g. spatial x velocity axes of a 5-D
 * distribution function; SURVEY.md §7 decision 6). */
int fm_scale_points(const double *pts, int64_t n, int32_t dim, const double *scale_host,
                    double *out, fm_stream_t stream);

/* ------------------------------------------------- a5: radial weights
 * rbf_weights(kind, a, r_c, r) (_ext.pyx:65-75). */
int fm_rbf_weights(int kind, double a, double r_c, const double *r, int64_t n, double *out,
                   fm_stream_t stream);

/* ------------------------------------------------------ a7: fit_many
 * fit_many (_ext.pyx:291-426) on caller-supplied supports: values[nt]
 * (NaN on failure), coeffs[nt*k] (NaN rows), status[nt].  sup_w are the
 * weights as passed to the reference's fit_many (already |w|).  src_val is
 * (ns,) -- one component.  max_m >= every support size.
 * stats (device int32[2], may be NULL; written by the call): [0] #targets
 * with status != FIT_OK, [1] first such target (INT32_MAX if none) --
 * pointwise.py:305-313 raises SingularFitError on the first one. */
int fm_fit_many(const fm_fit *fit, const double *targets, int64_t nt, const int64_t *sup_off,
                const int64_t *sup_idx, const double *sup_w, int32_t max_m, const double *src,
                const double *src_val, double *values, double *coeffs, uint8_t *status,
                int32_t *stats, fm_stream_t stream);

/* ----------------------------- a3/a4 + lists: the select pass (new)
 * Count pass that also emits every target's support (the reference's set,
 * in discovery order; fm_support_fill gives the id-sorted CSR of
 * _sort_by_id, _ext.pyx:155-169) into a fixed-stride slot buffer indexed by
 * PROCESSING POSITION k (the k-th entry of perm):
 * slot_pos[k*slot_cap + i] = index into sorted_pts (and, when slot_id is
 * not NULL, slot_id[k*slot_cap + i] = its source id; the build does not
 * need it: it reads ids as sorted_ids[slot_pos]).
 * counts/radii/status are indexed by target and equal fm_support_count's.
 * Adaptive selection evaluates several radii of the reference's growth
 * sequence per window scan (first scan at a density-guessed step) -- the
 * chosen radius is still the first of that exact sequence holding min_pts.
 * Targets whose support exceeds slot_cap are appended (as positions k) to
 * overflow[]; the build re-gathers them.  stats (device int32[8], written
 * by the call): fm_support_count's 6 entries, [6] #overflow, [7] 0.
 * pos_info (16 B per position: int32 target, int32 support size, f64 radius)
 * and pos_targets (dim doubles per position) are optional per-position
 * copies that let the build read everything by position (may be NULL). */
int fm_select_supports(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                       const int32_t *sorted_ids, const double *targets, int64_t nt,
                       const int32_t *perm, const fm_select *sel, int32_t min_required,
                       int32_t *counts, double *radii, uint8_t *status, int32_t *slot_id,
                       int32_t *slot_pos, int32_t slot_cap, int32_t *overflow, int32_t *stats,
                       void *pos_info, double *pos_targets, fm_stream_t stream);

/* fm_select_supports fused with what fm_offsets_ordered(_capped) derives
 * from its counts, for a step with no host round trip between the select
 * and the build: pos_counts[k] = the row length of position k (its support
 * size; 0 for a support beyond slot_cap when cap_rows != 0) -- scan it with
 * fm_offsets_from_counts for the row offsets -- and the size buckets
 * (bucket_list stride nt, bucket_count device int32[FM_NBUCKETS], zeroed by
 * the call) exactly as fm_offsets_ordered writes them (order within a bucket
 * unspecified).  1-D/2-D: written by the select kernel itself; dim >= 3: a
 * separate gather pass after it. */
int fm_select_supports_bucketed(const fm_grid *grid, const int32_t *cell_start,
                                const double *sorted_pts, const int32_t *sorted_ids,
                                const double *targets, int64_t nt, const int32_t *perm,
                                const fm_select *sel, int32_t min_required, int32_t *counts,
                                double *radii, uint8_t *status, int32_t *slot_id,
                                int32_t *slot_pos, int32_t slot_cap, int32_t *overflow,
                                int32_t *stats, void *pos_info, double *pos_targets,
                                int32_t cap_rows, int32_t *pos_counts, int32_t *bucket_list,
                                int32_t *bucket_count, fm_stream_t stream);

/* Row offsets of an operator stored in processing order:
 * offsets[k+1] = offsets[k] + counts[perm[k]] (perm may be NULL).
 * Optionally (bucket_list != NULL) also partitions the positions by support
 * size for the build: position k with counts[perm[k]] <= slot_cap goes to
 * bucket b = the first with size <= FM_BUCKET_EDGES[b], at
 * bucket_list[b * n + i] (order within a bucket unspecified), and
 * bucket_count (device int32[FM_NBUCKETS], written by the call) holds the
 * bucket sizes.  The build then runs one fit shape (lanes x rows per lane)
 * per bucket instead of sizing every fit for the largest support. */
#define FM_NBUCKETS 9
#define FM_BUCKET_EDGES {8, 16, 24, 32, 48, 64, 96, 128, 2147483647}
size_t fm_offsets_ordered_workspace(int64_t n);
int fm_offsets_ordered(const int32_t *counts, const int32_t *perm, int64_t n, int32_t slot_cap,
                       int64_t *offsets, int32_t *bucket_list, int32_t *bucket_count,
                       void *workspace, size_t workspace_bytes, fm_stream_t stream);

/* Bucket lists (as fm_offsets_ordered's) of the processing positions
 * [p0, p1) only: positions (absolute) by support size into
 * bucket_list[b * bucket_stride + i], sizes into the DEVICE array
 * bucket_count[FM_NBUCKETS].  With fm_target_order_blocked the positions of
 * a target block are such a range, so the operator rows of one block can be
 * built (fm_lists.bucket_count_dev) while another block's results move. */
int fm_bucket_positions(const int32_t *counts, const int32_t *perm, int64_t p0, int64_t p1,
                        int32_t slot_cap, int32_t *bucket_list, int64_t bucket_stride,
                        int32_t *bucket_count, fm_stream_t stream);

/* fm_offsets_ordered for a sync-free step when cap_rows != 0: rows of
 * supports larger than slot_cap get length 0, so the offsets never exceed
 * n * slot_cap (storage sized without reading the counts back) and the apply
 * writes 0 for those targets; the caller detects them from the select stats
 * (stats[6]) and redoes the step through the re-gather path. */
int fm_offsets_ordered_capped(const int32_t *counts, const int32_t *perm, int64_t n,
                              int32_t slot_cap, int32_t cap_rows, int64_t *offsets,
                              int32_t *bucket_list, int32_t *bucket_count, void *workspace,
                              size_t workspace_bytes, fm_stream_t stream);

/* Supports produced by fm_select (device pointers; n_overflow is the host
 * copy of stats[6]).  With bucket_list (fm_offsets_ordered's, stride
 * bucket_stride = nt, bucket_count = host copy of its counts) the build
 * launches once per non-empty bucket; without it once over every position. */
typedef struct fm_lists {
    const int32_t *counts;
    const int32_t *slot_id;     /* unused by the build (ids = sorted_ids[slot_pos]); may be NULL */
    const int32_t *slot_pos;
    int32_t slot_cap;
    int32_t n_overflow;
    const int32_t *overflow;
    const void *pos_info;       /* optional, from fm_select_supports */
    const double *pos_targets;  /* optional, from fm_select_supports */
    const int32_t *bucket_list; /* optional, from fm_offsets_ordered / fm_bucket_positions */
    int64_t bucket_stride;
    int32_t bucket_count[FM_NBUCKETS];
    /* optional device-side bucket sizes (fm_bucket_positions): when set, the
     * buckets whose bit is set in bucket_mask are launched with their sizes
     * read on the device (bucket_count is ignored; no host sync needed) */
    const int32_t *bucket_count_dev;
    int32_t bucket_mask;
    int32_t skip_overflow; /* nonzero: do not rebuild the overflow positions in this call */
} fm_lists;

/* --------------------------------- a8/a13: transfer operator (new)
 * Weights + fit producing the explicit transfer operator W (nt x ns) whose
 * rows are stored in PROCESSING ORDER: stored row k (target perm[k]) spans
 * [offsets[k], offsets[k+1]) with source ids ascending, so that W @ f
 * reproduces fit_many's `values` for every field f (the fit is linear in
 * src_val, _ext.pyx:394).  col[nnz] = source id, val[nnz] = weight (NaN row
 * on failure), status[nt] (by target) and stats[2] as fit_many.  With
 * `lists` (from fm_select) the supports are read from the slots and only
 * overflow targets are re-gathered; with lists == NULL every support is
 * re-gathered (max_count >= every support size).  This is what
 * PreparedTransfer (pointwise.py:399-431) caches instead of the raw support. */
int fm_build_operator(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                      const int32_t *sorted_ids, const double *targets, int64_t nt,
                      const int32_t *perm, const fm_select *sel, const double *radii,
                      const fm_lists *lists, const int64_t *offsets, int32_t max_count,
                      const fm_rbf *rbf, const fm_fit *fit, int32_t *col, double *val,
                      uint8_t *status, int32_t *stats, fm_stream_t stream);

/* One-shot transfer of a scalar field (fit_point_cloud, pointwise.py:434-451):
 * weights + fit_many per target straight from the supports (lists, or
 * re-gathered when lists == NULL) without materialising the operator.
 * values[nt] (NaN on failure), status[nt], stats[2] as fit_many. */
int fm_transfer_values(const fm_grid *grid, const int32_t *cell_start,
                       const double *sorted_pts, const int32_t *sorted_ids,
                       const double *targets, int64_t nt, const int32_t *perm,
                       const fm_select *sel, const double *radii, const fm_lists *lists,
                       int32_t max_count, const fm_rbf *rbf, const fm_fit *fit,
                       const double *src_val, double *values, uint8_t *status,
                       int32_t *stats, fm_stream_t stream);

/* Apply the operator to a multi-component field (PreparedTransfer.apply,
 * pointwise.py:418-431, without re-solving): for every stored row k,
 * Y[row_target[k], :] = sum_j val[j] * X[col[j], :] over [row_off[k],
 * row_off[k+1]).  X (ns, ncomp), Y (nrows, ncomp) row-major; row_target
 * (may be NULL: identity) is the perm the operator was built with. */
int fm_apply(int64_t nrows, const int64_t *row_off, const int32_t *col, const double *val,
             const int32_t *row_target, const double *X, int32_t ncomp, double *Y,
             fm_stream_t stream);

/* ------------------------------- f1: element point localization (next)
 * locate_batch (_ext.pyx:88-152; caller locate_arrays, locate.py:175-186):
 * per query point (n, 2), the first element -- in the stored order of its
 * cell of the element grid (the reference UniformGrid's CSR, row-major
 * cells iy*nx + ix) -- whose tol-halo contains it, barycentric coordinates
 * and its classification on the lowest-dimensional mesh entity within
 * tolerance: dim 0 (vertex gid), 1 (edge id), 2 (element gid).  Mesh arrays
 * as the reference's Mesh: tri_xy (ne, 3, 2), tri_verts/tri_edges (ne, 3),
 * vert_gid (nv), tri_gid (ne), inv2a (ne), epsfac (ne, 3).  Outputs (all n):
 * found u8, elem/dim/ent int64 (-1 when not found), bary (n, 3) f64 (NaN when
 * not found).  Bitwise equal to the reference. */
int fm_locate_batch(const double *points, int64_t n, const double *tri_xy,
                    const int64_t *tri_verts, const int64_t *tri_edges, const int64_t *vert_gid,
                    const int64_t *tri_gid, const double *inv2a, const double *epsfac, double gx0,
                    double gy0, double gdx, double gdy, int64_t nx, int64_t ny,
                    const int64_t *cell_off, const int64_t *cell_items, double tol,
                    uint8_t *found, int64_t *elem, int64_t *dim, int64_t *ent, double *bary,
                    fm_stream_t stream);

/* ---------------------------------------------------- measurement
 * FP64 FMA-chain peak probe (the build kernel's roofline denominator; the
 * driver's MEASURED_PEAKS.json has no FP64 figure).  Runs `iters` dependent
 * DFMA chains per thread; flops = 2 * 8 * iters * blocks * threads. */
int fm_fp64_probe(int blocks, int threads, int iters, double *sink, fm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FIELDMAP_H */
