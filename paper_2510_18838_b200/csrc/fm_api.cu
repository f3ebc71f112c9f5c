// fm_api.cu -- extern "C" entry points (include/fieldmap.h), the radial
// weight kernel, the operator apply (SpMM) kernel and the FP64 probe.
#include <algorithm>
#include <cstdlib>

#include "fm_kernels.cuh"
#include "fm_scan.cuh"

namespace fm {

// ---------------------------------------------------------------- rbf
// rbf_weights (_ext.pyx:65-75), elementwise
__global__ void k_rbf(int kind, double a, double r_c, const double *__restrict__ r, int64_t n,
                      double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rbf_one(kind, a, r_c, r[i]);
}

// ------------------------------------------------- per-axis metric
// out[i, a] = pts[i, a] * scale[a]: the per-axis coordinate scaling of an
// anisotropic metric (SURVEY.md §7 decision 6), applied to sources and
// targets before the isotropic search and fit (IEEE products, so a host
// oracle scaling the same way sees bit-identical coordinates)
struct Scale5 {
    double s[kMaxDim];
};
__global__ void k_scale_points(const double *__restrict__ pts, int64_t n, int dim, Scale5 sc,
                               double *__restrict__ out) {
    const int64_t total = n * dim;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __dmul_rn(pts[i], sc.s[i % dim]);
}

// -------------------------------------------------------------- apply
// Y[row_target[k], :] = sum_j val[j] * X[col[j], :] over stored row k.
// Rows are stored in processing (cell) order, so a warp's tile of 32/L
// consecutive rows is one contiguous nnz range: the warp stages its
// (col, val) stream through shared memory with coalesced loads, then each
// row group of L lanes (V consecutive components per lane, C = L*V) gathers
// the X rows -- one 16-byte load per lane per nonzero, 8 in flight.
// CH = staged nonzeros per warp and pass (measured: 256 beats 128 / 64 / 32,
// 0.150 vs 0.178 / 0.234 / 0.377 ms on C2 -- the per-pass overhead outweighs
// the L1 left to cache X); CS = evict-first (col, val) loads (no gain).
// A variant double-buffering the next tile's (col, val) with cp.async was
// slower (0.166 ms): the kernel is bound by L1 wavefronts, not by latency;
// so was (col, val) staged as 16-byte records read with one shared load per
// nonzero (0.186 ms: 32 KB of staging per block, weights held in registers).
// 4 blocks of 256 per SM = 64 registers (without the minimum, ptxas may
// settle on 48 and spill)
#ifndef FM_APPLY_MINB
#define FM_APPLY_MINB 4
#endif
#define FM_APPLY_BOUNDS __launch_bounds__(256, FM_APPLY_MINB)
template <int L, int V, int CH, bool CS>
__global__ void FM_APPLY_BOUNDS k_apply(int64_t nrows, const int64_t *__restrict__ row_off,
                                               const int32_t *__restrict__ col,
                                               const double *__restrict__ val,
                                               const int32_t *__restrict__ row_target,
                                               const double *__restrict__ X,
                                               double *__restrict__ Y) {
    constexpr int C = L * V;
    constexpr int RPW = 32 / L;
#ifndef FM_APPLY_U
#define FM_APPLY_U 8
#endif
    constexpr int U = FM_APPLY_U;
    __shared__ int32_t s_col[8][CH];
    __shared__ double s_val[8][CH];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int rr = lane / L, li = lane % L;
    int32_t *sc = s_col[wib];
    double *sv = s_val[wib];
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t tile = warp; tile * RPW < nrows; tile += nwarps) {
        const int64_t r0 = tile * RPW;
        const int64_t rend = r0 + RPW < nrows ? r0 + RPW : nrows;
        const int64_t r = r0 + rr;
        const bool active = r < nrows;
        const int64_t rb = active ? __ldg(row_off + r) : 0;
        const int64_t re = active ? __ldg(row_off + r + 1) : 0;
        const int64_t tb = __ldg(row_off + r0), te = __ldg(row_off + rend);
        // the output row's target, loaded now: its latency hides behind the
        // gathers instead of stalling the store
        const int64_t t_out = (active && row_target) ? (int64_t)__ldg(row_target + r) : r;
        double acc[V];
#pragma unroll
        for (int v = 0; v < V; v++) acc[v] = 0.0;
        for (int64_t cs = tb; cs < te; cs += CH) {
            const int n = (int)(te - cs < CH ? te - cs : CH);
            for (int i = lane; i < n; i += 32) {
                sc[i] = CS ? __ldcs(col + cs + i) : __ldg(col + cs + i);
                sv[i] = CS ? __ldcs(val + cs + i) : __ldg(val + cs + i);
            }
            __syncwarp();
            const int j0 = (int)((rb > cs ? rb : cs) - cs);
            const int j1 = (int)((re < cs + n ? re : cs + n) - cs);
            int j = j0;
            for (; j + U <= j1; j += U) {
                double x[U][V];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const double *xp = X + (int64_t)sc[j + u] * C + li * V;
                    if (V == 2) {
                        const double2 x2 = __ldg(reinterpret_cast<const double2 *>(xp));
                        x[u][0] = x2.x;
                        x[u][V - 1] = x2.y;
                    } else {
#pragma unroll
                        for (int v = 0; v < V; v++) x[u][v] = __ldg(xp + v);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int v = 0; v < V; v++) acc[v] = fma(sv[j + u], x[u][v], acc[v]);
            }
            for (; j < j1; j++) {
                const double *xp = X + (int64_t)sc[j] * C + li * V;
#pragma unroll
                for (int v = 0; v < V; v++) acc[v] = fma(sv[j], __ldg(xp + v), acc[v]);
            }
            __syncwarp();
        }
        if (active) {
            double *yp = Y + t_out * C + li * V;
            if (V == 2) {
                *reinterpret_cast<double2 *>(yp) = make_double2(acc[0], acc[V - 1]);
            } else {
#pragma unroll
                for (int v = 0; v < V; v++) yp[v] = acc[v];
            }
        }
    }
}

// any C: one thread per (stored row, component)
__global__ void k_apply_generic(int64_t nrows, const int64_t *__restrict__ row_off,
                                const int32_t *__restrict__ col, const double *__restrict__ val,
                                const int32_t *__restrict__ row_target,
                                const double *__restrict__ X, int C, double *__restrict__ Y) {
    const int64_t total = nrows * C;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / C;
        const int c = (int)(g % C);
        double acc = 0.0;
        for (int64_t j = row_off[r]; j < row_off[r + 1]; j++)
            acc = fma(__ldg(val + j), __ldg(X + (int64_t)__ldg(col + j) * C + c), acc);
        const int64_t t = row_target ? (int64_t)row_target[r] : r;
        Y[t * C + c] = acc;
    }
}

template <int L, int V, int CH = 256, bool CS = false>
static int launch_apply(int64_t nrows, const int64_t *row_off, const int32_t *col,
                        const double *val, const int32_t *row_target, const double *X, double *Y,
                        cudaStream_t st) {
    const int threads = 256;
    constexpr int RPW = 32 / L;
    const int64_t tiles = (nrows + RPW - 1) / RPW;
    const int64_t need = (tiles + 7) / 8;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)kSMs * 8));
    k_apply<L, V, CH, CS><<<blocks, threads, 0, st>>>(nrows, row_off, col, val, row_target, X, Y);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

// ---------------------------------------------------------- FP64 probe
__global__ void k_fp64_probe(int iters, double *sink) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    const double b = 0.999999999, c = 1e-12;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    if (s == 12345.0) sink[0] = s;  // never true; keeps the chains live
}

static SearchArgs make_search(const fm_grid *grid, const int32_t *cell_start,
                              const double *sorted_pts, const int32_t *sorted_ids,
                              const double *targets, int64_t nt, const int32_t *perm,
                              const fm_select *sel, const double *radii) {
    SearchArgs s;
    s.g = to_dev(grid);
    s.cell_start = cell_start;
    s.sorted_pts = sorted_pts;
    s.sorted_ids = sorted_ids;
    s.targets = targets;
    s.nt = nt;
    s.perm = perm;
    s.sel = *sel;
    s.radii = radii;
    return s;
}

static bool grid_ok(const fm_grid *g) {
    if (!g || g->dim < 1 || g->dim > kMaxDim || g->ncell < 1) return false;
    int64_t prod = 1;
    for (int a = 0; a < g->dim; a++) {
        if (g->n[a] < 1 || !(g->inv_d[a] > 0.0)) return false;
        prod *= g->n[a];
    }
    return prod == g->ncell;
}

static bool fit_ok(const fm_fit *f) {
    if (!f || f->dim < 1 || f->dim > kMaxDim || f->degree < 0 || f->degree > 3) return false;
    if (!(f->lam >= 0.0)) return false;
    return fm_n_monomials(f->dim, f->degree) <= 21;
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_version(void) { return 10000; }

const char *fm_error_string(int code) {
    switch (code) {
    case FM_OK: return "ok";
    case FM_ERR_ARG: return "invalid argument";
    case FM_ERR_CUDA: return "CUDA launch or runtime error";
    case FM_ERR_UNSUPPORTED: return "unsupported dimension/degree/size";
    case FM_ERR_WORKSPACE: return "workspace too small";
    }
    return "unknown error";
}

int fm_n_monomials(int dim, int degree) {
    if (dim < 1 || degree < 0) return 0;
    return binom(dim + degree, degree);
}

int fm_support_count(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                     const double *targets, int64_t nt, const int32_t *perm, const fm_select *sel,
                     int32_t min_required, int32_t *counts, double *radii, uint8_t *status,
                     int32_t *stats, fm_stream_t stream) {
    if (!grid_ok(grid) || !sel || nt < 0) return FM_ERR_ARG;
    if (sel->adaptive ? !(sel->r0 > 0.0 && sel->growth > 1.0 && sel->min_pts >= 1)
                      : !(sel->r_c > 0.0))
        return FM_ERR_ARG;
    const SearchArgs s = make_search(grid, cell_start, sorted_pts, nullptr, targets, nt, perm, sel,
                                     nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    switch (grid->dim) {
    case 1: return dim1_count(s, min_required, counts, radii, status, stats, st);
    case 2: return dim2_count(s, min_required, counts, radii, status, stats, st);
    case 3: return dim3_count(s, min_required, counts, radii, status, stats, st);
    case 4: return dim4_count(s, min_required, counts, radii, status, stats, st);
    default: return dim5_count(s, min_required, counts, radii, status, stats, st);
    }
}

int fm_support_fill(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                    const int32_t *sorted_ids, const double *targets, int64_t nt,
                    const int32_t *perm, const fm_select *sel, const double *radii,
                    const int64_t *offsets, int32_t max_count, int64_t *idx, double *dist,
                    const fm_rbf *rbf, double *w, fm_stream_t stream) {
    if (!grid_ok(grid) || !sel || nt < 0 || max_count < 0) return FM_ERR_ARG;
    if (sel->adaptive && !radii) return FM_ERR_ARG;
    if (w && (!rbf || rbf->kind < 0 || rbf->kind > 7)) return FM_ERR_ARG;
    const SearchArgs s = make_search(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm,
                                     sel, sel->adaptive ? radii : nullptr);
    const int kind = rbf ? rbf->kind : 0;
    const double a = rbf ? rbf->a : 0.0;
    cudaStream_t st = (cudaStream_t)stream;
    switch (grid->dim) {
    case 1: return dim1_fill(s, offsets, max_count, idx, dist, kind, a, w, st);
    case 2: return dim2_fill(s, offsets, max_count, idx, dist, kind, a, w, st);
    case 3: return dim3_fill(s, offsets, max_count, idx, dist, kind, a, w, st);
    case 4: return dim4_fill(s, offsets, max_count, idx, dist, kind, a, w, st);
    default: return dim5_fill(s, offsets, max_count, idx, dist, kind, a, w, st);
    }
}

int fm_scale_points(const double *pts, int64_t n, int32_t dim, const double *scale_host,
                    double *out, fm_stream_t stream) {
    if (n < 0 || dim < 1 || dim > kMaxDim || !scale_host) return FM_ERR_ARG;
    if (n == 0) return FM_OK;
    Scale5 sc{};
    for (int a = 0; a < dim; a++) sc.s[a] = scale_host[a];
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n * dim + threads - 1) / threads, (int64_t)kSMs * 16);
    k_scale_points<<<blocks, threads, 0, (cudaStream_t)stream>>>(pts, n, dim, sc, out);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

int fm_rbf_weights(int kind, double a, double r_c, const double *r, int64_t n, double *out,
                   fm_stream_t stream) {
    if (kind < 0 || kind > 7 || n < 0) return FM_ERR_ARG;
    if (n == 0) return FM_OK;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, (int64_t)kSMs * 16);
    k_rbf<<<blocks, threads, 0, (cudaStream_t)stream>>>(kind, a, r_c, r, n, out);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

int fm_fit_many(const fm_fit *fit, const double *targets, int64_t nt, const int64_t *sup_off,
                const int64_t *sup_idx, const double *sup_w, int32_t max_m, const double *src,
                const double *src_val, double *values, double *coeffs, uint8_t *status,
                int32_t *stats, fm_stream_t stream) {
    if (!fit_ok(fit)) return fit && fit->degree <= 3 && fit->dim >= 1 && fit->dim <= kMaxDim
                                 ? FM_ERR_UNSUPPORTED
                                 : FM_ERR_ARG;
    if (nt < 0 || max_m < 0) return FM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
#define FM_FITMANY_CASE(N, P)                                                                 \
    case N * 10 + P:                                                                          \
        return dim##N##_deg##P##_fit_many(*fit, targets, nt, sup_off, sup_idx, sup_w, max_m, \
                                          src, src_val, values, coeffs, status, stats, st);
    switch (fit->dim * 10 + fit->degree) {
        FM_FITMANY_CASE(1, 0) FM_FITMANY_CASE(1, 1) FM_FITMANY_CASE(1, 2) FM_FITMANY_CASE(1, 3)
        FM_FITMANY_CASE(2, 0) FM_FITMANY_CASE(2, 1) FM_FITMANY_CASE(2, 2) FM_FITMANY_CASE(2, 3)
        FM_FITMANY_CASE(3, 0) FM_FITMANY_CASE(3, 1) FM_FITMANY_CASE(3, 2) FM_FITMANY_CASE(3, 3)
        FM_FITMANY_CASE(4, 0) FM_FITMANY_CASE(4, 1) FM_FITMANY_CASE(4, 2)
        FM_FITMANY_CASE(5, 0) FM_FITMANY_CASE(5, 1) FM_FITMANY_CASE(5, 2)
    }
#undef FM_FITMANY_CASE
    return FM_ERR_UNSUPPORTED;
}

static int dispatch_build(int dim, int degree, bool solve, bool slots, const SearchArgs &s,
                          const BuildArgs &b, int max_m, cudaStream_t st) {
#define FM_BUILD_CASE(N, P) \
    case N * 10 + P: return dim##N##_deg##P##_build(solve, slots, s, b, max_m, st);
    switch (dim * 10 + degree) {
        FM_BUILD_CASE(1, 0) FM_BUILD_CASE(1, 1) FM_BUILD_CASE(1, 2) FM_BUILD_CASE(1, 3)
        FM_BUILD_CASE(2, 0) FM_BUILD_CASE(2, 1) FM_BUILD_CASE(2, 2) FM_BUILD_CASE(2, 3)
        FM_BUILD_CASE(3, 0) FM_BUILD_CASE(3, 1) FM_BUILD_CASE(3, 2) FM_BUILD_CASE(3, 3)
        FM_BUILD_CASE(4, 0) FM_BUILD_CASE(4, 1) FM_BUILD_CASE(4, 2)
        FM_BUILD_CASE(5, 0) FM_BUILD_CASE(5, 1) FM_BUILD_CASE(5, 2)
    }
#undef FM_BUILD_CASE
    return FM_ERR_UNSUPPORTED;
}

// Size-bucket launches of one build run concurrently on side streams
// (fork/join with events on the caller's stream): the buckets' kernels
// overlap each other's tails.  FM_BUILD_CONCURRENT=0 serialises them.
struct BucketStreams {
    cudaStream_t s[FM_NBUCKETS];
    cudaEvent_t fork, join[FM_NBUCKETS];
    bool ok = false;
};

static BucketStreams *bucket_streams() {
    static BucketStreams pool[64];
    static const bool enabled = [] {
        const char *e = getenv("FM_BUILD_CONCURRENT");
        return !(e && e[0] == '0');
    }();
    if (!enabled) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    BucketStreams &b = pool[dev];
    if (!b.ok) {
        bool good = cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; i < FM_NBUCKETS && good; i++)
            good = cudaStreamCreateWithFlags(&b.s[i], cudaStreamNonBlocking) == cudaSuccess &&
                   cudaEventCreateWithFlags(&b.join[i], cudaEventDisableTiming) == cudaSuccess;
        if (!good) return nullptr;
        b.ok = true;
    }
    return &b;
}

static int build_common(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                        const int32_t *sorted_ids, const double *targets, int64_t nt,
                        const int32_t *perm, const fm_select *sel, const double *radii,
                        const fm_lists *lists, const int64_t *offsets, int32_t max_count,
                        const fm_rbf *rbf, const fm_fit *fit, const double *src_val,
                        int32_t *col, double *val, double *values, uint8_t *status,
                        int32_t *stats, bool solve, fm_stream_t stream) {
    if (!grid_ok(grid) || !sel || !rbf || nt < 0 || max_count < 0) return FM_ERR_ARG;
    if (!fit_ok(fit)) return fit && fit->degree <= 3 ? FM_ERR_UNSUPPORTED : FM_ERR_ARG;
    if (fit->dim != grid->dim || rbf->kind < 0 || rbf->kind > 7) return FM_ERR_ARG;
    if (sel->adaptive && !radii) return FM_ERR_ARG;
    if (lists && (!lists->counts || !lists->slot_pos || lists->slot_cap < 1 ||
                  lists->n_overflow < 0 || (lists->n_overflow > 0 && !lists->overflow) ||
                  (lists->bucket_list && !lists->bucket_count_dev &&
                   lists->bucket_stride < nt)))
        return FM_ERR_ARG;
    const SearchArgs s = make_search(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm,
                                     sel, sel->adaptive ? radii : nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    if (stats) k_stats_init<<<1, 32, 0, st>>>(stats, 2, 1);
    BuildArgs b{};
    b.nk = nt;
    b.offsets = offsets;
    b.cap = max_count < 1 ? 1 : max_count;
    b.rbf_kind = rbf->kind;
    b.rbf_a = rbf->a;
    b.fp = *fit;
    b.src_val = src_val;
    b.col = col;
    b.val = val;
    b.values = values;
    b.status = status;
    b.stats = stats;
    int rc;
    if (lists) {
        b.slot_pos = lists->slot_pos;
        b.slot_cap = lists->slot_cap;
        b.counts = lists->counts;
        b.pos_info = reinterpret_cast<const PosInfo *>(lists->pos_info);
        b.pos_t = lists->pos_targets;
        const int mm = max_count < lists->slot_cap ? max_count : lists->slot_cap;
        if (lists->bucket_list) {
            // one launch per non-empty size bucket, each with the fit shape
            // (lanes x rows per lane) of the bucket's largest support.  With
            // bucket_count_dev the sizes are read on the device (no host
            // sync): the buckets of bucket_mask run over at most bucket_stride
            // positions each.
            constexpr int edges[FM_NBUCKETS] = FM_BUCKET_EDGES;
            const bool dev_counts = lists->bucket_count_dev != nullptr;
            int used[FM_NBUCKETS], nused = 0;
            for (int bk = 0; bk < FM_NBUCKETS; bk++)
                if (dev_counts ? (lists->bucket_mask & (1 << bk)) != 0
                               : lists->bucket_count[bk] > 0)
                    used[nused++] = bk;
            BucketStreams *bs = nused > 1 ? bucket_streams() : nullptr;
            if (bs) cudaEventRecord(bs->fork, st);
            for (int u = 0; u < nused; u++) {
                const int bk = used[u];
                BuildArgs bb = b;
                bb.klist = lists->bucket_list + (int64_t)bk * lists->bucket_stride;
                bb.nk = dev_counts ? lists->bucket_stride : lists->bucket_count[bk];
                bb.nk_dev = dev_counts ? lists->bucket_count_dev + bk : nullptr;
                cudaStream_t sb = st;
                if (bs) {
                    sb = bs->s[u];
                    cudaStreamWaitEvent(sb, bs->fork, 0);
                }
                rc = dispatch_build(grid->dim, fit->degree, solve, true, s, bb,
                                    edges[bk] < mm ? edges[bk] : mm, sb);
                if (bs) {
                    cudaEventRecord(bs->join[u], sb);
                    cudaStreamWaitEvent(st, bs->join[u], 0);
                }
                if (rc) return rc;
            }
        } else {
            rc = dispatch_build(grid->dim, fit->degree, solve, true, s, b, mm, st);
            if (rc) return rc;
        }
        if (lists->n_overflow == 0 || lists->skip_overflow) return FM_OK;
        b.klist = lists->overflow;
        b.nk = lists->n_overflow;
    }
    return dispatch_build(grid->dim, fit->degree, solve, false, s, b, b.cap, st);
}

int fm_build_operator(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                      const int32_t *sorted_ids, const double *targets, int64_t nt,
                      const int32_t *perm, const fm_select *sel, const double *radii,
                      const fm_lists *lists, const int64_t *offsets, int32_t max_count,
                      const fm_rbf *rbf, const fm_fit *fit, int32_t *col, double *val,
                      uint8_t *status, int32_t *stats, fm_stream_t stream) {
    if (!offsets || !col || !val || !status) return FM_ERR_ARG;
    return build_common(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm, sel, radii,
                        lists, offsets, max_count, rbf, fit, nullptr, col, val, nullptr, status,
                        stats, false, stream);
}

int fm_transfer_values(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                       const int32_t *sorted_ids, const double *targets, int64_t nt,
                       const int32_t *perm, const fm_select *sel, const double *radii,
                       const fm_lists *lists, int32_t max_count, const fm_rbf *rbf,
                       const fm_fit *fit, const double *src_val, double *values, uint8_t *status,
                       int32_t *stats, fm_stream_t stream) {
    if (!src_val || !values || !status) return FM_ERR_ARG;
    return build_common(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm, sel, radii,
                        lists, nullptr, max_count, rbf, fit, src_val, nullptr, nullptr, values,
                        status, stats, true, stream);
}

static int select_dispatch(const fm_grid *grid, const int32_t *cell_start,
                           const double *sorted_pts, const int32_t *sorted_ids,
                           const double *targets, int64_t nt, const int32_t *perm,
                           const fm_select *sel, int32_t min_required, int32_t *counts,
                           double *radii, uint8_t *status, int32_t *slot_id, int32_t *slot_pos,
                           int32_t slot_cap, int32_t *overflow, int32_t *stats, void *pos_info,
                           double *pos_targets, fm_stream_t stream, const SelectBuckets &bk) {
    if (!grid_ok(grid) || !sel || nt < 0 || slot_cap < 1 || !stats || !overflow || !counts)
        return FM_ERR_ARG;
    if (sel->adaptive ? !(sel->r0 > 0.0 && sel->growth > 1.0 && sel->min_pts >= 1 && radii)
                      : !(sel->r_c > 0.0))
        return FM_ERR_ARG;
    const SearchArgs s = make_search(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm,
                                     sel, nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    PosInfo *pi = reinterpret_cast<PosInfo *>(pos_info);
    switch (grid->dim) {
    case 1: return dim1_select(s, min_required, counts, radii, status, slot_id, slot_pos, slot_cap, overflow, stats, pi, pos_targets, st, bk);
    case 2: return dim2_select(s, min_required, counts, radii, status, slot_id, slot_pos, slot_cap, overflow, stats, pi, pos_targets, st, bk);
    case 3: return dim3_select(s, min_required, counts, radii, status, slot_id, slot_pos, slot_cap, overflow, stats, pi, pos_targets, st, bk);
    case 4: return dim4_select(s, min_required, counts, radii, status, slot_id, slot_pos, slot_cap, overflow, stats, pi, pos_targets, st, bk);
    default: return dim5_select(s, min_required, counts, radii, status, slot_id, slot_pos, slot_cap, overflow, stats, pi, pos_targets, st, bk);
    }
}

int fm_select_supports(const fm_grid *grid, const int32_t *cell_start, const double *sorted_pts,
                       const int32_t *sorted_ids, const double *targets, int64_t nt,
                       const int32_t *perm, const fm_select *sel, int32_t min_required,
                       int32_t *counts, double *radii, uint8_t *status, int32_t *slot_id,
                       int32_t *slot_pos, int32_t slot_cap, int32_t *overflow, int32_t *stats,
                       void *pos_info, double *pos_targets, fm_stream_t stream) {
    return select_dispatch(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm, sel,
                           min_required, counts, radii, status, slot_id, slot_pos, slot_cap,
                           overflow, stats, pos_info, pos_targets, stream,
                           SelectBuckets{nullptr, nullptr, nullptr, 0});
}

int fm_select_supports_bucketed(const fm_grid *grid, const int32_t *cell_start,
                                const double *sorted_pts, const int32_t *sorted_ids,
                                const double *targets, int64_t nt, const int32_t *perm,
                                const fm_select *sel, int32_t min_required, int32_t *counts,
                                double *radii, uint8_t *status, int32_t *slot_id,
                                int32_t *slot_pos, int32_t slot_cap, int32_t *overflow,
                                int32_t *stats, void *pos_info, double *pos_targets,
                                int32_t cap_rows, int32_t *pos_counts, int32_t *bucket_list,
                                int32_t *bucket_count, fm_stream_t stream) {
    if (!pos_counts || !bucket_list || !bucket_count) return FM_ERR_ARG;
    const SelectBuckets bk{pos_counts, bucket_list, bucket_count, cap_rows};
    int rc = select_dispatch(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm, sel,
                             min_required, counts, radii, status, slot_id, slot_pos, slot_cap,
                             overflow, stats, pos_info, pos_targets, stream, bk);
    if (rc != FM_ERR_UNSUPPORTED) return rc;
    // lane-group select (dim >= 3): the plain select, then the same outputs
    // from a separate gather pass
    rc = fm_select_supports(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm, sel,
                            min_required, counts, radii, status, slot_id, slot_pos, slot_cap,
                            overflow, stats, pos_info, pos_targets, stream);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(bucket_count, 0, sizeof(int32_t) * FM_NBUCKETS, st) != cudaSuccess)
        return FM_ERR_CUDA;
    if (nt > 0) {
        const int blocks = (int)std::min<int64_t>((nt + 1023) / 1024, (int64_t)kSMs * 8);
        k_gather_counts<<<blocks, 256, 0, st>>>(counts, perm, nt, pos_counts, slot_cap,
                                                bucket_list, bucket_count, 0, -1,
                                                cap_rows ? slot_cap : 0);
        FM_CHECK_LAUNCH();
    }
    return FM_OK;
}

size_t fm_offsets_ordered_workspace(int64_t n) {
    return align256(sizeof(int32_t) * (size_t)(n > 0 ? n : 1)) + scan_workspace_bytes(n);
}

int fm_offsets_ordered(const int32_t *counts, const int32_t *perm, int64_t n, int32_t slot_cap,
                       int64_t *offsets, int32_t *bucket_list, int32_t *bucket_count,
                       void *workspace, size_t workspace_bytes, fm_stream_t stream) {
    return fm_offsets_ordered_capped(counts, perm, n, slot_cap, 0, offsets, bucket_list,
                                     bucket_count, workspace, workspace_bytes, stream);
}

int fm_offsets_ordered_capped(const int32_t *counts, const int32_t *perm, int64_t n,
                              int32_t slot_cap, int32_t cap_rows, int64_t *offsets,
                              int32_t *bucket_list, int32_t *bucket_count, void *workspace,
                              size_t workspace_bytes, fm_stream_t stream) {
    if (n < 0 || (bucket_list && !bucket_count)) return FM_ERR_ARG;
    if (workspace_bytes < fm_offsets_ordered_workspace(n)) return FM_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t *tmp = reinterpret_cast<int32_t *>(workspace);
    char *scan_ws = reinterpret_cast<char *>(workspace) +
                    align256(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (bucket_list &&
        cudaMemsetAsync(bucket_count, 0, sizeof(int32_t) * FM_NBUCKETS, st) != cudaSuccess)
        return FM_ERR_CUDA;
    if (n > 0) {
        const int blocks = (int)std::min<int64_t>((n + 1023) / 1024, (int64_t)kSMs * 8);
        k_gather_counts<<<blocks, 256, 0, st>>>(counts, perm, n, tmp, slot_cap, bucket_list,
                                                bucket_count, 0, -1, cap_rows ? slot_cap : 0);
        FM_CHECK_LAUNCH();
    }
    return exclusive_scan<int32_t, int64_t>(tmp, n, offsets, scan_ws, scan_workspace_bytes(n), st);
}

int fm_bucket_positions(const int32_t *counts, const int32_t *perm, int64_t p0, int64_t p1,
                        int32_t slot_cap, int32_t *bucket_list, int64_t bucket_stride,
                        int32_t *bucket_count, fm_stream_t stream) {
    if (p0 < 0 || p1 < p0 || !counts || !bucket_list || !bucket_count ||
        bucket_stride < p1 - p0)
        return FM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(bucket_count, 0, sizeof(int32_t) * FM_NBUCKETS, st) != cudaSuccess)
        return FM_ERR_CUDA;
    const int64_t n = p1 - p0;
    if (n > 0) {
        const int blocks = (int)std::min<int64_t>((n + 1023) / 1024, (int64_t)kSMs * 8);
        k_gather_counts<<<blocks, 256, 0, st>>>(counts, perm, n, nullptr, slot_cap, bucket_list,
                                                bucket_count, p0, bucket_stride);
        FM_CHECK_LAUNCH();
    }
    return FM_OK;
}

int fm_apply(int64_t nt, const int64_t *row_off, const int32_t *col, const double *val,
             const int32_t *row_target, const double *X, int32_t ncomp, double *Y,
             fm_stream_t stream) {
    const int32_t *row_order = row_target;
    if (nt < 0 || ncomp < 1) return FM_ERR_ARG;
    if (nt == 0) return FM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const bool a16 = ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
    switch (ncomp) {
    case 1: return launch_apply<1, 1>(nt, row_off, col, val, row_order, X, Y, st);
    case 2: if (a16) return launch_apply<1, 2>(nt, row_off, col, val, row_order, X, Y, st); break;
    case 4: if (a16) return launch_apply<2, 2>(nt, row_off, col, val, row_order, X, Y, st); break;
    case 8: if (a16) return launch_apply<4, 2>(nt, row_off, col, val, row_order, X, Y, st); break;
    case 16: if (a16) return launch_apply<8, 2>(nt, row_off, col, val, row_order, X, Y, st); break;
    default: break;
    }
    const int threads = 256;
    const int blocks =
        (int)std::max<int64_t>(1, std::min<int64_t>((nt * ncomp + threads - 1) / threads, (int64_t)kSMs * 16));
    k_apply_generic<<<blocks, threads, 0, st>>>(nt, row_off, col, val, row_order, X, ncomp, Y);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

int fm_fp64_probe(int blocks, int threads, int iters, double *sink, fm_stream_t stream) {
    if (blocks < 1 || threads < 1 || iters < 1) return FM_ERR_ARG;
    k_fp64_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, sink);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

}  // extern "C"
