// fm_grid.cu -- a1: source binning on the device.
//
// Replaces the reference's PointGrid construction (locate.py:144-161 over the
// _CsrGrid CSR of locate.py:65-87: numpy clip/trunc cell keys, lexsort by
// (cell, id), add.at + cumsum).  Here: one counting (radix) sort pass on the
// cell key -- histogram, exclusive scan, scatter -- then an in-cell sort by id
// so the layout is deterministic, then the coordinates are gathered into cell
// order so the radius search reads candidates with coalesced loads.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "fm_common.cuh"
#include "fm_scan.cuh"

namespace fm {

template <int DIM>
__device__ __forceinline__ int64_t cell_key(const GridDev &g, const double *p) {
    int64_t c = 0, stride = 1;
#pragma unroll
    for (int a = 0; a < DIM; a++) {
        c += cell_of(p[a], g.lo[a], g.inv_d[a], g.n[a]) * stride;
        stride *= g.n[a];
    }
    return c;
}

// Processing-order key of a target: cells grouped into blocks of
// kOrderBlock^DIM cells (block-major, row-major inside a block), so that a
// run of consecutive targets covers a compact patch of the domain rather
// than a one-cell-high strip -- neighbouring targets share sources (L1 /
// shared-memory reuse in the build and the apply).  Dense in
// [0, order_keys(grid)).
template <int DIM>
struct OrderBlock {
    static constexpr int B = DIM == 1 ? 1 : DIM == 2 ? 8 : DIM == 3 ? 4 : 2;
};

template <int DIM>
__device__ __forceinline__ int64_t order_key(const GridDev &g, const double *p) {
    constexpr int B = OrderBlock<DIM>::B;
    int64_t blk = 0, bstride = 1, loc = 0, lstride = 1;
#pragma unroll
    for (int a = 0; a < DIM; a++) {
        const int64_t c = cell_of(p[a], g.lo[a], g.inv_d[a], g.n[a]);
        blk += (c / B) * bstride;
        bstride *= (g.n[a] + B - 1) / B;
        loc += (c % B) * lstride;
        lstride *= B;
    }
    return blk * lstride + loc;
}

static int64_t order_keys(const fm_grid *grid) {
    int B = grid->dim == 1 ? 1 : grid->dim == 2 ? 8 : grid->dim == 3 ? 4 : 2;
    int64_t nk = 1;
    for (int a = 0; a < grid->dim; a++) nk *= ((grid->n[a] + B - 1) / B) * B;
    return nk;
}

// nblocks > 1: targets in index blocks [n*b/nblocks, n*(b+1)/nblocks) come
// block by block (block-major keys), each block in cell-block order -- the
// positions of target block b are then the contiguous range of processing
// positions [n*b/nblocks, n*(b+1)/nblocks).
template <int DIM>
__global__ void k_order_keys(GridDev g, const double *__restrict__ pts, int64_t n,
                             int32_t *__restrict__ keys, int32_t *__restrict__ rank,
                             int32_t *__restrict__ counts, int nblocks, int64_t nkeys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double p[DIM];
#pragma unroll
        for (int a = 0; a < DIM; a++) p[a] = pts[i * DIM + a];
        int64_t blk = 0;
        if (nblocks > 1) {  // largest b with n*b/nblocks <= i
            blk = (i * nblocks) / n;
            while (blk + 1 < nblocks && n * (blk + 1) / nblocks <= i) blk++;
            while (blk > 0 && n * blk / nblocks > i) blk--;
        }
        const int32_t c = (int32_t)(blk * nkeys + order_key<DIM>(g, p));
        keys[i] = c;
        rank[i] = atomicAdd(&counts[c], 1);
    }
}

template <int DIM>
__global__ void k_cell_keys(GridDev g, const double *__restrict__ pts, int64_t n,
                            int32_t *__restrict__ keys, int32_t *__restrict__ rank,
                            int32_t *__restrict__ counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double p[DIM];
#pragma unroll
        for (int a = 0; a < DIM; a++) p[a] = pts[i * DIM + a];
        const int32_t c = (int32_t)cell_key<DIM>(g, p);
        keys[i] = c;
        rank[i] = atomicAdd(&counts[c], 1);
    }
}

// counting-sort placement: the point's rank in its cell came from the
// counting atomic (arrival order; the cells are sorted by id afterwards)
__global__ void k_scatter(const int32_t *__restrict__ keys, const int32_t *__restrict__ rank,
                          int64_t n, const int32_t *__restrict__ start,
                          int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[__ldg(start + __ldg(keys + i)) + __ldg(rank + i)] = (int32_t)i;
}

// heapsort helper of k_place (crowded cells)
__device__ __forceinline__ void sift_down(int32_t *a, int32_t root, int32_t n) {
    for (;;) {
        int32_t c = 2 * root + 1;
        if (c >= n) return;
        if (c + 1 < n && a[c + 1] > a[c]) c++;
        if (a[root] >= a[c]) return;
        const int32_t t = a[root];
        a[root] = a[c];
        a[c] = t;
        root = c;
    }
}

// One thread per cell-order position q (the scatter left the cell's points
// there in arrival order): the point i = arrival[q] goes to its place in the
// cell, the number of the cell's points with a smaller id, so ids come out
// ascending per cell (the lexsort tie order of locate.py:79) and its
// coordinates go straight to their slot.  Walking positions, not point ids,
// keeps the reads and writes local for any input order (random clouds).
// A cell of more than kPlaceMax points (clustered or coincident sources) is
// sorted by ONE thread -- the one at its first position -- with heapsort, so
// the cost stays n log n instead of k^2 per cell.
constexpr int kPlaceMax = 64;
template <int DIM>
__global__ void k_place(const int32_t *__restrict__ keys, int64_t n,
                        const int32_t *__restrict__ start, const int32_t *__restrict__ arrival,
                        const double *__restrict__ pts, int32_t *__restrict__ ids,
                        double *__restrict__ sorted_pts) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = __ldg(arrival + q);
        const int32_t c = __ldg(keys + i);
        const int32_t b = __ldg(start + c), e = __ldg(start + c + 1);
        if (e - b <= kPlaceMax) {
            int32_t r = 0;
            for (int32_t k = b; k < e; k++) r += __ldg(arrival + k) < i;
            const int64_t p = b + r;
            FM_DCHECK(b <= q && q < e && p < e && i >= 0 && i < n);
            ids[p] = i;
#pragma unroll
            for (int a = 0; a < DIM; a++) sorted_pts[p * DIM + a] = __ldg(pts + (int64_t)i * DIM + a);
        } else if (q == b) {
            int32_t *v = ids + b;
            const int32_t m = e - b;
            for (int32_t k = 0; k < m; k++) v[k] = arrival[b + k];
            for (int32_t r = m / 2 - 1; r >= 0; r--) sift_down(v, r, m);
            for (int32_t k = m - 1; k > 0; k--) {
                const int32_t t = v[0];
                v[0] = v[k];
                v[k] = t;
                sift_down(v, 0, k);
            }
            for (int32_t k = 0; k < m; k++) {
                const int64_t sidx = v[k];
#pragma unroll
                for (int a = 0; a < DIM; a++)
                    sorted_pts[(int64_t)(b + k) * DIM + a] = pts[sidx * DIM + a];
            }
        }
    }
}

// ---- bbox with order-preserving integer atomics
__device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

__global__ void k_bbox_init(unsigned long long *acc, int dim) {
    const int a = threadIdx.x;
    if (a < dim) {
        acc[a] = ~0ull;        // running min key
        acc[dim + a] = 0ull;   // running max key
    }
}

template <int DIM>
__global__ void k_bbox(const double *__restrict__ pts, int64_t n, unsigned long long *acc) {
    double mn[DIM], mx[DIM];
#pragma unroll
    for (int a = 0; a < DIM; a++) {
        mn[a] = INFINITY;
        mx[a] = -INFINITY;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < DIM; a++) {
            const double v = pts[i * DIM + a];
            mn[a] = fmin(mn[a], v);
            mx[a] = fmax(mx[a], v);
        }
    }
    // warp, then block reduction: one atomic pair per axis and block
    __shared__ double s_mn[8][DIM], s_mx[8][DIM];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int a = 0; a < DIM; a++) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fmin(mn[a], __shfl_xor_sync(FM_FULL_MASK, mn[a], o));
            mx[a] = fmax(mx[a], __shfl_xor_sync(FM_FULL_MASK, mx[a], o));
        }
        if (lane == 0) {
            s_mn[wid][a] = mn[a];
            s_mx[wid][a] = mx[a];
        }
    }
    __syncthreads();
    if (threadIdx.x < DIM) {
        const int a = threadIdx.x;
        double lo = s_mn[0][a], hi = s_mx[0][a];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
            lo = fmin(lo, s_mn[w][a]);
            hi = fmax(hi, s_mx[w][a]);
        }
        atomicMin(&acc[a], dkey(lo));
        atomicMax(&acc[DIM + a], dkey(hi));
    }
}

// Boxes of up to two point arrays in one launch (blockIdx.y = array), for
// fm_bbox_pair: keys accumulate with atomicMin only (the max as the
// complement of its key), so one memset of 0xff initialises everything.
template <int DIM>
__global__ void k_bbox_pair(const double *__restrict__ a, int64_t na, const double *__restrict__ b,
                            int64_t nb, unsigned long long *acc) {
    const double *pts = blockIdx.y ? b : a;
    const int64_t n = blockIdx.y ? nb : na;
    unsigned long long *out = acc + blockIdx.y * 2 * DIM;
    double mn[DIM], mx[DIM];
#pragma unroll
    for (int k = 0; k < DIM; k++) {
        mn[k] = INFINITY;
        mx[k] = -INFINITY;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {  // four points' loads in flight
        double v[4][DIM];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int k = 0; k < DIM; k++) v[u][k] = __ldg(pts + (i + u * stride) * DIM + k);
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int k = 0; k < DIM; k++) {
                mn[k] = fmin(mn[k], v[u][k]);
                mx[k] = fmax(mx[k], v[u][k]);
            }
    }
    for (; i < n; i += stride) {
#pragma unroll
        for (int k = 0; k < DIM; k++) {
            const double v = pts[i * DIM + k];
            mn[k] = fmin(mn[k], v);
            mx[k] = fmax(mx[k], v);
        }
    }
    __shared__ double s_mn[8][DIM], s_mx[8][DIM];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < DIM; k++) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[k] = fmin(mn[k], __shfl_xor_sync(FM_FULL_MASK, mn[k], o));
            mx[k] = fmax(mx[k], __shfl_xor_sync(FM_FULL_MASK, mx[k], o));
        }
        if (lane == 0) {
            s_mn[wid][k] = mn[k];
            s_mx[wid][k] = mx[k];
        }
    }
    __syncthreads();
    if (threadIdx.x < DIM && n > 0) {
        const int k = threadIdx.x;
        double lo = s_mn[0][k], hi = s_mx[0][k];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
            lo = fmin(lo, s_mn[w][k]);
            hi = fmax(hi, s_mx[w][k]);
        }
        if (lo <= hi) {
            atomicMin(&out[k], dkey(lo));
            atomicMin(&out[DIM + k], ~dkey(hi));
        }
    }
}

__global__ void k_bbox_final(const unsigned long long *acc, int dim, double *lohi) {
    const int a = threadIdx.x;
    if (a < 2 * dim) lohi[a] = dval(acc[a]);
}

template <int DIM>
static int launch_keys(const GridDev &g, const double *pts, int64_t n, int32_t *keys,
                       int32_t *rank, int32_t *counts, cudaStream_t s, bool order = false,
                       int nblocks = 1, int64_t nkeys = 0) {
    const int threads = 256;
    const int64_t blocks = n > 0 ? std::min<int64_t>((n + threads - 1) / threads, kSMs * 16) : 0;
    if (blocks && order)
        k_order_keys<DIM><<<(unsigned)blocks, threads, 0, s>>>(g, pts, n, keys, rank, counts,
                                                                 nblocks, nkeys);
    else if (blocks)
        k_cell_keys<DIM><<<(unsigned)blocks, threads, 0, s>>>(g, pts, n, keys, rank, counts);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

}  // namespace fm

using namespace fm;

extern "C" {

size_t fm_grid_workspace(int64_t n, int64_t ncell) {
    return align256(sizeof(int32_t) * (size_t)n) * 3     // keys, ranks, arrival order
           + align256(sizeof(int32_t) * (size_t)ncell)  // counts
           + align256(scan_workspace_bytes(ncell));
}

int fm_grid_build(const fm_grid *grid, const double *pts, int64_t n, int32_t *cell_start,
                  int32_t *sorted_ids, double *sorted_pts, void *workspace,
                  size_t workspace_bytes, fm_stream_t stream) {
    if (!grid || grid->dim < 1 || grid->dim > kMaxDim || n < 0 || grid->ncell < 1)
        return FM_ERR_ARG;
    if (n >= (int64_t)INT32_MAX || grid->ncell >= (int64_t)INT32_MAX) return FM_ERR_UNSUPPORTED;
    if (workspace_bytes < fm_grid_workspace(n, grid->ncell)) return FM_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ncell = grid->ncell;
    char *w = (char *)workspace;
    int32_t *keys = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)n);
    int32_t *rank = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)n);
    int32_t *arrival = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)n);
    int32_t *counts = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)ncell);
    void *scan_ws = w;
    const GridDev g = to_dev(grid);
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)ncell, s);
    int rc;
    switch (grid->dim) {
    case 1: rc = launch_keys<1>(g, pts, n, keys, rank, counts, s); break;
    case 2: rc = launch_keys<2>(g, pts, n, keys, rank, counts, s); break;
    case 3: rc = launch_keys<3>(g, pts, n, keys, rank, counts, s); break;
    case 4: rc = launch_keys<4>(g, pts, n, keys, rank, counts, s); break;
    default: rc = launch_keys<5>(g, pts, n, keys, rank, counts, s); break;
    }
    if (rc) return rc;
    rc = exclusive_scan<int32_t, int32_t>(counts, ncell, cell_start, scan_ws,
                                           scan_workspace_bytes(ncell), s);
    if (rc) return rc;
    const int threads = 256;
    if (n > 0) {
        const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, kSMs * 16);
        k_scatter<<<(unsigned)blocks, threads, 0, s>>>(keys, rank, n, cell_start, arrival);
        switch (grid->dim) {
        case 1: k_place<1><<<(unsigned)blocks, threads, 0, s>>>(keys, n, cell_start, arrival, pts, sorted_ids, sorted_pts); break;
        case 2: k_place<2><<<(unsigned)blocks, threads, 0, s>>>(keys, n, cell_start, arrival, pts, sorted_ids, sorted_pts); break;
        case 3: k_place<3><<<(unsigned)blocks, threads, 0, s>>>(keys, n, cell_start, arrival, pts, sorted_ids, sorted_pts); break;
        case 4: k_place<4><<<(unsigned)blocks, threads, 0, s>>>(keys, n, cell_start, arrival, pts, sorted_ids, sorted_pts); break;
        default: k_place<5><<<(unsigned)blocks, threads, 0, s>>>(keys, n, cell_start, arrival, pts, sorted_ids, sorted_pts); break;
        }
    }
    FM_CHECK_LAUNCH();
    return FM_OK;
}

int fm_bbox(int dim, const double *pts, int64_t n, double *lohi, fm_stream_t stream) {
    if (dim < 1 || dim > kMaxDim || n < 0) return FM_ERR_ARG;
    // accumulate order-preserving integer keys in place of the output
    // (same size: 2*dim x 8 B), converted back by k_bbox_final
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(lohi);
    cudaStream_t s = (cudaStream_t)stream;
    k_bbox_init<<<1, 32, 0, s>>>(acc, dim);
    const int threads = 256;
    const int64_t blocks = n > 0 ? std::min<int64_t>((n + threads - 1) / threads, kSMs * 8) : 0;
    if (blocks) {
        switch (dim) {
        case 1: k_bbox<1><<<(unsigned)blocks, threads, 0, s>>>(pts, n, acc); break;
        case 2: k_bbox<2><<<(unsigned)blocks, threads, 0, s>>>(pts, n, acc); break;
        case 3: k_bbox<3><<<(unsigned)blocks, threads, 0, s>>>(pts, n, acc); break;
        case 4: k_bbox<4><<<(unsigned)blocks, threads, 0, s>>>(pts, n, acc); break;
        default: k_bbox<5><<<(unsigned)blocks, threads, 0, s>>>(pts, n, acc); break;
        }
    }
    k_bbox_final<<<1, 32, 0, s>>>(acc, dim, lohi);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

size_t fm_order_workspace_blocked(int64_t nt, const fm_grid *grid, int32_t nblocks) {
    if (!grid || grid->dim < 1 || grid->dim > kMaxDim || nblocks < 1) return 0;
    const int64_t nk = order_keys(grid) * nblocks;
    return fm_grid_workspace(nt, nk) + align256(sizeof(int32_t) * (size_t)(nk + 1));
}

size_t fm_order_workspace(int64_t nt, const fm_grid *grid) {
    return fm_order_workspace_blocked(nt, grid, 1);
}

int fm_target_order_blocked(const fm_grid *grid, const double *targets, int64_t nt,
                            int32_t nblocks, int32_t *perm, void *workspace,
                            size_t workspace_bytes, fm_stream_t stream) {
    if (!grid || grid->dim < 1 || grid->dim > kMaxDim || nt < 0 || grid->ncell < 1 ||
        nblocks < 1)
        return FM_ERR_ARG;
    const int64_t nkeys = order_keys(grid);
    const int64_t ncell = nkeys * nblocks;  // key range of the (block-major) blocked order
    if (nt >= (int64_t)INT32_MAX || ncell >= (int64_t)INT32_MAX) return FM_ERR_UNSUPPORTED;
    if (workspace_bytes < fm_order_workspace_blocked(nt, grid, nblocks)) return FM_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    char *w = (char *)workspace;
    int32_t *keys = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)nt);
    int32_t *rank = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)nt);
    int32_t *counts = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)ncell);
    int32_t *start = (int32_t *)w;
    w += align256(sizeof(int32_t) * (size_t)(ncell + 1));
    void *scan_ws = w;
    const GridDev g = to_dev(grid);
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)ncell, s);
    int rc;
    switch (grid->dim) {
    case 1: rc = launch_keys<1>(g, targets, nt, keys, rank, counts, s, true, nblocks, nkeys); break;
    case 2: rc = launch_keys<2>(g, targets, nt, keys, rank, counts, s, true, nblocks, nkeys); break;
    case 3: rc = launch_keys<3>(g, targets, nt, keys, rank, counts, s, true, nblocks, nkeys); break;
    case 4: rc = launch_keys<4>(g, targets, nt, keys, rank, counts, s, true, nblocks, nkeys); break;
    default: rc = launch_keys<5>(g, targets, nt, keys, rank, counts, s, true, nblocks, nkeys); break;
    }
    if (rc) return rc;
    rc = exclusive_scan<int32_t, int32_t>(counts, ncell, start, scan_ws,
                                           scan_workspace_bytes(ncell), s);
    if (rc) return rc;
    if (nt > 0) {
        const int threads = 256;
        const int64_t blocks = std::min<int64_t>((nt + threads - 1) / threads, kSMs * 16);
        k_scatter<<<(unsigned)blocks, threads, 0, s>>>(keys, rank, nt, start, perm);
    }
    FM_CHECK_LAUNCH();
    return FM_OK;
}

int fm_target_order(const fm_grid *grid, const double *targets, int64_t nt, int32_t *perm,
                    void *workspace, size_t workspace_bytes, fm_stream_t stream) {
    return fm_target_order_blocked(grid, targets, nt, 1, perm, workspace, workspace_bytes, stream);
}

static double host_dval(unsigned long long k) {
    const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    memcpy(&v, &b, sizeof v);
    return v;
}

int fm_bbox_pair_async(int dim, const double *a, int64_t na, const double *b, int64_t nb,
                       unsigned long long *keys_host, void *workspace, fm_stream_t stream) {
    if (dim < 1 || dim > kMaxDim || na < 0 || nb < 0 || !keys_host || !workspace)
        return FM_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(workspace);
    const size_t bytes = sizeof(unsigned long long) * 4 * (size_t)dim;
    if (cudaMemsetAsync(acc, 0xff, bytes, s) != cudaSuccess) return FM_ERR_CUDA;
    const int threads = 256;
    const int64_t nmax = na > nb ? na : nb;
    const unsigned bx =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>((nmax + threads - 1) / threads, kSMs * 4));
    const dim3 grid(bx, nb > 0 ? 2 : 1);
    switch (dim) {
    case 1: k_bbox_pair<1><<<grid, threads, 0, s>>>(a, na, b, nb, acc); break;
    case 2: k_bbox_pair<2><<<grid, threads, 0, s>>>(a, na, b, nb, acc); break;
    case 3: k_bbox_pair<3><<<grid, threads, 0, s>>>(a, na, b, nb, acc); break;
    case 4: k_bbox_pair<4><<<grid, threads, 0, s>>>(a, na, b, nb, acc); break;
    default: k_bbox_pair<5><<<grid, threads, 0, s>>>(a, na, b, nb, acc); break;
    }
    FM_CHECK_LAUNCH();
    if (cudaMemcpyAsync(keys_host, acc, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return FM_ERR_CUDA;
    return FM_OK;
}

int fm_bbox_decode(int dim, const unsigned long long *keys_host, double *lohi_host) {
    if (dim < 1 || dim > kMaxDim || !keys_host || !lohi_host) return FM_ERR_ARG;
    for (int arr = 0; arr < 2; arr++)
        for (int k = 0; k < dim; k++) {
            lohi_host[arr * 2 * dim + k] = host_dval(keys_host[arr * 2 * dim + k]);
            lohi_host[arr * 2 * dim + dim + k] = host_dval(~keys_host[arr * 2 * dim + dim + k]);
        }
    return FM_OK;
}

int fm_bbox_pair(int dim, const double *a, int64_t na, const double *b, int64_t nb,
                 double *lohi_host, void *workspace, fm_stream_t stream) {
    if (!lohi_host) return FM_ERR_ARG;
    unsigned long long h[4 * kMaxDim];
    const int rc = fm_bbox_pair_async(dim, a, na, b, nb, h, workspace, stream);
    if (rc) return rc;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return FM_ERR_CUDA;
    return fm_bbox_decode(dim, h, lohi_host);
}

/* locate.py:50-62 (_pad_bbox) and 34-47 (_grid_shape) in C, for any dim
 * (dim != 2: cells of equal side), bit for bit the Python grid_geometry(). */
int fm_grid_geometry(int dim, const double *bbox_lo, const double *bbox_hi, int64_t n_points,
                     double cells_per_point, fm_grid *out, double *lo_out, double *hi_out) {
    if (dim < 1 || dim > kMaxDim || !out || !(cells_per_point > 0.0) || n_points < 0)
        return FM_ERR_ARG;
    double lo[kMaxDim], hi[kMaxDim];
    double span = 0.0;
    for (int k = 0; k < dim; k++) {
        lo[k] = bbox_lo[k];
        hi[k] = bbox_hi[k];
        const double e = hi[k] - lo[k];
        if (k == 0 || e > span) span = e;
    }
    span = span > 1.0 ? span : 1.0;  // max(float(np.max(hi - lo)), 1.0)
    const double pad = 1e-12 * span;
    for (int k = 0; k < dim; k++) {
        if (hi[k] - lo[k] <= 0.0) {
            const double h = 0.5 * (span > 1.0 ? span : 1.0);
            lo[k] -= h;
            hi[k] += h;
        } else {
            lo[k] -= pad;
            hi[k] += pad;
        }
    }
    int64_t shape[kMaxDim];
    const double target = 1.0 > cells_per_point * (double)n_points ? 1.0
                                                                    : cells_per_point * (double)n_points;
    if (dim == 2) {
        const double w = hi[0] - lo[0] > 0.0 ? hi[0] - lo[0] : 0.0;
        const double h = hi[1] - lo[1] > 0.0 ? hi[1] - lo[1] : 0.0;
        int64_t nx, ny;
        if (w <= 0.0 && h <= 0.0) {
            nx = ny = 1;
        } else if (w <= 0.0) {
            nx = 1;
            ny = std::max<int64_t>(1, (int64_t)nearbyint(target));
        } else if (h <= 0.0) {
            nx = std::max<int64_t>(1, (int64_t)nearbyint(target));
            ny = 1;
        } else {
            nx = std::max<int64_t>(1, (int64_t)nearbyint(sqrt(target * w / h)));
            ny = std::max<int64_t>(1, (int64_t)nearbyint(target / (double)nx));
        }
        shape[0] = nx;
        shape[1] = ny;
    } else {
        double prod = 1.0;
        for (int k = 0; k < dim; k++) prod *= hi[k] - lo[k];
        const double side = pow(prod / target, 1.0 / dim);
        for (int k = 0; k < dim; k++)
            shape[k] = std::max<int64_t>(1, (int64_t)nearbyint((hi[k] - lo[k]) / side));
    }
    memset(out, 0, sizeof *out);
    out->dim = dim;
    int64_t ncell = 1;
    for (int k = 0; k < kMaxDim; k++) {
        if (k < dim) {
            out->n[k] = shape[k];
            out->lo[k] = lo[k];
            out->inv_d[k] = 1.0 / ((hi[k] - lo[k]) / (double)shape[k]);
            ncell *= shape[k];
            if (lo_out) lo_out[k] = lo[k];
            if (hi_out) hi_out[k] = hi[k];
        } else {
            out->n[k] = 1;
            out->lo[k] = 0.0;
            out->inv_d[k] = 1.0;
        }
    }
    out->ncell = ncell;
    return FM_OK;
}

size_t fm_scan_workspace(int64_t n) { return scan_workspace_bytes(n); }

int fm_offsets_from_counts(const int32_t *counts, int64_t n, int64_t *offsets, void *workspace,
                           size_t workspace_bytes, fm_stream_t stream) {
    return exclusive_scan<int32_t, int64_t>(counts, n, offsets, workspace, workspace_bytes,
                                            (cudaStream_t)stream);
}

}  // extern "C"
