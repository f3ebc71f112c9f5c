// fm_kernels.cuh -- kernel templates (instantiated per dimension in fm_dimN.cu).
//
// Work split: one lane group (G lanes) per target; a warp holds 32/G groups
// and walks the targets in tiles of 32/G consecutive entries of the
// processing order `perm` (cell order of the source grid, so the groups of
// a warp/CTA touch neighbouring sources).  All loops that contain warp
// collectives have warp-uniform trip counts.
#pragma once

#include "fm_fit.cuh"
#include "fm_search.cuh"

#include <algorithm>
#include <cstdlib>

namespace fm {

constexpr int kBlock = 128;

// Per processing position k, written by the select pass so the build's first
// loads are indexed by k only (no perm -> target -> count chain):
// (target id, support size, final radius).
struct __align__(16) PosInfo {
    int32_t tid;
    int32_t m;
    double r;
};
__device__ __forceinline__ PosInfo make_pos_info(int32_t tid, int32_t m, double r) {
    PosInfo p;
    p.tid = tid;
    p.m = m;
    p.r = r;
    return p;
}

struct SearchArgs {
    GridDev g;
    const int32_t *cell_start;
    const double *sorted_pts;
    const int32_t *sorted_ids;
    const double *targets;
    int64_t nt;
    const int32_t *perm;
    fm_select sel;
    const double *radii;  // final per-target radius (adaptive), or null
};

template <int DIM>
__device__ __forceinline__ void load_target(const double *__restrict__ targets, int64_t i,
                                            bool active, double *t) {
#pragma unroll
    for (int a = 0; a < DIM; a++) t[a] = active ? targets[i * DIM + a] : 0.0;
}

// --------------------------------------------------------- stats helpers
// stats arrays: pairs of (count, first index) plus min/max slots; written
// with warp-aggregated atomics.
static __global__ void k_stats_init(int32_t *stats, int n, int kind,
                                    int32_t *zero = nullptr, int nzero = 0) {
    const int i = threadIdx.x;
    if (zero && i < nzero) zero[i] = 0;
    if (i >= n) return;
    if (kind == 0)  // count stats: max, min, nshort, first, nstatus, first
        stats[i] = (i == 1 || i == 3 || i == 5) ? INT32_MAX : 0;
    else  // fit stats: nfail, first
        stats[i] = i == 1 ? INT32_MAX : 0;
}

__device__ __forceinline__ void warp_flush_pair(int32_t *slot, int n, int first) {
    n = __reduce_add_sync(FM_FULL_MASK, n);
    first = __reduce_min_sync(FM_FULL_MASK, (unsigned)first);
    if ((threadIdx.x & 31) == 0 && n > 0) {
        atomicAdd(slot, n);
        atomicMin(slot + 1, first);
    }
}

// ------------------------------------------------------------ count pass
template <int DIM, int G>
__global__ void __launch_bounds__(kBlock) k_support_count(SearchArgs s, int32_t min_required,
                                                          int32_t *__restrict__ counts,
                                                          double *__restrict__ radii,
                                                          uint8_t *__restrict__ status,
                                                          int32_t *__restrict__ stats) {
    __shared__ RowTable<G> rts[kBlock / G];
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, glane = lane & (G - 1);
    RowTable<G> &rt = rts[threadIdx.x / G];
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    int local_max = 0, local_min = INT32_MAX;
    int nshort = 0, first_short = INT32_MAX, nstat = 0, first_stat = INT32_MAX;
    for (int64_t tile = warp; tile * GPW < s.nt; tile += nwarps) {
        const int64_t k = tile * GPW + lane / G;
        const bool active = k < s.nt;
        const int64_t tid = active ? (s.perm ? (int64_t)s.perm[k] : k) : 0;
        double t[DIM];
        load_target<DIM>(s.targets, tid, active, t);
        int m;
        if (s.sel.adaptive) {
            double r;
            uint8_t st;
            m = adaptive_radius<DIM, G>(s.g, s.cell_start, s.sorted_pts, t, s.sel, active, lane,
                                        glane, rt, r, st);
            if (active && glane == 0) {
                if (radii) radii[tid] = r;
                if (status) status[tid] = st;
                if (st) {
                    nstat++;
                    first_stat = min(first_stat, (int)tid);
                }
            }
        } else {
            m = count_within<DIM, G>(s.g, s.cell_start, s.sorted_pts, t, s.sel.r_c, active, lane,
                                     glane, rt);
        }
        if (active && glane == 0) {
            counts[tid] = m;
            local_max = max(local_max, m);
            local_min = min(local_min, m);
            if (m < min_required) {
                nshort++;
                first_short = min(first_short, (int)tid);
            }
        }
    }
    if (stats) {
        local_max = __reduce_max_sync(FM_FULL_MASK, local_max);
        local_min = __reduce_min_sync(FM_FULL_MASK, (unsigned)local_min);
        if (lane == 0) {
            atomicMax(stats + 0, local_max);
            atomicMin(stats + 1, local_min);
        }
        warp_flush_pair(stats + 2, nshort, first_short);
        warp_flush_pair(stats + 4, nstat, first_stat);
    }
}

// per-group dynamic shared layout for the fill / fused kernels
template <int G>
struct GroupSmem {
    RowTable<G> *rt;
    int32_t *id, *pos, *sid, *spos;
    double *sR, *sQ;
};

template <int G>
__host__ __device__ inline size_t group_smem_bytes(int cap, int K) {
    return sizeof(RowTable<G>) + (size_t)cap * 4 * sizeof(int32_t) +
           (size_t)(K * K + 4 * K) * sizeof(double) + 16;
}

template <int G>
__device__ __forceinline__ GroupSmem<G> carve(char *base, int cap, int K) {
    const int grp = threadIdx.x / G;
    char *p = base + (size_t)grp * ((group_smem_bytes<G>(cap, K) + 15) & ~(size_t)15);
    GroupSmem<G> gs;
    gs.sR = reinterpret_cast<double *>(p);
    p += (size_t)K * K * sizeof(double);
    gs.sQ = reinterpret_cast<double *>(p);
    p += (size_t)4 * K * sizeof(double);  // sQ, then the reflector scalars (fit_rows)
    gs.rt = reinterpret_cast<RowTable<G> *>(p);
    p += sizeof(RowTable<G>);
    gs.id = reinterpret_cast<int32_t *>(p);
    gs.pos = gs.id + cap;
    gs.sid = gs.pos + cap;
    gs.spos = gs.sid + cap;
    return gs;
}

template <int G>
__host__ __device__ inline size_t block_smem_bytes(int cap, int K) {
    return (size_t)(kBlock / G) * ((group_smem_bytes<G>(cap, K) + 15) & ~(size_t)15);
}

// ------------------------------------------------------------- fill pass
// CSR of (idx, dist[, w]) in ascending id order at offsets[t].
template <int DIM, int G>
__global__ void __launch_bounds__(kBlock) k_support_fill(SearchArgs s, const int64_t *__restrict__ offsets,
                                                         int cap, int64_t *__restrict__ idx,
                                                         double *__restrict__ dist, int rbf_kind,
                                                         double rbf_a, double *__restrict__ w) {
    extern __shared__ __align__(16) char smem[];
    GroupSmem<G> gs = carve<G>(smem, cap, 0);
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, glane = lane & (G - 1);
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t tile = warp; tile * GPW < s.nt; tile += nwarps) {
        const int64_t k = tile * GPW + lane / G;
        const bool active = k < s.nt;
        const int64_t tid = active ? (s.perm ? (int64_t)s.perm[k] : k) : 0;
        double t[DIM];
        load_target<DIM>(s.targets, tid, active, t);
        const double r = active ? (s.radii ? s.radii[tid] : s.sel.r_c) : 0.0;
        const int m = collect_sorted<DIM, G>(s.g, s.cell_start, s.sorted_pts, s.sorted_ids, t, r,
                                             active, lane, glane, *gs.rt, gs.id, gs.pos, gs.sid,
                                             gs.spos, cap);
        if (active) {
            const int64_t off = offsets[tid];
            const int mm = m < cap ? m : cap;
            for (int e = glane; e < mm; e += G) {
                double p[DIM];
                load_point<DIM>(s.sorted_pts, gs.spos[e], p);
                const double d = __dsqrt_rn(dist2_rn<DIM>(p, t));
                idx[off + e] = gs.sid[e];
                dist[off + e] = d;
                if (w) w[off + e] = rbf_one(rbf_kind, rbf_a, r, d);
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------- operator build
// One launch builds the fits of positions k = klist[i] (or i) of the
// processing order; target t = perm[k].  The support of each target comes
// from the select pass's slot buffer (FROM_SLOTS: sorted ids + grid
// positions, no search) or is re-gathered here (rescan: overflow targets,
// and the standalone fm_build_operator / fm_transfer_values ABI).
// OP: operator row written at offsets[k] (rows stored in processing order).
// SOLVE: values[t] for the scalar field src_val.
struct BuildArgs {
    const int32_t *klist;  // positions to process, or null for 0..nk-1
    int stage;             // shared memory sized for the cp.async pipeline
    int64_t nk;            // positions (upper bound when nk_dev is set)
    const int32_t *nk_dev;  // optional device-side position count (read at kernel start)
    const int32_t *slot_pos;
    int slot_cap;
    const int32_t *counts;  // support size per target (FROM_SLOTS)
    const PosInfo *pos_info;  // optional per-position (tid, m, r) from the select pass
    const double *pos_t;      // optional per-position target coordinates
    const int64_t *offsets;
    int cap;  // rescan list capacity
    int rbf_kind;
    double rbf_a;
    fm_fit fp;
    const double *src_val;
    int32_t *col;
    double *val;
    double *values;
    uint8_t *status;
    int32_t *stats;
};

// One target of the build from its gathered support rows (coordinates p,
// source ids): weights -> fit -> operator row (or value).  A function, not a
// lambda: a non-inlined lambda capturing the kernel arguments by reference
// puts them in a local-memory stack frame.
template <int DIM, int DEG, int G, int ROWS, bool SOLVE>
__device__ __forceinline__ void build_core(const BuildArgs &b, const GroupSmem<G> &gs, int lane,
                                           int glane, bool active, int64_t tid,
                                           const double (&t)[DIM], double r, int m,
                                           const double (&p)[ROWS][DIM],
                                           const int32_t (&ids)[ROWS], int64_t off, int &nfail,
                                           int &first_fail) {
    constexpr int K = Monos<DIM, DEG>::K;
    bool valid[ROWS];
    double w[ROWS], f[ROWS];
    const double inv_r = active ? 1.0 / r : 0.0;
    FM_DCHECK(!active || (m >= 0 && m <= ROWS * G));
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        const int i = q * G + glane;
        valid[q] = i < m;
        w[q] = 0.0;
        f[q] = 0.0;
        if (valid[q]) {
            const double d = __dsqrt_rn(dist2_rn<DIM>(p[q], t));
            w[q] = fabs(rbf_fast(b.rbf_kind, b.rbf_a, r, inv_r, d));  // pointwise.py:301
            if (SOLVE) f[q] = __ldg(b.src_val + ids[q]);
        }
    }
    double y[ROWS], coeffs[K], value = 0.0;
    const int st = fit_rows<DIM, DEG, G, ROWS, SOLVE>(b.fp, t, m, valid, p, w, f, lane, glane,
                                                      gs.sR, gs.sQ, y, coeffs, value);
    if (active) {
        if (glane == 0) {
            b.status[tid] = (uint8_t)st;
            if (st != FM_FIT_OK) {
                nfail++;
                first_fail = min(first_fail, (int)tid);
            }
        }
        if (SOLVE) {
            if (glane == 0) b.values[tid] = st == FM_FIT_OK ? value : NAN;
        } else {
#pragma unroll
            for (int q = 0; q < ROWS; q++) {
                if (valid[q]) {
                    const int i = q * G + glane;
                    b.col[off + i] = ids[q];
                    b.val[off + i] = st == FM_FIT_OK ? y[q] : NAN;
                }
            }
        }
    }
    __syncwarp();
}

// build_core with the support rows gathered from global memory by grid position
template <int DIM, int DEG, int G, int ROWS, bool SOLVE>
__device__ __forceinline__ void build_one(const SearchArgs &s, const BuildArgs &b,
                                          const GroupSmem<G> &gs, int lane, int glane,
                                          bool active, int64_t k, int64_t tid,
                                          const double (&t)[DIM], double r, int m,
                                          const int32_t (&spos)[ROWS], int64_t off, int &nfail,
                                          int &first_fail) {
    int32_t ids[ROWS];  // source ids of the support rows (col of the operator)
    double p[ROWS][DIM];
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        const bool v = q * G + glane < m;
        ids[q] = v ? __ldg(s.sorted_ids + spos[q]) : 0;
#pragma unroll
        for (int a = 0; a < DIM; a++) p[q][a] = 0.0;
        if (v) load_point<DIM>(s.sorted_pts, spos[q], p[q]);
    }
    build_core<DIM, DEG, G, ROWS, SOLVE>(b, gs, lane, glane, active, tid, t, r, m, p, ids, off,
                                         nfail, first_fail);
}

// ---------------------------------------------------- staged (cp.async) build
// Per group, in shared memory: three record slots (the select pass's
// position record, target coordinates, row offset, and the support's grid
// positions) and two buffers of gathered support rows (coordinates, source
// ids).  While tile n is fitted, tile n+1's support rows and tile n+2's
// records are in flight as cp.async copies -- no registers held, no
// dependent-load stalls in the fit.
template <int DIM, int G, int ROWS>
struct StageSmem {
    struct __align__(16) Rec {
        PosInfo pi;
        double t[DIM];
        int64_t off;
    };
    Rec rec[3];
    int32_t spos[3][ROWS * G];
    double pts[2][ROWS * G][DIM];
    int32_t ids[2][ROWS * G];
};

template <int DIM, int G, int ROWS>
__host__ __device__ constexpr size_t stage_bytes() {
    return (sizeof(StageSmem<DIM, G, ROWS>) + 15) & ~(size_t)15;
}

// records + grid positions of position k (slot `sl`); inactive: zero record
template <int DIM, int G, int ROWS, bool SOLVE>
__device__ __forceinline__ void stage_records(const BuildArgs &b, StageSmem<DIM, G, ROWS> &S,
                                              int sl, bool act, int64_t k, int glane) {
    auto &R = S.rec[sl];
    if (glane == 0) cp_async16(&R.pi, b.pos_info + k, act);
    if (glane == (1 % G)) {
        if (DIM == 2)
            cp_async16(&R.t[0], b.pos_t + k * DIM, act);
        else
#pragma unroll
            for (int a = 0; a < DIM; a++) cp_async8(&R.t[a], b.pos_t + k * DIM + a, act);
    }
    if (!SOLVE && glane == (2 % G)) cp_async8(&R.off, b.offsets + k, act);
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        const int i = q * G + glane;
        cp_async4(&S.spos[sl][i], b.slot_pos + k * b.slot_cap + i, act && i < b.slot_cap);
    }
}

// support rows (coordinates + ids) of the record in slot `sl` into buffer `pb`
template <int DIM, int G, int ROWS>
__device__ __forceinline__ void stage_rows(const SearchArgs &s, const BuildArgs &b,
                                           StageSmem<DIM, G, ROWS> &S, int sl, int pb,
                                           int glane) {
    const int m = S.rec[sl].pi.m;
    const bool fits = m <= b.slot_cap;
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        const int i = q * G + glane;
        const bool v = fits && i < m;
        const int64_t sp = v ? S.spos[sl][i] : 0;
        FM_DCHECK(sp >= 0 && (!v || i < b.slot_cap));
        if (DIM == 2)
            cp_async16(&S.pts[pb][i][0], s.sorted_pts + sp * DIM, v);
        else
#pragma unroll
            for (int a = 0; a < DIM; a++) cp_async8(&S.pts[pb][i][a], s.sorted_pts + sp * DIM + a, v);
        cp_async4(&S.ids[pb][i], s.sorted_ids + sp, v);
    }
}

#ifndef FM_BUILD_MINB8
#define FM_BUILD_MINB8 4
#endif
#ifndef FM_BUILD_MINB8_R2
#define FM_BUILD_MINB8_R2 4
#endif
#ifndef FM_BUILD_MINB4
#define FM_BUILD_MINB4 4
#endif
#ifndef FM_BUILD_MINB4_R6
#define FM_BUILD_MINB4_R6 3
#endif
template <int DIM, int DEG, int G, int ROWS, bool SOLVE, bool FROM_SLOTS>
__global__ void __launch_bounds__(kBlock, (G == 8 && ROWS <= 2)   ? FM_BUILD_MINB8_R2
                                          : (G == 8 && ROWS <= 4) ? FM_BUILD_MINB8
                                          : (G == 4)              ? (ROWS <= 4 ? FM_BUILD_MINB4 : FM_BUILD_MINB4_R6)
                                                                  : 1) k_build(SearchArgs s,
                                                                                 BuildArgs b) {
    constexpr int K = Monos<DIM, DEG>::K;
    extern __shared__ __align__(16) char smem[];
    int nfail = 0, first_fail = INT32_MAX;
    GroupSmem<G> gs = carve<G>(smem, FROM_SLOTS ? 0 : b.cap, K);
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, glane = lane & (G - 1);
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t stride = nwarps * GPW;
    const bool staged = FROM_SLOTS && b.pos_info != nullptr && b.stage;
    const int64_t nk = b.nk_dev ? (int64_t)*b.nk_dev : b.nk;
    auto kof = [&](int64_t ii) -> int64_t {
        return b.klist ? (ii < nk ? (int64_t)b.klist[ii] : 0) : ii;
    };
    // the pipeline's look-ahead position: a branch-free load kept as int32
    // until its use a tile later (a guarded load widened to int64 made the
    // warp wait for it at once: 6% of the build's stall samples)
    auto kof32 = [&](int64_t ii) -> int32_t {
        if (!b.klist) return (int32_t)ii;
        const int64_t j = ii < nk ? ii : (nk > 0 ? nk - 1 : 0);
        return __ldg(b.klist + j);
    };

    if (staged) {
        // cp.async pipeline (StageSmem): records two tiles ahead, support
        // rows one tile ahead, the fit of the current tile from shared memory
        using SS = StageSmem<DIM, G, ROWS>;
        SS &S = *reinterpret_cast<SS *>(smem + block_smem_bytes<G>(0, K) +
                                        (threadIdx.x / G) * stage_bytes<DIM, G, ROWS>());
        const int64_t ii0 = warp * GPW + lane / G;
        stage_records<DIM, G, ROWS, SOLVE>(b, S, 0, ii0 < nk, kof(ii0), glane);
        cp_async_commit();
        stage_records<DIM, G, ROWS, SOLVE>(b, S, 1, ii0 + stride < nk, kof(ii0 + stride),
                                           glane);
        cp_async_commit();
        int32_t k_next = kof32(ii0 + 2 * stride);
        cp_async_wait_all();
        __syncwarp();
        stage_rows<DIM, G, ROWS>(s, b, S, 0, 0, glane);
        cp_async_commit();
        int n = 0;
        for (int64_t tile = warp; tile * GPW < nk; tile += nwarps, n++) {
            const int64_t ii = tile * GPW + lane / G;
            const int cs = n % 3, cb = n & 1;
            cp_async_wait_all();  // rows of tile n, records of tile n+1
            __syncwarp();
            stage_rows<DIM, G, ROWS>(s, b, S, (n + 1) % 3, cb ^ 1, glane);
            cp_async_commit();
            stage_records<DIM, G, ROWS, SOLVE>(b, S, (n + 2) % 3, ii + 2 * stride < nk, k_next,
                                               glane);
            cp_async_commit();
            k_next = kof32(ii + 3 * stride);
            const auto &R = S.rec[cs];
            const PosInfo pi = R.pi;
            int m = pi.m;
            bool active = ii < nk;
            if (m > b.slot_cap) {  // overflow: built by the rescan launch
                active = false;
                m = 0;
            }
            double t[DIM], p[ROWS][DIM];
            int32_t ids[ROWS];
#pragma unroll
            for (int a = 0; a < DIM; a++) t[a] = R.t[a];
#pragma unroll
            for (int q = 0; q < ROWS; q++) {
                const int i = q * G + glane;
#pragma unroll
                for (int a = 0; a < DIM; a++) p[q][a] = S.pts[cb][i][a];
                ids[q] = S.ids[cb][i];
            }
            build_core<DIM, DEG, G, ROWS, SOLVE>(b, gs, lane, glane, active, pi.tid, t, pi.r, m,
                                                 p, ids, SOLVE ? 0 : R.off, nfail, first_fail);
        }
        cp_async_wait_all();
    } else {
        for (int64_t tile = warp; tile * GPW < nk; tile += nwarps) {
            const int64_t ii = tile * GPW + lane / G;
            bool active = ii < nk;
            const int64_t k = active ? kof(ii) : 0;
            const int64_t tid = active ? (s.perm ? (int64_t)s.perm[k] : k) : 0;
            double t[DIM];
            load_target<DIM>(s.targets, tid, active, t);
            const double r = active ? (s.radii ? s.radii[tid] : s.sel.r_c) : 0.0;
            int m = 0;
            int32_t spos[ROWS];
            if (FROM_SLOTS) {
                m = active ? b.counts[tid] : 0;
                if (m > b.slot_cap) {  // overflow: built by the rescan launch
                    active = false;
                    m = 0;
                }
#pragma unroll
                for (int q = 0; q < ROWS; q++) {
                    const int i = q * G + glane;
                    spos[q] = i < m ? __ldg(b.slot_pos + k * b.slot_cap + i) : 0;
                }
            } else {
                m = collect_sorted<DIM, G>(s.g, s.cell_start, s.sorted_pts, s.sorted_ids, t, r,
                                           active, lane, glane, *gs.rt, gs.id, gs.pos, gs.sid,
                                           gs.spos, b.cap);
                if (m > b.cap) m = b.cap;  // host sizes cap >= max count
#pragma unroll
                for (int q = 0; q < ROWS; q++) {
                    const int i = q * G + glane;
                    spos[q] = i < m ? gs.spos[i] : 0;
                }
            }
            const int64_t off = (!SOLVE && active) ? b.offsets[k] : 0;
            build_one<DIM, DEG, G, ROWS, SOLVE>(s, b, gs, lane, glane, active, k, tid, t, r, m,
                                                spos, off, nfail, first_fail);
        }
    }
    if (b.stats) warp_flush_pair(b.stats, nfail, first_fail);
}

// ----------------------------------------------------- select pass
// Count pass that also emits each target's support, sorted by source id,
// into a fixed-stride slot buffer indexed by processing position
// (slot_id/slot_pos[k*slot_cap + i]).  Targets whose support exceeds the
// slot (or the per-group list) are appended to overflow (positions k) and
// rebuilt by the rescan build.
// stats[8]: max, min, #short, first short, #status, first status, #overflow, 0.
template <int DIM, int G>
// 8-lane groups (1-D/2-D): 8 CTAs/SM (64 registers; measured 0.74 -> 0.64 ms
// on C2 against the unconstrained 80-register build at 6 CTAs/SM)
__global__ void __launch_bounds__(kBlock, G == 8 ? 8 : 1) k_select(SearchArgs s, int32_t min_required, int lcap,
                                                   int32_t *__restrict__ counts,
                                                   double *__restrict__ radii,
                                                   uint8_t *__restrict__ status,
                                                   int32_t *__restrict__ slot_id,
                                                   int32_t *__restrict__ slot_pos, int slot_cap,
                                                   int32_t *__restrict__ overflow,
                                                   int32_t *__restrict__ stats,
                                                   PosInfo *__restrict__ pos_info,
                                                   double *__restrict__ pos_t) {
    extern __shared__ __align__(16) char smem[];
    constexpr int GPW = 32 / G;
    const int grp = threadIdx.x / G;
    const size_t per = ((size_t)lcap * 16 + sizeof(RowTable<G>) + 15) & ~(size_t)15;
    char *base = smem + grp * per;
    ListBuf lb;
    lb.d = reinterpret_cast<double *>(base);
    lb.id = reinterpret_cast<int32_t *>(base + (size_t)lcap * 8);
    lb.pos = lb.id + lcap;
    lb.cap = lcap;
    RowTable<G> &rt = *reinterpret_cast<RowTable<G> *>(base + (size_t)lcap * 16);
    __shared__ RadiusTable tab;
    fill_radius_table(tab, s.sel);
    const int lane = threadIdx.x & 31, glane = lane & (G - 1);
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    int local_max = 0, local_min = INT32_MAX;
    int nshort = 0, first_short = INT32_MAX, nstat = 0, first_stat = INT32_MAX;
    for (int64_t tile = warp; tile * GPW < s.nt; tile += nwarps) {
        const int64_t k = tile * GPW + lane / G;
        const bool active = k < s.nt;
        const int64_t tid = active ? (s.perm ? (int64_t)s.perm[k] : k) : 0;
        double t[DIM];
        load_target<DIM>(s.targets, tid, active, t);
        double r;
        uint8_t st;
        bool listed;
        const int m = select_target<DIM, G>(s.g, s.cell_start, s.sorted_pts, s.sorted_ids, t, s.sel,
                                            tab, active, lane, glane, rt, lb, r, st, listed);
        if (active) {
            if (listed && m <= slot_cap) {
                // supports in discovery order (the fit does not need id order;
                // the reference-format CSR is sorted by fm_support_fill)
                int32_t *opos = slot_pos + k * slot_cap;
                for (int e = glane; e < m; e += G) {
                    if (slot_id) slot_id[k * slot_cap + e] = lb.id[e];
                    opos[e] = lb.pos[e];
                }
            } else if (glane == 0) {
                overflow[atomicAdd(stats + 6, 1)] = (int32_t)k;
            }
            if (pos_info && glane == 0)
                pos_info[k] = make_pos_info((int32_t)tid, m, s.sel.adaptive ? r : s.sel.r_c);
            if (pos_t && glane < DIM) {
#pragma unroll
                for (int a = 0; a < DIM; a++)
                    if (a == glane) pos_t[k * DIM + a] = t[a];
            }
            if (glane == 0) {
                counts[tid] = m;
                if (s.sel.adaptive) {
                    if (radii) radii[tid] = r;
                    if (status) status[tid] = st;
                    if (st) {
                        nstat++;
                        first_stat = min(first_stat, (int)tid);
                    }
                }
                local_max = max(local_max, m);
                local_min = min(local_min, m);
                if (m < min_required) {
                    nshort++;
                    first_short = min(first_short, (int)tid);
                }
            }
        }
        __syncwarp();
    }
    local_max = __reduce_max_sync(FM_FULL_MASK, local_max);
    local_min = __reduce_min_sync(FM_FULL_MASK, (unsigned)local_min);
    if (lane == 0) {
        atomicMax(stats + 0, local_max);
        atomicMin(stats + 1, local_min);
    }
    warp_flush_pair(stats + 2, nshort, first_short);
    warp_flush_pair(stats + 4, nstat, first_stat);
}

// size bucket of a support (fieldmap.h FM_BUCKET_EDGES)
__device__ __forceinline__ int bucket_of(int m) {
    constexpr int edges[FM_NBUCKETS] = FM_BUCKET_EDGES;
    int b = 0;
#pragma unroll
    for (int i = 0; i < FM_NBUCKETS - 1; i++) b += m > edges[i];
    return b;
}

// Optional fused outputs of the thread select (fm_select_supports_bucketed):
// per position the row length of the ordered offsets (0 for a support beyond
// the slot when cap_rows) and the size-bucket lists of fm_offsets_ordered.
struct SelectBuckets {
    int32_t *pos_counts;    // NULL: not requested
    int32_t *bucket_list;   // FM_NBUCKETS lists of stride nt
    int32_t *bucket_count;  // zeroed before the launch
    int cap_rows;
};

// Thread-per-target select pass (1-D / 2-D): same outputs as k_select.
// The supports go from the per-thread shared-memory lists to the slots with
// one coalesced warp store per target (lanes over entries).
constexpr int kThreadListCap = 48;  // default 2-D slot: 8 CTAs/SM of 25 KB lists

template <int DIM>
__global__ void __launch_bounds__(kBlock, 8) k_select_t(SearchArgs s, int32_t min_required, int lcap,
                                                     int32_t *__restrict__ counts,
                                                     double *__restrict__ radii,
                                                     uint8_t *__restrict__ status,
                                                     int32_t *__restrict__ slot_id,
                                                     int32_t *__restrict__ slot_pos, int slot_cap,
                                                     int32_t *__restrict__ overflow,
                                                     int32_t *__restrict__ stats,
                                                     PosInfo *__restrict__ pos_info,
                                                     double *__restrict__ pos_t,
                                                     SelectBuckets bk) {
    extern __shared__ __align__(16) char smem[];
    const int stride = lcap | 1;  // odd: a warp's appends spread over the banks
    int32_t *lpos_all = reinterpret_cast<int32_t *>(smem);
    __shared__ RadiusTable tab;
    fill_radius_table(tab, s.sel);
    ThreadList L;
    L.e = lpos_all + threadIdx.x * stride;
    L.cap = lcap;
    const int lane = threadIdx.x & 31;
    const int wbase = threadIdx.x & ~31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    int local_max = 0, local_min = INT32_MAX;
    int nshort = 0, first_short = INT32_MAX, nstat = 0, first_stat = INT32_MAX;
    for (int64_t tile = warp; tile * 32 < s.nt; tile += nwarps) {
        const int64_t k = tile * 32 + lane;
        const bool active = k < s.nt;
        int m = 0;
        bool slotted = false;
        if (active) {
            const int64_t tid = s.perm ? (int64_t)__ldg(s.perm + k) : k;
            FM_DCHECK(tid >= 0 && tid < s.nt);
            double t[DIM];
            load_target<DIM>(s.targets, tid, true, t);
            double r;
            uint8_t st;
            bool listed;
            m = select_thread<DIM>(s.g, s.cell_start, s.sorted_pts, t, s.sel, tab, L, r, st,
                                   listed);
            slotted = listed && m <= slot_cap;
            if (!slotted) overflow[atomicAdd(stats + 6, 1)] = (int32_t)k;
            if (pos_info) pos_info[k] = make_pos_info((int32_t)tid, m, s.sel.adaptive ? r : s.sel.r_c);
            if (pos_t) {
#pragma unroll
                for (int a = 0; a < DIM; a++) pos_t[k * DIM + a] = t[a];
            }
            counts[tid] = m;
            if (s.sel.adaptive) {
                if (radii) radii[tid] = r;
                if (status) status[tid] = st;
                if (st) {
                    nstat++;
                    first_stat = min(first_stat, (int)tid);
                }
            }
            local_max = max(local_max, m);
            local_min = min(local_min, m);
            if (m < min_required) {
                nshort++;
                first_short = min(first_short, (int)tid);
            }
        }
        if (bk.pos_counts) {  // what fm_offsets_ordered(_capped) derives, fused
            if (active) bk.pos_counts[k] = (bk.cap_rows && !slotted) ? 0 : m;
            const int b = (active && slotted) ? bucket_of(m) : -1;
            const unsigned peers = __match_any_sync(FM_FULL_MASK, b);
            const int leader = __ffs(peers) - 1;
            int at = 0;
            if (lane == leader && b >= 0) at = atomicAdd(bk.bucket_count + b, __popc(peers));
            at = __shfl_sync(FM_FULL_MASK, at, leader);
            FM_DCHECK(b < 0 || at + __popc(peers) <= s.nt);
            if (b >= 0)
                bk.bucket_list[(int64_t)b * s.nt + at + __popc(peers & ((1u << lane) - 1u))] =
                    (int32_t)k;
        }
        __syncwarp();
        // supports -> slots: one target at a time, lanes over its entries
        const int mine = slotted ? m : 0;
        unsigned todo = __ballot_sync(FM_FULL_MASK, mine > 0);
        while (todo) {
            const int r = __ffs(todo) - 1;
            todo &= todo - 1;
            const int mr = __shfl_sync(FM_FULL_MASK, mine, r);
            const int64_t kr = tile * 32 + r;
            const int32_t *lp = lpos_all + (wbase + r) * stride;
            int32_t *op = slot_pos + kr * slot_cap;
            FM_DCHECK(kr < s.nt && mr <= slot_cap);
            for (int e = lane; e < mr; e += 32) {
                const int32_t p = lp[e] & kPosMask;
                op[e] = p;
                if (slot_id) slot_id[kr * slot_cap + e] = __ldg(s.sorted_ids + p);
            }
        }
        __syncwarp();
    }
    local_max = __reduce_max_sync(FM_FULL_MASK, local_max);
    local_min = __reduce_min_sync(FM_FULL_MASK, (unsigned)local_min);
    if (lane == 0) {
        atomicMax(stats + 0, local_max);
        atomicMin(stats + 1, local_min);
    }
    warp_flush_pair(stats + 2, nshort, first_short);
    warp_flush_pair(stats + 4, nstat, first_stat);
}


// counts in processing order (input of the ordered offsets scan) and,
// with bucket_list, the positions partitioned by support size.  Appends are
// aggregated per block: warps count into shared memory, then ONE global
// atomic per bucket and block tile of 1024 positions reserves the block's
// range (per-warp global atomics on the 9 bucket counters serialized).
// positions p0 + [0, n): out (may be NULL) indexed from 0, bucket lists
// with stride lstride holding absolute positions
constexpr int kGatherItems = 4;
static __global__ void __launch_bounds__(256) k_gather_counts(
    const int32_t *__restrict__ counts, const int32_t *__restrict__ perm, int64_t n,
    int32_t *__restrict__ out, int slot_cap, int32_t *__restrict__ bucket_list,
    int32_t *__restrict__ bucket_count, int64_t p0 = 0, int64_t lstride = -1,
    int row_cap = 0) {
    __shared__ int s_cnt[FM_NBUCKETS];
    __shared__ int s_base[FM_NBUCKETS];
    const int lane = threadIdx.x & 31;
    if (lstride < 0) lstride = n;
    constexpr int kTile = 256 * kGatherItems;
    for (int64_t base = (int64_t)blockIdx.x * kTile; base < n; base += (int64_t)gridDim.x * kTile) {
        int b[kGatherItems], at[kGatherItems];
        if (bucket_list && threadIdx.x < FM_NBUCKETS) s_cnt[threadIdx.x] = 0;
        if (bucket_list) __syncthreads();
#pragma unroll
        for (int it = 0; it < kGatherItems; it++) {
            const int64_t j = base + it * 256 + threadIdx.x;
            const int64_t i = p0 + j;
            const int m = j < n ? __ldg(counts + (perm ? __ldg(perm + i) : i)) : 0;
            if (j < n && out) out[j] = (row_cap > 0 && m > row_cap) ? 0 : m;
            b[it] = (j < n && m <= slot_cap) ? bucket_of(m) : -1;
            at[it] = 0;
            if (bucket_list) {
                const unsigned peers = __match_any_sync(FM_FULL_MASK, b[it]);
                const int leader = __ffs(peers) - 1;
                int a0 = 0;
                if (lane == leader && b[it] >= 0) a0 = atomicAdd(&s_cnt[b[it]], __popc(peers));
                at[it] = __shfl_sync(FM_FULL_MASK, a0, leader) +
                         __popc(peers & ((1u << lane) - 1u));
            }
        }
        if (!bucket_list) continue;
        __syncthreads();
        if (threadIdx.x < FM_NBUCKETS) {
            const int c = s_cnt[threadIdx.x];
            s_base[threadIdx.x] = c ? atomicAdd(bucket_count + threadIdx.x, c) : 0;
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < kGatherItems; it++)
            if (b[it] >= 0)
                bucket_list[(int64_t)b[it] * lstride + s_base[b[it]] + at[it]] =
                    (int32_t)(p0 + base + it * 256 + threadIdx.x);
    }
}

// ------------------------------------------------- fit_many (CSR input)
template <int DIM, int DEG, int G, int ROWS>
__global__ void __launch_bounds__(kBlock) k_fit_many(fm_fit fp, const double *__restrict__ targets,
                                                     int64_t nt, const int64_t *__restrict__ sup_off,
                                                     const int64_t *__restrict__ sup_idx,
                                                     const double *__restrict__ sup_w,
                                                     const double *__restrict__ src,
                                                     const double *__restrict__ src_val,
                                                     double *__restrict__ values,
                                                     double *__restrict__ coeffs_out,
                                                     uint8_t *__restrict__ status,
                                                     int32_t *__restrict__ stats) {
    constexpr int K = Monos<DIM, DEG>::K;
    int nfail = 0, first_fail = INT32_MAX;
    __shared__ double sRs[kBlock / G][K * K + 4 * K];
    double *sR = sRs[threadIdx.x / G];
    double *sQ = sR + K * K;
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31, glane = lane & (G - 1);
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t tile = warp; tile * GPW < nt; tile += nwarps) {
        const int64_t tid = tile * GPW + lane / G;
        const bool active = tid < nt;
        double t[DIM];
        load_target<DIM>(targets, tid, active, t);
        const int64_t off = active ? sup_off[tid] : 0;
        const int m = active ? (int)(sup_off[tid + 1] - off) : 0;
        bool valid[ROWS];
        double p[ROWS][DIM], w[ROWS], f[ROWS];
#pragma unroll
        for (int q = 0; q < ROWS; q++) {
            const int i = q * G + glane;
            valid[q] = i < m;
            w[q] = 0.0;
            f[q] = 0.0;
#pragma unroll
            for (int a = 0; a < DIM; a++) p[q][a] = 0.0;
            if (valid[q]) {
                const int64_t id = sup_idx[off + i];
                w[q] = sup_w[off + i];
#pragma unroll
                for (int a = 0; a < DIM; a++) p[q][a] = __ldg(src + id * DIM + a);
                f[q] = __ldg(src_val + id);
            }
        }
        double y[ROWS], coeffs[K], value = 0.0;
        const int st = fit_rows<DIM, DEG, G, ROWS, true>(fp, t, m, valid, p, w, f, lane, glane, sR,
                                                         sQ, y, coeffs, value);
        if (active) {
            if (glane == 0) {
                status[tid] = (uint8_t)st;
                values[tid] = st == FM_FIT_OK ? value : NAN;
                if (st != FM_FIT_OK) {
                    nfail++;
                    first_fail = min(first_fail, (int)tid);
                }
            }
            if (coeffs_out) {
#pragma unroll
                for (int c = 0; c < K; c++)
                    if (glane == (c % G)) coeffs_out[tid * K + c] = st == FM_FIT_OK ? coeffs[c] : NAN;
            }
        }
        __syncwarp();
    }
    if (stats) warp_flush_pair(stats, nfail, first_fail);
}

}  // namespace fm

#include "fm_big.cuh"

namespace fm {

// ------------------------------------------------------------ launchers
inline int grid_blocks(int64_t nt, int groups_per_block, int per_sm) {
    const int64_t need = (nt + groups_per_block - 1) / groups_per_block;
    const int64_t cap = (int64_t)kSMs * per_sm;
    return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

template <int DIM>
int launch_count(const SearchArgs &s, int32_t min_required, int32_t *counts, double *radii,
                 uint8_t *status, int32_t *stats, cudaStream_t st) {
    constexpr int G = 16;
    if (stats) k_stats_init<<<1, 32, 0, st>>>(stats, 6, 0);
    if (s.nt == 0) return FM_OK;
    k_support_count<DIM, G><<<grid_blocks(s.nt, kBlock / G, 16), kBlock, 0, st>>>(
        s, min_required, counts, radii, status, stats);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

template <int DIM>
int launch_fill(const SearchArgs &s, const int64_t *offsets, int cap, int64_t *idx, double *dist,
                int rbf_kind, double rbf_a, double *w, cudaStream_t st) {
    constexpr int G = 16;
    if (s.nt == 0) return FM_OK;
    if (cap < 1) cap = 1;
    const size_t sm = block_smem_bytes<G>(cap, 0);
    if (sm > 200 * 1024) return FM_ERR_UNSUPPORTED;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_support_fill<DIM, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
    k_support_fill<DIM, G><<<grid_blocks(s.nt, kBlock / G, 16), kBlock, sm, st>>>(
        s, offsets, cap, idx, dist, rbf_kind, rbf_a, w);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

// FM_BUILD_STAGE=0 disables the cp.async build pipeline (A/B checks)
inline bool build_stage_enabled() {
    static const int v = [] {
        const char *e = getenv("FM_BUILD_STAGE");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return v != 0;
}

// Largest fit (rows) built with 4-lane groups; FM_BUILD_G4=<rows> overrides
// (0 disables them; A/B checks)
inline int build_g4_rows() {
    static const int v = [] {
        const char *e = getenv("FM_BUILD_G4");
        return e ? atoi(e) : 24;
    }();
    return v;
}

// FM_SELECT_GROUPS=1 forces the lane-group select in 1-D/2-D (A/B checks)
inline bool select_groups_forced() {
    static const int v = [] {
        const char *e = getenv("FM_SELECT_GROUPS");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return v != 0;
}

// per-group candidate list of the select pass (at least slot_cap): 64 keeps
// 8 CTAs/SM within shared memory for the 2-D slots
constexpr int kSelectListCap = 64;

template <int DIM>
int launch_select(const SearchArgs &s, int32_t min_required, int32_t *counts, double *radii,
                  uint8_t *status, int32_t *slot_id, int32_t *slot_pos, int slot_cap,
                  int32_t *overflow, int32_t *stats, PosInfo *pos_info, double *pos_t,
                  cudaStream_t st, SelectBuckets bk = SelectBuckets{nullptr, nullptr, nullptr, 0}) {
    // 1-D/2-D: one thread per target (k_select_t); dim >= 3: 16-lane groups
    // (windows of many rows)
    constexpr int G = DIM <= 2 ? 8 : 16;
    k_stats_init<<<1, 32, 0, st>>>(stats, 8, 0, bk.pos_counts ? bk.bucket_count : nullptr,
                                   FM_NBUCKETS);
    if (s.nt == 0) return FM_OK;
    if (DIM <= 2 && slot_cap <= 2 * kThreadListCap && !select_groups_forced()) {
        // the per-thread list IS the slot: a position is slotted iff its
        // support fits slot_cap (what the size buckets and the build assume)
        const int lcap = slot_cap;
        const size_t sm = (size_t)kBlock * (lcap | 1) * sizeof(int32_t);
        if (sm > 48 * 1024)
            cudaFuncSetAttribute(k_select_t<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        const int64_t tiles = (s.nt + 31) / 32;
        const int blocks = (int)std::min<int64_t>((tiles + 3) / 4, (int64_t)kSMs * 8);
        k_select_t<DIM><<<blocks, kBlock, sm, st>>>(s, min_required, lcap, counts, radii, status,
                                                    slot_id, slot_pos, slot_cap, overflow, stats,
                                                    pos_info, pos_t, bk);
        FM_CHECK_LAUNCH();
        return FM_OK;
    }
    if (bk.pos_counts) return FM_ERR_UNSUPPORTED;  // lane-group select: not fused
    const int lcap = slot_cap > kSelectListCap ? slot_cap : kSelectListCap;
    const size_t per = ((size_t)lcap * 16 + sizeof(RowTable<G>) + 15) & ~(size_t)15;
    const size_t sm = per * (kBlock / G);
    if (sm > 200 * 1024) return FM_ERR_UNSUPPORTED;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_select<DIM, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
    k_select<DIM, G><<<grid_blocks(s.nt, kBlock / G, 16), kBlock, sm, st>>>(
        s, min_required, lcap, counts, radii, status, slot_id, slot_pos, slot_cap, overflow,
        stats, pos_info, pos_t);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

// rows needed by a fit: support + ridge rows, at least K
inline int fit_rows_needed(int max_m, int K, double lam) {
    int r = max_m + (lam > 0.0 ? K : 0);
    return r < K ? K : r;
}

template <int DIM, int DEG, int G, int ROWS, bool SOLVE, bool FROM_SLOTS>
int launch_build_rows(const SearchArgs &s, const BuildArgs &b0, cudaStream_t st) {
    constexpr int K = Monos<DIM, DEG>::K;
    BuildArgs b = b0;
    size_t sm = block_smem_bytes<G>(FROM_SLOTS ? 0 : b.cap, K);
    if (sm > 200 * 1024) return FM_ERR_UNSUPPORTED;
    const size_t staged = sm + (size_t)(kBlock / G) * stage_bytes<DIM, G, ROWS>();
    b.stage = FROM_SLOTS && b.pos_info && staged <= 75 * 1024 && build_stage_enabled();
    if (b.stage) sm = staged;
    auto kern = k_build<DIM, DEG, G, ROWS, SOLVE, FROM_SLOTS>;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    // persistent grid: the resident CTAs of every SM, grid-striding over
    // the positions (no waves of CTAs that only run the pipeline prologue,
    // e.g. when the count is read on the device and nk is an upper bound)
    static size_t occ_sm = (size_t)-1;
    static int occ = 1;
    if (occ_sm != sm) {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kBlock, sm) != cudaSuccess ||
            o < 1)
            o = 1;
        occ = o;
        occ_sm = sm;
    }
    kern<<<grid_blocks(b.nk, kBlock / G, occ), kBlock, sm, st>>>(s, b);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

// (G lanes, ROWS rows per lane) with G*ROWS >= rows needed: groups of
// FitShape::G lanes (8/16/32 by k) while ROWS <= 4, 32-lane groups beyond.
template <int DIM, int DEG, bool SOLVE, bool FROM_SLOTS>
int launch_build(const SearchArgs &s, const BuildArgs &b, int max_m, cudaStream_t st) {
    constexpr int K = Monos<DIM, DEG>::K;
    constexpr int G0 = FitShape<DIM, DEG>::G;
    if (b.nk == 0) return FM_OK;
    const int need = fit_rows_needed(max_m, K, b.fp.lam);
#define FM_BUILD(GG, R) launch_build_rows<DIM, DEG, GG, R, SOLVE, FROM_SLOTS>(s, b, st)
    // small supports of k <= 6 fits: 4-lane groups (8 targets per warp: a
    // third of the butterfly levels and half the replicated scalar work of
    // the 8-lane shape per target)
    if constexpr (G0 == 8) {
        const int g4 = build_g4_rows();
        if (need <= 8 && need <= g4) return FM_BUILD(4, 2);
        if (need <= 16 && need <= g4) return FM_BUILD(4, 4);
        if (need <= 24 && need <= g4) return FM_BUILD(4, 6);
    }
    if (need <= G0) return FM_BUILD(G0, 1);
    if (need <= 2 * G0) return FM_BUILD(G0, 2);
    if (need <= 3 * G0) return FM_BUILD(G0, 3);
    if (need <= 4 * G0) return FM_BUILD(G0, 4);
    if constexpr (G0 < 32) {
        if (need <= 128) return FM_BUILD(32, 4);
    }
    if (need <= 256) return FM_BUILD(32, 8);
#undef FM_BUILD
    if constexpr (!FROM_SLOTS) {
        // beyond 256 rows (only reached by re-gathered supports): the
        // warp-per-target fit with the rows in global scratch
        BigArgs g{};
        g.klist = b.klist;
        g.nk = b.nk;
        return launch_fit_big<DIM, DEG, SOLVE, false>(s, b, g, need, st);
    }
    return FM_ERR_UNSUPPORTED;
}

template <int DIM, int DEG>
int launch_fit_many(const fm_fit &fp, const double *targets, int64_t nt, const int64_t *sup_off,
                    const int64_t *sup_idx, const double *sup_w, int max_m, const double *src,
                    const double *src_val, double *values, double *coeffs, uint8_t *status,
                    int32_t *stats, cudaStream_t st) {
    constexpr int K = Monos<DIM, DEG>::K;
    constexpr int G0 = FitShape<DIM, DEG>::G;
    if (stats) k_stats_init<<<1, 32, 0, st>>>(stats, 2, 1);
    if (nt == 0) return FM_OK;
    const int need = fit_rows_needed(max_m, K, fp.lam);
#define FM_FITMANY(GG, R)                                                                    \
    do {                                                                                     \
        k_fit_many<DIM, DEG, GG, R><<<grid_blocks(nt, kBlock / GG, 16), kBlock, 0, st>>>(    \
            fp, targets, nt, sup_off, sup_idx, sup_w, src, src_val, values, coeffs, status,  \
            stats);                                                                          \
        FM_CHECK_LAUNCH();                                                                   \
        return FM_OK;                                                                        \
    } while (0)
    if (need <= G0) FM_FITMANY(G0, 1);
    if (need <= 2 * G0) FM_FITMANY(G0, 2);
    if (need <= 4 * G0) FM_FITMANY(G0, 4);
    if constexpr (G0 < 32) {
        if (need <= 128) FM_FITMANY(32, 4);
    }
    if (need <= 256) FM_FITMANY(32, 8);
#undef FM_FITMANY
    // beyond 256 rows: warp per target, rows in global scratch (fm_big.cuh)
    SearchArgs s{};
    s.targets = targets;
    s.nt = nt;
    BuildArgs b{};
    b.fp = fp;
    b.src_val = src_val;
    b.values = values;
    b.status = status;
    b.stats = stats;
    BigArgs g{};
    g.nk = nt;
    g.sup_off = sup_off;
    g.sup_idx = sup_idx;
    g.sup_w = sup_w;
    g.src = src;
    g.coeffs = coeffs;
    return launch_fit_big<DIM, DEG, true, true>(s, b, g, need, st);
}

// ------------------------------------------------- instantiation units
// Entry points per dimension (search) and per (dimension, degree) (fits),
// defined in fm_dN.cu / fm_dN_pP.cu so the heavy fit instantiations compile
// in parallel.  Degree 3 exists for dim <= 3 only (k <= 21).
#define FM_DECLARE_DIM(N)                                                                         \
    int dim##N##_count(const SearchArgs &, int32_t, int32_t *, double *, uint8_t *, int32_t *,   \
                       cudaStream_t);                                                             \
    int dim##N##_fill(const SearchArgs &, const int64_t *, int, int64_t *, double *, int,        \
                      double, double *, cudaStream_t);                                            \
    int dim##N##_select(const SearchArgs &, int32_t, int32_t *, double *, uint8_t *, int32_t *,  \
                        int32_t *, int, int32_t *, int32_t *, PosInfo *, double *,            \
                        cudaStream_t, const SelectBuckets &);
#define FM_DECLARE_DEG(N, P)                                                                      \
    int dim##N##_deg##P##_build(bool, bool, const SearchArgs &, const BuildArgs &, int,          \
                                cudaStream_t);                                                    \
    int dim##N##_deg##P##_fit_many(const fm_fit &, const double *, int64_t, const int64_t *,     \
                                   const int64_t *, const double *, int, const double *,         \
                                   const double *, double *, double *, uint8_t *, int32_t *,     \
                                   cudaStream_t);
FM_DECLARE_DIM(1)
FM_DECLARE_DIM(2)
FM_DECLARE_DIM(3)
FM_DECLARE_DIM(4)
FM_DECLARE_DIM(5)
FM_DECLARE_DEG(1, 0) FM_DECLARE_DEG(1, 1) FM_DECLARE_DEG(1, 2) FM_DECLARE_DEG(1, 3)
FM_DECLARE_DEG(2, 0) FM_DECLARE_DEG(2, 1) FM_DECLARE_DEG(2, 2) FM_DECLARE_DEG(2, 3)
FM_DECLARE_DEG(3, 0) FM_DECLARE_DEG(3, 1) FM_DECLARE_DEG(3, 2) FM_DECLARE_DEG(3, 3)
FM_DECLARE_DEG(4, 0) FM_DECLARE_DEG(4, 1) FM_DECLARE_DEG(4, 2)
FM_DECLARE_DEG(5, 0) FM_DECLARE_DEG(5, 1) FM_DECLARE_DEG(5, 2)

#define FM_DEFINE_DIM(N)                                                                           \
    int dim##N##_count(const SearchArgs &s, int32_t need, int32_t *c, double *r, uint8_t *st,     \
                       int32_t *stats, cudaStream_t stream) {                                      \
        return launch_count<N>(s, need, c, r, st, stats, stream);                                  \
    }                                                                                              \
    int dim##N##_fill(const SearchArgs &s, const int64_t *o, int cap, int64_t *idx, double *d,    \
                      int kind, double a, double *w, cudaStream_t stream) {                        \
        return launch_fill<N>(s, o, cap, idx, d, kind, a, w, stream);                              \
    }                                                                                              \
    int dim##N##_select(const SearchArgs &s, int32_t need, int32_t *c, double *r, uint8_t *st,    \
                        int32_t *sid, int32_t *spos, int scap, int32_t *ovf, int32_t *stats,       \
                        PosInfo *pinfo, double *pt,                                                \
                        cudaStream_t stream, const SelectBuckets &bk) {                            \
        return launch_select<N>(s, need, c, r, st, sid, spos, scap, ovf, stats, pinfo, pt,       \
                                stream, bk);       \
    }

#define FM_DEFINE_DEG(N, P)                                                                        \
    int dim##N##_deg##P##_build(bool solve, bool slots, const SearchArgs &s, const BuildArgs &b,  \
                                int max_m, cudaStream_t stream) {                                  \
        if (slots)                                                                                 \
            return solve ? launch_build<N, P, true, true>(s, b, max_m, stream)                     \
                         : launch_build<N, P, false, true>(s, b, max_m, stream);                   \
        return solve ? launch_build<N, P, true, false>(s, b, max_m, stream)                        \
                     : launch_build<N, P, false, false>(s, b, max_m, stream);                      \
    }                                                                                              \
    int dim##N##_deg##P##_fit_many(const fm_fit &fp, const double *t, int64_t nt,                 \
                                   const int64_t *so, const int64_t *si, const double *sw, int mm, \
                                   const double *src, const double *sv, double *vals, double *co,  \
                                   uint8_t *st, int32_t *stats, cudaStream_t stream) {             \
        return launch_fit_many<N, P>(fp, t, nt, so, si, sw, mm, src, sv, vals, co, st, stats,      \
                                     stream);                                                      \
    }

}  // namespace fm
