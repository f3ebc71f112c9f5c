// fm_search.cuh -- warp-cooperative radius search over the cell-sorted sources.
//
// Semantics (the reference's _gather_radius, _ext.pyx:172-200): the support
// of target t at radius r is { j : fl(sqrt(sum_a fl(fl(p_ja - t_a)^2))) < r },
// with the sum taken left to right and no FMA contraction.  The reference
// visits every source binned in the cell box [cell(t - r), cell(t + r)]; here
// the window is cut into "rows" (all axes but axis 0 fixed) and each row is
// clipped to the chord of the sphere, which visits fewer candidates.  Both
// windows are supersets of the exact set (the clipping is conservative by a
// relative 1e-9 plus an ulp-level absolute term), and the
// distance test is bitwise the reference's, so the kept sets are identical.
//
// Sources are stored in cell order (fm_grid_build), so every row of the
// window is ONE contiguous range of sorted_pts: a group of G lanes
// flattens the ranges of up to G rows with a prefix sum and then reads the
// candidates with consecutive lanes on consecutive points (coalesced).
#pragma once

#include "fm_common.cuh"

namespace fm {

constexpr double kSlackRel = 1e-9;

// per-group shared scratch for the row table
template <int G>
struct RowTable {
    int32_t start[G];
    int32_t pref[G];
};

// Enumerate the candidates of the window of (t, r) for the calling group.
// Every lane of the WARP must call this (collectives inside); `active` false
// makes the group's window empty.  `visit(pos, valid)` is called the same
// (warp-uniform) number of times on every lane; pos is an index into the
// cell-sorted arrays when valid.
template <int DIM, int G, class Visit>
__device__ __forceinline__ void for_each_candidate(const GridDev &g,
                                                   const int32_t *__restrict__ cell_start,
                                                   const double *t, double r, bool active,
                                                   int glane, RowTable<G> &rt, Visit &&visit) {
    const double rs = r * (1.0 + kSlackRel);
    int64_t clo[kMaxDim], chi[kMaxDim], stride[kMaxDim];
    int64_t nrows = active ? 1 : 0;
    int64_t st = 1;
#pragma unroll
    for (int a = 0; a < DIM; a++) {
        clo[a] = cell_of(t[a] - rs, g.lo[a], g.inv_d[a], g.n[a]);
        chi[a] = cell_of(t[a] + rs, g.lo[a], g.inv_d[a], g.n[a]);
        stride[a] = st;
        st *= g.n[a];
        if (a > 0) nrows *= (chi[a] - clo[a] + 1);
    }
    const int nchunks = (int)((nrows + G - 1) / G);
    const int nchunks_w = warp_max_int(nchunks);
    const double rs2 = rs * rs;
    const double eps_r2 = 8.0 * 2.220446049250313e-16 * rs2;
    for (int ch = 0; ch < nchunks_w; ch++) {
        const int64_t row = (int64_t)ch * G + glane;
        int32_t start = 0, len = 0;
        if (row < nrows) {
            // unravel the row index over axes 1..DIM-1 and measure the squared
            // distance from t to the row's cell box along those axes
            int64_t rem = row, base = 0;
            double off2 = 0.0;
#pragma unroll
            for (int a = 1; a < DIM; a++) {
                const int64_t span = chi[a] - clo[a] + 1;
                const int64_t ia = clo[a] + rem % span;
                rem /= span;
                base += ia * stride[a];
                const double d = g.d[a];
                const double blo = ia == 0 ? -INFINITY : g.lo[a] + (double)ia * d;
                const double bhi = ia == g.n[a] - 1 ? INFINITY : g.lo[a] + (double)(ia + 1) * d;
                const double slack = 8.0 * 2.220446049250313e-16 *
                                         (fabs(g.lo[a]) + fabs(t[a]) + (double)(ia + 1) * d) +
                                     kSlackRel * d;
                double gap = fmax(blo - t[a], t[a] - bhi) - slack;
                gap = fmax(gap, 0.0);
                off2 += gap * gap;
            }
            const double hw2 = rs2 - off2;
            if (hw2 >= -eps_r2) {
                const double hw = sqrt(fmax(hw2, 0.0) + eps_r2) * (1.0 + kSlackRel);
                const int64_t x0 = cell_of(t[0] - hw, g.lo[0], g.inv_d[0], g.n[0]);
                const int64_t x1 = cell_of(t[0] + hw, g.lo[0], g.inv_d[0], g.n[0]);
                start = cell_start[base + x0];
                len = cell_start[base + x1 + 1] - start;
            }
        }
        const int incl = group_scan_incl<G>(len, glane);
        const int total = __shfl_sync(FM_FULL_MASK, incl, (threadIdx.x & 31 & ~(G - 1)) + G - 1);
        rt.start[glane] = start;
        rt.pref[glane] = incl - len;
        __syncwarp();
        const int iters = warp_max_int((total + G - 1) / G);
        int cursor = 0;
        for (int it = 0; it < iters; it++) {
            const int c = it * G + glane;
            const bool valid = c < total;
            int pos = 0;
            if (valid) {
                while (cursor + 1 < G && c >= rt.pref[cursor + 1]) cursor++;
                pos = rt.start[cursor] + (c - rt.pref[cursor]);
            }
            visit(pos, valid);
        }
        __syncwarp();
    }
}

template <int DIM>
__device__ __forceinline__ void load_point(const double *__restrict__ pts, int64_t i, double *p) {
    if (DIM == 2) {
        const double2 v = __ldg(reinterpret_cast<const double2 *>(pts) + i);
        p[0] = v.x;
        p[1] = v.y;
    } else {
#pragma unroll
        for (int a = 0; a < DIM; a++) p[a] = __ldg(pts + i * DIM + a);
    }
}

// number of sources strictly inside radius r (group-uniform result)
template <int DIM, int G>
__device__ __forceinline__ int count_within(const GridDev &g, const int32_t *__restrict__ cell_start,
                                            const double *__restrict__ sorted_pts, const double *t,
                                            double r, bool active, int lane, int glane,
                                            RowTable<G> &rt) {
    int cnt = 0;
    for_each_candidate<DIM, G>(g, cell_start, t, r, active, glane, rt, [&](int pos, bool valid) {
        bool keep = false;
        if (valid) {
            double p[DIM];
            load_point<DIM>(sorted_pts, pos, p);
            keep = __dsqrt_rn(dist2_rn<DIM>(p, t)) < r;
        }
        cnt += __popc(group_bits<G>(__ballot_sync(FM_FULL_MASK, keep), lane));
    });
    return cnt;
}

// Reference radius loop of adaptive_radius_supports (_ext.pyx:258-271):
// r = r0; until count(r) >= min_pts: if r >= r_max: status 1; r = min(r*growth, r_max).
// Returns the count at the final radius; radius/status out.
template <int DIM, int G>
__device__ __forceinline__ int adaptive_radius(const GridDev &g, const int32_t *__restrict__ cell_start,
                                               const double *__restrict__ sorted_pts, const double *t,
                                               const fm_select &sel, bool active, int lane, int glane,
                                               RowTable<G> &rt, double &r_out, uint8_t &status) {
    double r = sel.r0;
    bool done = !active;
    int m = 0;
    status = 0;
    while (__any_sync(FM_FULL_MASK, !done)) {
        const int c = count_within<DIM, G>(g, cell_start, sorted_pts, t, r, !done, lane, glane, rt);
        if (!done) {
            m = c;
            if (c >= sel.min_pts) {
                done = true;
            } else if (r >= sel.r_max) {
                status = 1;
                done = true;
            } else {
                r = r * sel.growth;
                if (r > sel.r_max) r = sel.r_max;
            }
        }
    }
    r_out = r;
    return m;
}

// Collect the (id, pos) of the kept candidates into per-group shared buffers
// (discovery order), then rank-sort them by source id into sid/spos.
// Returns the kept count; entries beyond `cap` are dropped (count still
// exact) -- callers size cap >= max count.
template <int DIM, int G>
__device__ __forceinline__ int collect_sorted(const GridDev &g, const int32_t *__restrict__ cell_start,
                                              const double *__restrict__ sorted_pts,
                                              const int32_t *__restrict__ sorted_ids, const double *t,
                                              double r, bool active, int lane, int glane,
                                              RowTable<G> &rt, int32_t *s_id, int32_t *s_pos,
                                              int32_t *s_sid, int32_t *s_spos, int cap) {
    int m = 0;
    const unsigned lt_mask = (1u << glane) - 1u;
    for_each_candidate<DIM, G>(g, cell_start, t, r, active, glane, rt, [&](int pos, bool valid) {
        bool keep = false;
        if (valid) {
            double p[DIM];
            load_point<DIM>(sorted_pts, pos, p);
            keep = __dsqrt_rn(dist2_rn<DIM>(p, t)) < r;
        }
        const unsigned bits = group_bits<G>(__ballot_sync(FM_FULL_MASK, keep), lane);
        if (keep) {
            const int o = m + __popc(bits & lt_mask);
            if (o < cap) {
                s_id[o] = __ldg(sorted_ids + pos);
                s_pos[o] = pos;
            }
        }
        m += __popc(bits);
    });
    __syncwarp();
    const int mm = m < cap ? m : cap;
    for (int e = glane; e < mm; e += G) {
        const int32_t id = s_id[e];
        int rank = 0;
        for (int f = 0; f < mm; f++) rank += s_id[f] < id;
        s_sid[rank] = id;
        s_spos[rank] = s_pos[e];
    }
    __syncwarp();
    return m;
}

}  // namespace fm
