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

// Window of (t, r) for the calling group, enumerated as row chunks of up to
// G rows each, flattened to candidate indices with a group prefix sum.
//   Window<DIM,G> w(g, t, r, active);
//   for (int ch = 0; ch < w.nchunks_w; ch++) {
//       const int iters = w.chunk(g, cell_start, t, ch, glane, rt);
//       for (int it = 0; it < iters; it++) { bool v; int pos = w.pos(it, glane, rt, v); ... }
//       __syncwarp();
//   }
// Every lane of the WARP must run the loops (collectives inside; the trip
// counts are warp-uniform); `active` false makes the group's window empty.
template <int DIM, int G>
struct Window {
    int64_t clo[kMaxDim], chi[kMaxDim], stride[kMaxDim];
    int64_t nrows;
    int nchunks_w;
    double rs2, eps_r2;
    int total, cursor;

    __device__ __forceinline__ Window(const GridDev &g, const double *t, double r, bool active) {
        const double rs = r * (1.0 + kSlackRel);
        nrows = active ? 1 : 0;
        int64_t st = 1;
#pragma unroll
        for (int a = 0; a < DIM; a++) {
            clo[a] = cell_of(t[a] - rs, g.lo[a], g.inv_d[a], g.n[a]);
            chi[a] = cell_of(t[a] + rs, g.lo[a], g.inv_d[a], g.n[a]);
            stride[a] = st;
            st *= g.n[a];
            if (a > 0) nrows *= (chi[a] - clo[a] + 1);
        }
        nchunks_w = warp_max_int((int)((nrows + G - 1) / G));
        rs2 = rs * rs;
        eps_r2 = 8.0 * 2.220446049250313e-16 * rs2;
    }

    // Row table of chunk ch (rows ch*G .. ch*G+G-1); returns the warp-uniform
    // number of candidate iterations.
    __device__ __forceinline__ int chunk(const GridDev &g, const int32_t *__restrict__ cell_start,
                                         const double *t, int ch, int glane, RowTable<G> &rt) {
        const int64_t row = (int64_t)ch * G + glane;
        int32_t start = 0, len = 0;
        if (row < nrows) {
            // unravel the row index over axes 1..DIM-1 and measure the squared
            // distance from t to the row's cell box along those axes
            int32_t rem = (int32_t)row;  // window rows fit in 32 bits
            int64_t base = 0;
            double off2 = 0.0;
#pragma unroll
            for (int a = 1; a < DIM; a++) {
                int64_t ia;
                if (a == DIM - 1) {  // last axis: no division needed
                    ia = clo[a] + rem;
                } else {
                    const int32_t span = (int32_t)(chi[a] - clo[a] + 1);
                    ia = clo[a] + rem % span;
                    rem /= span;
                }
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
        total = __shfl_sync(FM_FULL_MASK, incl, (threadIdx.x & 31 & ~(G - 1)) + G - 1);
        rt.start[glane] = start;
        rt.pref[glane] = incl - len;
        __syncwarp();
        cursor = 0;
        return warp_max_int((total + G - 1) / G);
    }

    // Candidate of iteration it for this lane (index into the cell-sorted arrays).
    __device__ __forceinline__ int pos(int it, int glane, const RowTable<G> &rt, bool &valid) {
        const int c = it * G + glane;
        valid = c < total;
        if (!valid) return 0;
        while (cursor + 1 < G && c >= rt.pref[cursor + 1]) cursor++;
        return rt.start[cursor] + (c - rt.pref[cursor]);
    }
};

// Lambda form of the enumeration for the less hot paths.
template <int DIM, int G, class Visit>
__device__ __forceinline__ void for_each_candidate(const GridDev &g,
                                                   const int32_t *__restrict__ cell_start,
                                                   const double *t, double r, bool active,
                                                   int glane, RowTable<G> &rt, Visit &&visit) {
    Window<DIM, G> w(g, t, r, active);
    for (int ch = 0; ch < w.nchunks_w; ch++) {
        const int iters = w.chunk(g, cell_start, t, ch, glane, rt);
        for (int it = 0; it < iters; it++) {
            bool valid;
            const int pos = w.pos(it, glane, rt, valid);
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

// ======================================================================
// Selection with support lists (count pass that also emits the supports)
// ======================================================================
constexpr int kMaxGuess = 8;  // radii evaluated by the first multi-radius scan: r_0..r_8

// Per-group list buffer in shared memory (discovery order): source id,
// sorted position and distance of each kept candidate.
struct ListBuf {
    int32_t *id;
    int32_t *pos;
    double *d;
    int cap;
};

// One window scan at radius radii[nr-1] that counts #{d < radii[j]} for all
// j < nr at once (the reference's count at each radius of its growth
// sequence, _ext.pyx:258-271) and appends every candidate with
// d < radii[nr-1] to the group's list (entries beyond cap are counted, not
// stored).  Warp-collective.
// Smallest double T with fl(sqrt(T)) >= r (r > 0).  fl o sqrt is monotone,
// so the reference's test fl(sqrt(d2)) < r (_ext.pyx:194-195) is exactly
// d2 < T: the scans compare squared distances and never take a square root.
__device__ __forceinline__ double sqrt_threshold(double r) {
    double x = mul_rn(r, r);
    if (!(x < INFINITY) || !(x > 0.0)) return x;
    if (__dsqrt_rn(x) < r) {
        do {  // x passes: step up to the first failing double
            x = __longlong_as_double(__double_as_longlong(x) + 1);
        } while (__dsqrt_rn(x) < r);
        return x;
    }
    for (int it = 0; it < 64; it++) {  // x fails: step down while the predecessor fails too
        const double xp = __longlong_as_double(__double_as_longlong(x) - 1);
        if (xp > 0.0 && __dsqrt_rn(xp) >= r) x = xp;
        else break;
    }
    return x;
}

// One window scan at radius r (threshold thr = sqrt_threshold(r)): returns
// #{d < r} and appends every candidate with d < r (id, grid position, d^2)
// to the group's list (entries beyond cap are counted, not stored).
// Warp-collective.
template <int DIM, int G>
__device__ __forceinline__ int scan_list(const GridDev &g, const int32_t *__restrict__ cell_start,
                                         const double *__restrict__ sorted_pts,
                                         const int32_t *__restrict__ sorted_ids, const double *t,
                                         double r, double thr, bool active, int lane, int glane,
                                         RowTable<G> &rt, ListBuf &lb, int &nlist) {
    const unsigned lt_mask = (1u << glane) - 1u;
    int cnt = 0;
    Window<DIM, G> w(g, t, r, active);
    for (int ch = 0; ch < w.nchunks_w; ch++) {
        const int iters = w.chunk(g, cell_start, t, ch, glane, rt);
        for (int it = 0; it < iters; it++) {
            bool valid;
            const int pos = w.pos(it, glane, rt, valid);
            double d2 = INFINITY;
            int32_t id = 0;
            if (valid) {
                double p[DIM];
                id = __ldg(sorted_ids + pos);  // issued with the point load
                load_point<DIM>(sorted_pts, pos, p);
                d2 = dist2_rn<DIM>(p, t);
            }
            const bool keep = d2 < thr;
            const unsigned bits = group_bits<G>(__ballot_sync(FM_FULL_MASK, keep), lane);
            if (keep) {
                const int o = nlist + __popc(bits & lt_mask);
                if (o < lb.cap) {
                    lb.id[o] = id;
                    lb.pos[o] = pos;
                    lb.d[o] = d2;
                }
            }
            nlist += __popc(bits);
            cnt += __popc(bits);
        }
        __syncwarp();
    }
    return cnt;
}

// The reference's radius sequence r_0 = r0, r_{j+1} = min(r_j * growth, r_max)
// (_ext.pyx:258-270) -- the same for every target -- with the exact
// thresholds T(r_j), tabulated once per CTA.  Fixed radius: entry 0 = r_c.
constexpr int kRadTab = 64;
struct RadiusTable {
    double r[kRadTab];
    double thr[kRadTab];
};

__device__ __forceinline__ void fill_radius_table(RadiusTable &tab, const fm_select &sel) {
    const int j = threadIdx.x;
    if (j < kRadTab) {
        double r;
        if (sel.adaptive) {
            r = sel.r0;
            for (int i = 0; i < j && r < sel.r_max; i++) {
                r = r * sel.growth;
                if (r > sel.r_max) r = sel.r_max;
            }
        } else {
            r = sel.r_c;
        }
        tab.r[j] = r;
        tab.thr[j] = sqrt_threshold(r);
    }
    __syncthreads();
}

// radius j of the sequence (beyond the table: continued on the fly)
__device__ __forceinline__ void seq_radius(const RadiusTable &tab, const fm_select &sel, int j,
                                           double &r, double &thr) {
    if (j < kRadTab) {
        r = tab.r[j];
        thr = tab.thr[j];
        return;
    }
    r = tab.r[kRadTab - 1];
    for (int i = kRadTab - 1; i < j && r < sel.r_max; i++) {
        r = r * sel.growth;
        if (r > sel.r_max) r = sel.r_max;
    }
    thr = sqrt_threshold(r);
}

// Density guess of the number of growth steps (2-D): sources in the 3x3
// cell block around the target -> radius holding min_pts at that density.
// Only a starting point: the result is exact whatever the guess.
template <int DIM, int G>
__device__ __forceinline__ int guess_steps(const GridDev &g, const int32_t *__restrict__ cell_start,
                                           const double *t, const fm_select &sel, bool active,
                                           int glane) {
    if (DIM != 2) return 0;
    const int64_t nx = g.n[0], ny = g.n[1];
    const int64_t cx = cell_of(t[0], g.lo[0], g.inv_d[0], nx);
    const int64_t cy = cell_of(t[1], g.lo[1], g.inv_d[1], ny);
    const int64_t x0 = cx > 0 ? cx - 1 : 0, x1 = cx + 1 < nx ? cx + 1 : nx - 1;
    const int64_t y0 = cy > 0 ? cy - 1 : 0, y1 = cy + 1 < ny ? cy + 1 : ny - 1;
    int n = 0;
    if (active && glane <= y1 - y0) {
        const int64_t row = (y0 + glane) * nx;
        n = cell_start[row + x1 + 1] - cell_start[row + x0];
    }
    n = group_sum_int<G>(n);
    if (!active) return 0;
    const double area = (double)((x1 - x0 + 1) * (y1 - y0 + 1)) * g.d[0] * g.d[1];
    // smallest k with r0 * growth^k >= r_est, r_est^2 = min_pts / (pi rho)
    const float r2_est = (float)((double)sel.min_pts * area /
                                 (3.14159265f * (n > 0 ? (float)n : 0.5f)));
    float r = (float)sel.r0, g2 = (float)sel.growth;
    int k = 0;
    while (k < kMaxGuess && r * r < r2_est) {
        r *= g2;
        k++;
    }
    return k;
}

// Number of list entries with squared distance below thr (group-cooperative).
template <int G>
__device__ __forceinline__ int count_list(const ListBuf &lb, int n, double thr, int lane,
                                          int glane) {
    const int iters = warp_max_int((n + G - 1) / G);
    int c = 0;
    for (int it = 0; it < iters; it++) {
        const int e = it * G + glane;
        const bool in = e < n && lb.d[e] < thr;
        c += __popc(group_bits<G>(__ballot_sync(FM_FULL_MASK, in), lane));
    }
    return c;
}

// Final support of one target for fixed or adaptive selection, exactly the
// reference's (fixed: d < r_c; adaptive: the first radius of the sequence
// r0, min(r*growth, r_max), ... holding >= min_pts sources, status 1 when
// r_max is reached short).  Returns the count m; when `listed` is true the
// group's buffer holds all m supports (discovery order), otherwise m > cap.
//
// Adaptive: one window scan at the density-guessed step r_kg collects every
// candidate with d < r_kg (and d^2).  If it holds min_pts, the counts at the
// smaller radii r_0..r_kg-1 of the same sequence are taken from that list and
// the first radius reaching min_pts wins; otherwise the sequence continues
// one radius (one scan) at a time, exactly like _ext.pyx:258-271.
// Warp-collective.
template <int DIM, int G>
__device__ __forceinline__ int select_target(const GridDev &g, const int32_t *__restrict__ cell_start,
                                             const double *__restrict__ sorted_pts,
                                             const int32_t *__restrict__ sorted_ids,
                                             const double *t, const fm_select &sel,
                                             const RadiusTable &tab, bool active, int lane,
                                             int glane, RowTable<G> &rt, ListBuf &lb,
                                             double &r_out, uint8_t &status, bool &listed) {
    // first scan at step kg of the sequence (stopping at r_max)
    int kg = 0;
    if (sel.adaptive) {
        kg = guess_steps<DIM, G>(g, cell_start, t, sel, active, glane);
        int j = 0;
        while (j < kg && tab.r[j < kRadTab ? j : kRadTab - 1] < sel.r_max && j + 1 < kRadTab) j++;
        kg = j;
    }
    double rscan, thr_scan;
    seq_radius(tab, sel, kg, rscan, thr_scan);
    int nlist = 0;
    int m = scan_list<DIM, G>(g, cell_start, sorted_pts, sorted_ids, t, rscan, thr_scan, active,
                              lane, glane, rt, lb, nlist);
    int jf = kg;  // index of the final radius in the sequence
    double rf = rscan;
    status = 0;
    bool done = !active || !sel.adaptive;
    bool slow = false;  // guess too high and the list overflowed: restart at r0
    if (!done) {
        if (m >= sel.min_pts) {
            done = true;
            slow = kg > 0 && nlist > lb.cap;
        } else if (rf >= sel.r_max) {
            status = 1;
            done = true;
        }
    }
    // smaller radii of the sequence, counted on the list (kg is small)
    const bool recount = active && sel.adaptive && !slow && m >= sel.min_pts && kg > 0;
    const int kg_w = warp_max_int(recount ? kg : 0);
    {
        bool found = !recount;
        for (int j = 0; j < kg_w; j++) {
            const bool mine = !found && j < kg;
            const double thr = mine ? tab.thr[j] : 0.0;
            const int c = count_list<G>(lb, mine ? nlist : 0, thr, lane, glane);
            if (mine && c >= sel.min_pts) {
                found = true;
                m = c;
                jf = j;
                rf = tab.r[j];
            }
        }
    }
    if (slow) {  // rare: recount from r0 one scan per radius
        jf = -1;
        done = false;
    }
    // continue the sequence one radius at a time (_ext.pyx:259-270)
    bool fresh = false;  // list rebuilt at exactly rf
    while (__any_sync(FM_FULL_MASK, !done)) {
        const bool go = !done;
        double r1 = 0.0, thr1 = 0.0;
        if (go) {
            jf++;
            seq_radius(tab, sel, jf, r1, thr1);
            rf = r1;
            nlist = 0;
        }
        int nl = nlist;
        const int c = scan_list<DIM, G>(g, cell_start, sorted_pts, sorted_ids, t, r1, thr1, go,
                                        lane, glane, rt, lb, nl);
        if (go) {
            nlist = nl;
            m = c;
            fresh = true;
            if (m >= sel.min_pts) {
                done = true;
            } else if (rf >= sel.r_max) {
                status = 1;
                done = true;
            }
        }
    }
    // keep only d < rf when the list came from the wider first scan; rescan
    // when that scan overflowed the buffer but the final support fits
    const bool wide = active && !fresh && jf < kg;
    const bool rescan = wide && nlist > lb.cap && m <= lb.cap;
    double rthr = 0.0;
    if (wide) {
        double rr;
        seq_radius(tab, sel, jf, rr, rthr);
    }
    if (__any_sync(FM_FULL_MASK, rescan)) {
        int nl = 0;
        scan_list<DIM, G>(g, cell_start, sorted_pts, sorted_ids, t, rescan ? rf : 0.0,
                          rescan ? rthr : 0.0, rescan, lane, glane, rt, lb, nl);
        if (rescan) nlist = nl;
    }
    const bool filter = wide && !rescan && nlist <= lb.cap;
    const int nf = filter ? nlist : 0;
    const int iters = warp_max_int((nf + G - 1) / G);
    int kept = 0;
    const unsigned lt_mask = (1u << glane) - 1u;
    for (int it = 0; it < iters; it++) {
        const int e = it * G + glane;
        int32_t id = 0, pos = 0;
        double d = 0.0;  // squared distance
        const bool in = e < nf;
        if (in) {
            id = lb.id[e];
            pos = lb.pos[e];
            d = lb.d[e];
        }
        const bool keep = in && d < rthr;
        const unsigned bits = group_bits<G>(__ballot_sync(FM_FULL_MASK, keep), lane);
        if (keep) {
            const int o = kept + __popc(bits & lt_mask);
            lb.id[o] = id;
            lb.pos[o] = pos;
            lb.d[o] = d;
        }
        kept += __popc(bits);
    }
    __syncwarp();
    r_out = rf;
    listed = active && m <= lb.cap;
    return m;
}

// ======================================================================
// Thread-per-target selection (1-D / 2-D)
// ======================================================================
// One thread owns one target and walks its window rows sequentially; the
// kept candidates go to a per-thread list in shared memory (source grid
// position + "level", the index of the first radius of the sequence whose
// threshold the candidate passes).  Compared with the lane-group scan this
// removes the per-candidate ballots, prefix sums and row-table cursor walks
// (the group select issued ~370 warp instructions per target on C2).
// Exactness is unchanged: the same conservative row clipping as Window, the
// same d^2 < T(r) test against the same thresholds.

// Per-thread list in shared memory: entry e of thread i at i*stride + e
// (stride odd: appends of a warp spread over the banks; a cooperative read
// of one thread's list is contiguous).  An entry is the candidate's source
// grid position (< 2^30) with a 2-bit code in bits 30-31: the number of the
// two lower thresholds of the scan (T[j-2], T[j-1]) that its d^2 reaches.
struct ThreadList {
    int32_t *e;
    int cap;
};
constexpr int kCodeShift = 30;
constexpr int32_t kPosMask = (1 << kCodeShift) - 1;

// One window scan of target t at radius r with thresholds thr_hi = T(r) and
// two lower ones thr_mid <= thr_hi, thr_lo <= thr_mid (0: unused): appends
// every candidate with d^2 < thr_hi (entries beyond cap are counted, not
// stored).  Returns the kept count; c_mid / c_lo receive #{d^2 < thr_mid},
// #{d^2 < thr_lo}.
template <int DIM>
__device__ __forceinline__ int scan_thread(const GridDev &g, const int32_t *__restrict__ cell_start,
                                           const double *__restrict__ sorted_pts, const double *t,
                                           double r, double thr_hi, double thr_mid, double thr_lo,
                                           ThreadList &L, int &c_mid, int &c_lo) {
    const double rs = r * (1.0 + kSlackRel);
    const double rs2 = rs * rs;
    const double eps_r2 = 8.0 * 2.220446049250313e-16 * rs2;
    int32_t clo[kMaxDim], span[kMaxDim];
    int64_t stride[kMaxDim];
    int32_t nrows = 1;
    int64_t st = 1;
#pragma unroll
    for (int a = 0; a < DIM; a++) {
        clo[a] = (int32_t)cell_of(t[a] - rs, g.lo[a], g.inv_d[a], g.n[a]);
        span[a] = (int32_t)cell_of(t[a] + rs, g.lo[a], g.inv_d[a], g.n[a]) - clo[a] + 1;
        stride[a] = st;
        st *= g.n[a];
        if (a > 0) nrows *= span[a];
    }
    int n = 0, nm = 0, nl = 0;
    auto visit = [&](int32_t p, double d2) {
        if (d2 < thr_hi) {
            const int code = (d2 >= thr_mid ? 1 : 0) + (d2 >= thr_lo ? 1 : 0);
            nm += d2 < thr_mid;
            nl += d2 < thr_lo;
            if (n < L.cap) {
                FM_DCHECK(p >= 0 && p <= kPosMask);
                L.e[n] = p | (code << kCodeShift);
            }
            n++;
        }
    };
    // the source range [q0, q1) of window row `row` (empty when the row
    // misses the sphere); the row's cell_start loads are only issued here
    auto row_span = [&](int32_t row, int32_t &q0, int32_t &q1) {
        int32_t rem = row;
        int64_t base = 0;
        double off2 = 0.0;
#pragma unroll
        for (int a = 1; a < DIM; a++) {
            int64_t ia;
            if (a == DIM - 1) {
                ia = clo[a] + rem;
            } else {
                ia = clo[a] + rem % span[a];
                rem /= span[a];
            }
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
        if (!(hw2 >= -eps_r2)) {
            q0 = q1 = 0;
            return;
        }
        const double hw = sqrt(fmax(hw2, 0.0) + eps_r2) * (1.0 + kSlackRel);
        const int64_t x0 = cell_of(t[0] - hw, g.lo[0], g.inv_d[0], g.n[0]);
        const int64_t x1 = cell_of(t[0] + hw, g.lo[0], g.inv_d[0], g.n[0]);
        FM_DCHECK(x0 >= 0 && x1 < g.n[0] && base >= 0 && base + x1 + 1 <= st);
        q0 = __ldg(cell_start + base + x0);
        q1 = __ldg(cell_start + base + x1 + 1);
    };
    // one row ahead: row r+1's cell_start loads are in flight while row r's
    // points are scanned (C2 select 0.422 -> 0.412 ms)
    int32_t n0, n1;
    row_span(0, n0, n1);
    for (int32_t row = 0; row < nrows; row++) {
        const int32_t p0 = n0, p1 = n1;
        if (row + 1 < nrows) row_span(row + 1, n0, n1);
        FM_DCHECK(0 <= p0 && p0 <= p1 && p1 <= __ldg(cell_start + st));
        int32_t p = p0;
        for (; p + 1 < p1; p += 2) {  // two point loads in flight
            double pa[DIM], pb[DIM];
            load_point<DIM>(sorted_pts, p, pa);
            load_point<DIM>(sorted_pts, p + 1, pb);
            visit(p, dist2_rn<DIM>(pa, t));
            visit(p + 1, dist2_rn<DIM>(pb, t));
        }
        if (p < p1) {
            double pa[DIM];
            load_point<DIM>(sorted_pts, p, pa);
            visit(p, dist2_rn<DIM>(pa, t));
        }
    }
    c_mid = nm;
    c_lo = nl;
    return n;
}

// Density guess of the growth step for one thread (2-D; see guess_steps).
template <int DIM>
__device__ __forceinline__ int guess_steps_thread(const GridDev &g,
                                                  const int32_t *__restrict__ cell_start,
                                                  const double *t, const fm_select &sel) {
    if (DIM != 2) return 0;
    const int64_t nx = g.n[0], ny = g.n[1];
    const int64_t cx = cell_of(t[0], g.lo[0], g.inv_d[0], nx);
    const int64_t cy = cell_of(t[1], g.lo[1], g.inv_d[1], ny);
    const int64_t x0 = cx > 0 ? cx - 1 : 0, x1 = cx + 1 < nx ? cx + 1 : nx - 1;
    const int64_t y0 = cy > 0 ? cy - 1 : 0, y1 = cy + 1 < ny ? cy + 1 : ny - 1;
    int n = 0;
    for (int64_t y = y0; y <= y1; y++)
        n += __ldg(cell_start + y * nx + x1 + 1) - __ldg(cell_start + y * nx + x0);
    const double area = (double)((x1 - x0 + 1) * (y1 - y0 + 1)) * g.d[0] * g.d[1];
    const float r2_est = (float)((double)sel.min_pts * area /
                                 (3.14159265f * (n > 0 ? (float)n : 0.5f)));
    float r = (float)sel.r0, g2 = (float)sel.growth;
    int k = 0;
    while (k < kMaxGuess && r * r < r2_est) {
        r *= g2;
        k++;
    }
    return k;
}

// Final support of one target (thread version of select_target): returns m;
// on return the list holds exactly the m supports (discovery order, code
// bits cleared) when `listed`, otherwise m > L.cap.
//
// Adaptive: ONE scan at the density-guessed step kg (exact for 82% of the C2
// targets, one too high for 14%) counts the sequence's radii kg-2, kg-1, kg at
// once; the first of them holding min_pts is the reference's radius unless
// the count at kg-2 already suffices (then: restart at r0) or the count at kg
// does not (then: continue the sequence one scan per radius, _ext.pyx:258-271).
template <int DIM>
__device__ __forceinline__ int select_thread(const GridDev &g, const int32_t *__restrict__ cell_start,
                                             const double *__restrict__ sorted_pts, const double *t,
                                             const fm_select &sel, const RadiusTable &tab,
                                             ThreadList &L, double &r_out, uint8_t &status,
                                             bool &listed) {
    status = 0;
    int kg = 0;
    if (sel.adaptive) {
        kg = guess_steps_thread<DIM>(g, cell_start, t, sel);
        int j = 0;
        while (j < kg && tab.r[j] < sel.r_max && j + 1 < kRadTab) j++;
        kg = j;
    }
    const double t_mid = kg >= 1 ? tab.thr[kg - 1] : 0.0;
    const double t_lo = kg >= 2 ? tab.thr[kg - 2] : 0.0;
    int c_mid, c_lo;
    int n = scan_thread<DIM>(g, cell_start, sorted_pts, t, tab.r[kg], tab.thr[kg], t_mid, t_lo,
                             L, c_mid, c_lo);
    int jf = -1, m = n;
    bool exact_list = false;
    if (!sel.adaptive) {
        jf = 0;
        exact_list = true;
    } else if (c_lo >= sel.min_pts) {
        jf = -1;  // the guess was at least two steps high: restart at r0
    } else if (c_mid >= sel.min_pts) {
        jf = kg - 1;
        m = c_mid;
    } else if (n >= sel.min_pts) {
        jf = kg;
        exact_list = true;
    } else if (tab.r[kg] >= sel.r_max) {  // r_max reached short (_ext.pyx:266)
        jf = kg;
        status = 1;
        exact_list = true;
    } else {
        jf = -2;  // continue the sequence
    }
    if (jf < 0) {
        int j = jf == -1 ? 0 : kg + 1;
        for (;;) {
            double r, thr;
            seq_radius(tab, sel, j, r, thr);
            int cm, cl;
            m = scan_thread<DIM>(g, cell_start, sorted_pts, t, r, thr, 0.0, 0.0, L, cm, cl);
            if (m >= sel.min_pts) break;
            if (r >= sel.r_max) {
                status = 1;
                break;
            }
            j++;
        }
        jf = j;
        n = m;
        exact_list = true;
    }
    double rf, thr_f;
    seq_radius(tab, sel, jf, rf, thr_f);
    r_out = sel.adaptive ? rf : sel.r_c;
    listed = m <= L.cap;
    if (!listed) return m;
    if (!exact_list && n > L.cap) {  // the wider scan overflowed the list; the support fits
        int cm, cl;
        scan_thread<DIM>(g, cell_start, sorted_pts, t, rf, thr_f, 0.0, 0.0, L, cm, cl);
    } else if (!exact_list) {  // jf = kg - 1: keep codes 0 and 1 (d^2 < T[kg-1])
        int c = 0;
        for (int e = 0; e < n; e++) {
            const uint32_t v = (uint32_t)L.e[e];
            if ((v >> kCodeShift) <= 1u) L.e[c++] = (int32_t)v;
        }
    }
    return m;
}

}  // namespace fm
