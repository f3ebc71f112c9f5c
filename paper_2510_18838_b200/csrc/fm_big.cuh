// fm_big.cuh -- fits of any support size (the reference has no bound:
// fit_many sizes its LAPACK workspace from the largest support,
// _ext.pyx:305-312).  The register-resident lane-group fit (fm_fit.cuh)
// holds at most 256 rows; larger supports -- big fixed radii, many patch
// layers -- come here: one warp per target, the weighted scaled Vandermonde
// in global scratch (column-major, L2-resident), the same unpivoted
// Householder QR with warp reductions over the rows, the same rank test,
// the same SOLVE / OP outputs.  Slow next to the register fit, and only
// reached by the few targets that need it.
#pragma once

#include "fm_fit.cuh"
#include "fm_search.cuh"

namespace fm {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FM_FULL_MASK, v, o);
    return v;
}
__device__ __forceinline__ double warp_maxd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FM_FULL_MASK, v, o));
    return v;
}

// Support of position k at radius r, gathered by one warp (window rows in
// chunks of 32, the exact d^2 < T(r) test) into pos[0..) (grid positions,
// discovery order).  Returns the count.
template <int DIM>
__device__ int gather_warp(const GridDev &g, const int32_t *__restrict__ cell_start,
                           const double *__restrict__ sorted_pts, const double *t, double r,
                           int lane, RowTable<32> &rt, int32_t *pos, int cap) {
    const double thr = sqrt_threshold(r);
    const unsigned lt = (1u << lane) - 1u;
    int n = 0;
    Window<DIM, 32> w(g, t, r, true);
    for (int ch = 0; ch < w.nchunks_w; ch++) {
        const int iters = w.chunk(g, cell_start, t, ch, lane, rt);
        for (int it = 0; it < iters; it++) {
            bool valid;
            const int p = w.pos(it, lane, rt, valid);
            bool keep = false;
            if (valid) {
                double q[DIM];
                load_point<DIM>(sorted_pts, p, q);
                keep = dist2_rn<DIM>(q, t) < thr;
            }
            const unsigned bits = __ballot_sync(FM_FULL_MASK, keep);
            if (keep) {
                const int o = n + __popc(bits & lt);
                if (o < cap) pos[o] = p;
            }
            n += __popc(bits);
        }
        __syncwarp();
    }
    return n;
}

struct BigArgs {
    // rows: either grid positions (build: pos[k*stride + i], coordinates
    // sorted_pts, ids sorted_ids, weights |rbf(d, r)|) or a CSR (fit_many:
    // sup_off/sup_idx/sup_w into src by id)
    const int32_t *klist;  // positions (build) / targets (fit_many) of this launch
    int64_t nk;
    int64_t stride;        // scratch rows per warp (>= max rows incl. ridge)
    double *A;             // scratch: nk x (NC + 2) x stride doubles (column-major per warp)
    int32_t *pos;          // scratch: nk x stride grid positions (build)
    const int64_t *sup_off;
    const int64_t *sup_idx;
    const double *sup_w;
    const double *src;
    double *coeffs;        // fit_many (nt x K) or null
};

// One warp per target: rows -> weighted scaled Vandermonde in scratch ->
// Householder QR -> outputs as build_core / k_fit_many.
template <int DIM, int DEG, bool SOLVE, bool CSR>
__global__ void __launch_bounds__(128) k_fit_big(SearchArgs s, BuildArgs b, BigArgs g) {
    constexpr Monos<DIM, DEG> M{};
    constexpr int K = Monos<DIM, DEG>::K;
    constexpr int NC = K + (SOLVE ? 1 : 0);
    __shared__ RowTable<32> rts[4];
    __shared__ double sRs[4][K * K + 3 * K];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double *sR = sRs[wib], *sGam = sR + K * K, *sIb = sGam + K, *sV0 = sIb + K;
    int nfail = 0, first_fail = INT32_MAX;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t ii = warp; ii < g.nk; ii += nwarps) {
        const int64_t k = g.klist ? (int64_t)g.klist[ii] : ii;
        int64_t tid;
        double t[DIM], r = 0.0;
        int m;
        int64_t rb = 0;
        if (CSR) {
            tid = k;
            load_target<DIM>(s.targets, tid, true, t);
            rb = g.sup_off[k];
            m = (int)(g.sup_off[k + 1] - rb);
        } else {
            tid = s.perm ? (int64_t)s.perm[k] : k;
            load_target<DIM>(s.targets, tid, true, t);
            r = s.radii ? s.radii[tid] : s.sel.r_c;
            m = gather_warp<DIM>(s.g, s.cell_start, s.sorted_pts, t, r, lane, rts[wib],
                                 g.pos + ii % nwarps * g.stride, (int)g.stride);
        }
        const bool ridge = b.fp.lam > 0.0;
        const int nr = m + (ridge ? K : 0);
        double *A = g.A + (ii % nwarps) * g.stride * (NC + 2);  // columns 0..NC-1, w, y
        double *Wc = A + NC * g.stride, *Yc = A + (NC + 1) * g.stride;
        const int32_t *pos = g.pos + (ii % nwarps) * g.stride;
        // ---- rows: coordinates, weights, EMPTY test, scale s
        double smax = 0.0;
        int npos = 0;
        for (int i = lane; i < m; i += 32) {
            double p[DIM], w;
            if (CSR) {
                const int64_t id = g.sup_idx[rb + i];
#pragma unroll
                for (int a = 0; a < DIM; a++) p[a] = __ldg(g.src + id * DIM + a);
                w = g.sup_w[rb + i];
            } else {
                load_point<DIM>(s.sorted_pts, pos[i], p);
                const double d = __dsqrt_rn(dist2_rn<DIM>(p, t));
                w = fabs(rbf_fast(b.rbf_kind, b.rbf_a, r, 1.0 / r, d));
            }
            npos += w > 0.0;
            double d2 = 0.0;
#pragma unroll
            for (int a = 0; a < DIM; a++) {
                const double dx = b.fp.centering ? sub_rn(p[a], t[a]) : p[a];
                d2 = add_rn(d2, mul_rn(dx, dx));
            }
            smax = fmax(smax, d2);
            Wc[i] = w;
        }
        smax = warp_maxd(smax);
        npos = __reduce_add_sync(FM_FULL_MASK, npos);
        const bool empty = m == 0 || npos == 0;
        double sc = __dsqrt_rn(smax);
        if (sc == 0.0) sc = 1.0;
        const double inv_s = 1.0 / sc;
        auto spow = [&](int c) {
            return M.deg[c] == 0 ? 1.0 : M.deg[c] == 1 ? sc : M.deg[c] == 2 ? mul_rn(sc, sc)
                                                                         : mul_rn(mul_rn(sc, sc), sc);
        };
        __syncwarp();
        for (int i = lane; i < nr; i += 32) {
            double row[NC];
            if (i < m) {
                double p[DIM], u[DIM], mono[K];
                if (CSR) {
                    const int64_t id = g.sup_idx[rb + i];
#pragma unroll
                    for (int a = 0; a < DIM; a++) p[a] = __ldg(g.src + id * DIM + a);
                } else {
                    load_point<DIM>(s.sorted_pts, pos[i], p);
                }
#pragma unroll
                for (int a = 0; a < DIM; a++)
                    u[a] = (b.fp.centering ? sub_rn(p[a], t[a]) : p[a]) * inv_s;
                eval_monos<DIM, DEG>(u, mono);
                const double w = Wc[i];
                row[0] = w;
#pragma unroll
                for (int c = 1; c < K; c++) row[c] = mul_rn(mono[c], w);
                if (SOLVE) {
                    double f;
                    if (CSR) f = __ldg(b.src_val + g.sup_idx[rb + i]);
                    else f = __ldg(b.src_val + __ldg(s.sorted_ids + pos[i]));
                    row[NC - 1] = mul_rn(w, f);
                }
            } else {  // ridge rows sqrt(lam)/s^deg on the diagonal (_ext.pyx:395-400)
#pragma unroll
                for (int c = 0; c < NC; c++)
                    row[c] = (c == i - m) ? __ddiv_rn(sqrt(b.fp.lam), spow(c)) : 0.0;
            }
#pragma unroll
            for (int c = 0; c < NC; c++) A[c * g.stride + i] = row[c];
        }
        __syncwarp();
        // ---- Householder QR over the rows (warp reductions)
        for (int j = 0; j < K; j++) {
            double *Aj = A + j * g.stride;
            const double x0 = Aj[j];
            double sl = 0.0;
            for (int i = j + 1 + lane; i < nr; i += 32) sl = fma(Aj[i], Aj[i], sl);
            const double sigma = warp_sum(sl);
            double gj, bj, vj, ib;
            if (sigma == 0.0) {
                gj = 0.0;
                bj = x0;
                vj = 0.0;
                ib = rcp_fast(x0);
            } else {
                const double s2 = fma(x0, x0, sigma);
                const double rn = rsqrt_fast(s2);
                const double nrm = s2 * rn;
                bj = x0 >= 0.0 ? -nrm : nrm;
                ib = x0 >= 0.0 ? -rn : rn;
                vj = x0 - bj;
                gj = rcp_fast(nrm * (nrm + fabs(x0)));
            }
            if (lane == 0) {
                sGam[j] = gj;
                sIb[j] = ib;
                sV0[j] = vj;
            }
            for (int l = j + 1; l < NC; l++) {
                double *Al = A + l * g.stride;
                double pl = lane == 0 ? vj * Al[j] : 0.0;
                for (int i = j + 1 + lane; i < nr; i += 32) pl = fma(Aj[i], Al[i], pl);
                const double td = gj * warp_sum(pl);
                if (lane == 0) Al[j] = fma(-td, vj, Al[j]);
                for (int i = j + 1 + lane; i < nr; i += 32) Al[i] = fma(-td, Aj[i], Al[i]);
                __syncwarp();
            }
            if (lane == 0) Aj[j] = bj;
            __syncwarp();
        }
        // R (and Q^T b) to shared memory
        for (int e = lane; e < K * K; e += 32) {
            const int i = e / K, l = e % K;
            sR[e] = l >= i ? A[l * g.stride + i] : 0.0;
        }
        __syncwarp();
        // ---- rank test (lam = 0): exact kappa_1(R) >= 1.5/eps (fm_fit.cuh)
        bool singular = false;
        if (!ridge) {
            double colsum = 0.0, invsum = 0.0;
            for (int l = lane; l < K; l += 32) {
                double x[K];
                double cs = 0.0, is = 0.0;
#pragma unroll
                for (int ii2 = 0; ii2 < K; ii2++) {
                    const int i = K - 1 - ii2;
                    double acc = (i == l) ? 1.0 : 0.0;
#pragma unroll
                    for (int c = i + 1; c < K; c++) acc = fma(-sR[i * K + c], x[c], acc);
                    x[i] = (i <= l) ? acc * sIb[i] : 0.0;
                    if (i <= l) {
                        cs += fabs(sR[i * K + l]);
                        is += fabs(x[i]);
                    }
                }
                colsum = fmax(colsum, cs);
                invsum = fmax(invsum, is);
            }
            const double kappa = warp_maxd(colsum) * warp_maxd(invsum);
            singular = !(kappa < kSingularKappa);
        }
        const int st = empty ? FM_FIT_EMPTY : (singular ? FM_FIT_SINGULAR : FM_FIT_OK);
        if (lane == 0) {
            b.status[tid] = (uint8_t)st;
            if (st != FM_FIT_OK) {
                nfail++;
                first_fail = min(first_fail, (int)tid);
            }
        }
        if (SOLVE) {
            double cs[K], co[K];
#pragma unroll
            for (int i = K - 1; i >= 0; i--) {
                double acc = A[(NC - 1) * g.stride + i];
#pragma unroll
                for (int c = i + 1; c < K; c++) acc = fma(-sR[i * K + c], cs[c], acc);
                cs[i] = acc * sIb[i];
            }
#pragma unroll
            for (int c = 0; c < K; c++) co[c] = __ddiv_rn(cs[c], spow(c));
            double value = co[0];
            if (!b.fp.centering) {
                double mt[K];
                eval_monos<DIM, DEG>(t, mt);
                value = 0.0;
#pragma unroll
                for (int c = 0; c < K; c++) value = add_rn(value, mul_rn(co[c], mt[c]));
            }
            if (lane == 0 && b.values) b.values[tid] = st == FM_FIT_OK ? value : NAN;
            if (g.coeffs)
                for (int c = lane; c < K; c += 32) g.coeffs[tid * K + c] = st == FM_FIT_OK ? co[c] : NAN;
        } else {
            // z = R^-T g, y = H_0 ... H_{K-1} [z; 0], W = w .* y
            double gv[K], z[K];
            if (b.fp.centering) {
#pragma unroll
                for (int i = 0; i < K; i++) gv[i] = i == 0 ? 1.0 : 0.0;
            } else {
                double mt[K];
                eval_monos<DIM, DEG>(t, mt);
#pragma unroll
                for (int i = 0; i < K; i++) gv[i] = __ddiv_rn(mt[i], spow(i));
            }
#pragma unroll
            for (int i = 0; i < K; i++) {
                double acc = gv[i];
#pragma unroll
                for (int c = 0; c < i; c++) acc = fma(-sR[c * K + i], z[c], acc);
                z[i] = acc * sIb[i];
            }
            for (int i = lane; i < nr; i += 32) {
                double v = 0.0;
#pragma unroll
                for (int c = 0; c < K; c++)
                    if (i == c) v = z[c];
                Yc[i] = v;
            }
            __syncwarp();
            for (int j = K - 1; j >= 0; j--) {
                const double *Aj = A + j * g.stride;
                double pl = lane == 0 ? sV0[j] * Yc[j] : 0.0;
                for (int i = j + 1 + lane; i < nr; i += 32) pl = fma(Aj[i], Yc[i], pl);
                const double td = sGam[j] * warp_sum(pl);
                if (lane == 0) Yc[j] = fma(-td, sV0[j], Yc[j]);
                for (int i = j + 1 + lane; i < nr; i += 32) Yc[i] = fma(-td, Aj[i], Yc[i]);
                __syncwarp();
            }
            const int64_t off = b.offsets[k];
            for (int i = lane; i < m; i += 32) {
                b.col[off + i] = CSR ? (int32_t)g.sup_idx[rb + i] : __ldg(s.sorted_ids + pos[i]);
                b.val[off + i] = st == FM_FIT_OK ? Wc[i] * Yc[i] : NAN;
            }
        }
        __syncwarp();
    }
    if (b.stats) warp_flush_pair(b.stats, nfail, first_fail);
}

// Launch the warp-per-target fit over `nk` positions/targets in chunks
// whose scratch stays within ~1 GB (stream-ordered allocation).
template <int DIM, int DEG, bool SOLVE, bool CSR>
int launch_fit_big(const SearchArgs &s, const BuildArgs &b, BigArgs g, int max_rows,
                   cudaStream_t st) {
    constexpr int K = Monos<DIM, DEG>::K;
    constexpr int NC = K + (SOLVE ? 1 : 0);
    if (g.nk <= 0) return FM_OK;
    g.stride = (max_rows + 31) & ~31;
    const size_t per_warp = (size_t)g.stride * ((NC + 2) * sizeof(double) + sizeof(int32_t));
    int64_t warps = (int64_t)((size_t)1 << 30) / (int64_t)per_warp;
    warps = warps < 4 ? 4 : (warps > kSMs * 16 ? kSMs * 16 : warps);
    if (warps > g.nk) warps = g.nk;
    // the kernel's scratch slot is its warp index: one slot per launched warp
    const int blocks = (int)((warps + 3) / 4);
    const size_t slots = (size_t)blocks * 4;
    void *scratch = nullptr;
    if (cudaMallocAsync(&scratch, per_warp * slots, st) != cudaSuccess) return FM_ERR_CUDA;
    g.A = reinterpret_cast<double *>(scratch);
    g.pos = reinterpret_cast<int32_t *>(g.A + slots * g.stride * (NC + 2));
    k_fit_big<DIM, DEG, SOLVE, CSR><<<blocks, 128, 0, st>>>(s, b, g);
    const bool ok = cudaPeekAtLastError() == cudaSuccess;
    cudaFreeAsync(scratch, st);
    if (!ok) {
        (void)cudaGetLastError();
        return FM_ERR_CUDA;
    }
    return FM_OK;
}

}  // namespace fm
