// fm_fit.cuh -- per-target weighted least squares on a lane group (fp64).
//
// Semantics: fit_many, _ext.pyx:291-426.  Per target: shift the support to
// the target (centering), scale by s = sqrt(max d^2), build the weighted
// scaled Vandermonde A (m x k) and b = w*f, append ridge rows
// sqrt(lam)/s^deg when lam > 0, solve min ||A c - b|| and map back
// c /= s^deg.  value = c[0] (centered) or mono(t) . c.
//
// B200 formulation.  One group of G lanes owns one target (G = 8 for k <= 6,
// 16 for k <= 10, 32 up to k = 21; 4 lanes for small 2-D supports);
// lane l holds rows l, l+G, ... (ROWS per lane) of A in registers,
// zero-padded -- a zero row changes neither R nor Q^T b.  The solve is an
// unpivoted Householder QR with unnormalised reflectors v = x - beta e_j,
// H = I - gamma v v^T, gamma = 1/(|x|(|x| + |x_0|)) (one division per
// column); column norms and reflector dot products are butterfly reductions
// over the group (bitwise identical on every lane).  Instead of LAPACK
// dgelsy's column-pivoted QR + incremental condition estimate, rank
// deficiency is declared when kappa_1(R) = ||R||_1 ||R^-1||_1 >= 1.5/eps
// (calibrated against dgelsy; status differs only for cond(A) within a
// factor ~2 of 1/eps).  For a well-posed fit the LS solution
// is unique, so values agree with the reference to ~eps*cond(A).
//
// Two outputs:
//   SOLVE  (fit_many):  Q^T b rides along as column k; c = R^-1 (Q^T b).
//   OP     (operator):  the value functional g^T c (g = e0 centered, or
//                       mono(t)/s^deg) is linear in f: value = sum_i W_i f_i
//                       with W = w .* (Q [R^-T g; 0]).  Q is applied as the
//                       stored reflectors (stable), never formed as A R^-1.
#pragma once

#include "fm_common.cuh"

namespace fm {

constexpr double kSingularKappa = 1.5 / 2.220446049250313e-16;

// Row i = q*G + glane against pivot column j; with q and j compile-time
// (unrolled loops) the tests fold to constants for q*G > j.
template <int G>
__device__ __forceinline__ bool row_below(int q, int j, int glane) {
    return q * G > j ? true : glane > j - q * G;
}
template <int G>
__device__ __forceinline__ bool row_diag(int q, int j, int glane) {
    return q * G > j ? false : glane == j - q * G;
}

template <int DIM, int DEG>
struct FitShape {
    static constexpr int K = Monos<DIM, DEG>::K;
    static constexpr int G = K <= 6 ? 8 : (K <= 10 ? 16 : 32);
};

// Returns the group-uniform status (FM_FIT_*).
// Inputs per lane/row q (row index i = q*G + glane): valid[q] (i < m),
// p[q] source coordinates, w[q] weight (already |w|), f[q] field value
// (SOLVE only).  sR: K*K doubles, sQ: 4K doubles of per-group shared memory
// (Q^T b, then gamma, 1/beta and v_0 of every reflector: lane-uniform values
// kept out of registers between the factorisation and the back-substitution).
// OP: y[q] receives the operator weight of row i (0 for invalid rows).
// SOLVE: coeffs[K] (lane-uniform) and value.
template <int DIM, int DEG, int G, int ROWS, bool SOLVE>
__device__ __forceinline__ int fit_rows(const fm_fit &fp, const double *t, int m,
                                        const bool (&valid)[ROWS], const double (&p)[ROWS][DIM],
                                        const double (&w)[ROWS], const double (&f)[ROWS],
                                        int lane, int glane, double *sR, double *sQ,
                                        double (&y)[ROWS], double (&coeffs)[Monos<DIM, DEG>::K],
                                        double &value) {
    constexpr Monos<DIM, DEG> M{};
    constexpr int K = Monos<DIM, DEG>::K;
    constexpr int NC = K + (SOLVE ? 1 : 0);
    static_assert(G * ROWS >= K, "a fit needs at least K row slots");
    const int gbase = lane & ~(G - 1);
    const bool centering = fp.centering != 0;

    // ---- EMPTY: no rows, or no positive weight (_ext.pyx:340-350)
    int npos = 0;
#pragma unroll
    for (int q = 0; q < ROWS; q++) npos += (valid[q] && w[q] > 0.0) ? 1 : 0;
    npos = group_sum_int<G>(npos);
    const bool empty = (m == 0) || (npos == 0);

    // ---- support scale s = sqrt(max |dx|^2) (_ext.pyx:353-366)
    double dx[ROWS][DIM];
    if (centering) {
#pragma unroll
        for (int q = 0; q < ROWS; q++)
#pragma unroll
            for (int a = 0; a < DIM; a++) dx[q][a] = sub_rn(p[q][a], t[a]);
    } else {
#pragma unroll
        for (int q = 0; q < ROWS; q++)
#pragma unroll
            for (int a = 0; a < DIM; a++) dx[q][a] = p[q][a];
    }
    double smax_l = 0.0;
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        double d2 = mul_rn(dx[q][0], dx[q][0]);
#pragma unroll
        for (int a = 1; a < DIM; a++) d2 = add_rn(d2, mul_rn(dx[q][a], dx[q][a]));
        if (valid[q] && d2 > smax_l) smax_l = d2;
    }
    double s = __dsqrt_rn(group_max<G>(smax_l));
    if (s == 0.0) s = 1.0;
    const double inv_s = 1.0 / s;
    // s^deg(c), recomputed where needed rather than held in registers
    auto spow = [&](int c) {
        return M.deg[c] == 0 ? 1.0
               : M.deg[c] == 1 ? s
               : M.deg[c] == 2 ? mul_rn(s, s)
                               : mul_rn(mul_rn(s, s), s);
    };
    double *sGam = sQ + K, *sIb = sQ + 2 * K, *sV0 = sQ + 3 * K;

    // ---- weighted scaled Vandermonde rows (_ext.pyx:374-394)
    double A[ROWS][NC];
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        if (valid[q]) {
            double u[DIM], mono[K];
            // u = dx / s as a product with 1/s: <= 1 ulp from the reference's
            // quotient, far below the 1e-10 value tolerance
#pragma unroll
            for (int a = 0; a < DIM; a++) u[a] = dx[q][a] * inv_s;
            eval_monos<DIM, DEG>(u, mono);
            A[q][0] = w[q];
#pragma unroll
            for (int c = 1; c < K; c++) A[q][c] = mul_rn(mono[c], w[q]);
            if (SOLVE) A[q][NC - 1] = mul_rn(w[q], f[q]);
        } else {
#pragma unroll
            for (int c = 0; c < NC; c++) A[q][c] = 0.0;
        }
    }
    // ridge rows m .. m+K-1: sqrt(lam) / s^deg on the diagonal (_ext.pyx:395-400)
    const bool ridge = fp.lam > 0.0;
    if (ridge) {
        const double sl = sqrt(fp.lam);
        double rdiag[K];
#pragma unroll
        for (int c = 0; c < K; c++) rdiag[c] = __ddiv_rn(sl, spow(c));
#pragma unroll
        for (int q = 0; q < ROWS; q++) {
            const int col = q * G + glane - m;
#pragma unroll
            for (int c = 0; c < K; c++)
                if (c == col) A[q][c] = rdiag[c];
        }
    }

    // ---- Householder QR, column by column
    static_for<0, K>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const double x0 = __shfl_sync(FM_FULL_MASK, A[j / G][j], gbase + (j % G));
        // reflector entries of this lane's rows: 0 above the pivot, v_j on it,
        // A[i][j] below -- selected once per column, so the dot products and
        // updates below are unconditional (a zero entry is an exact no-op)
        double v[ROWS];
#pragma unroll
        for (int q = 0; q < ROWS; q++) v[q] = row_below<G>(q, j, glane) ? A[q][j] : 0.0;
        double sl = 0.0;
#pragma unroll
        for (int q = 0; q < ROWS; q++) sl = fma(v[q], v[q], sl);
        const double sigma = group_sum<G>(sl);
        double gj, bj, vj, ib;
        if (sigma == 0.0) {
            gj = 0.0;  // H = I
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
        if (glane == 0) {
            sGam[j] = gj;
            sIb[j] = ib;
            sV0[j] = vj;
        }
#pragma unroll
        for (int q = 0; q < ROWS; q++)
            if (row_diag<G>(q, j, glane)) v[q] = vj;
        double dot[NC];
#pragma unroll
        for (int l = j + 1; l < NC; l++) {
            double pl = 0.0;
#pragma unroll
            for (int q = 0; q < ROWS; q++) pl = fma(v[q], A[q][l], pl);
            dot[l] = pl;
        }
#pragma unroll
        for (int l = j + 1; l < NC; l++) dot[l] = group_sum<G>(dot[l]);
#pragma unroll
        for (int l = j + 1; l < NC; l++) {
            const double td = gj * dot[l];
#pragma unroll
            for (int q = 0; q < ROWS; q++) A[q][l] = fma(-td, v[q], A[q][l]);
        }
#pragma unroll
        for (int q = 0; q < ROWS; q++)
            if (q * G + glane == j) A[q][j] = bj;  // R_jj; v_j lives in v0[j]
    });

    // ---- R (and Q^T b) to shared memory
#pragma unroll
    for (int q = 0; q < ROWS; q++) {
        const int i = q * G + glane;
        if (i < K) {
#pragma unroll
            for (int l = 0; l < K; l++)
                if (l >= i) sR[i * K + l] = A[q][l];
            if (SOLVE) sQ[i] = A[q][NC - 1];
        }
    }
    __syncwarp();

    // ---- rank test: kappa_1(R) = ||R||_1 ||R^-1||_1 >= 1.5/eps (lam = 0 only).
    // A cheap upper bound first -- with delta = min|r_ii|, M = max|r_ij| (i<j),
    // D = max|r_ii|: kappa_1 <= K max(M, D) (1 + M/delta)^(K-1) / delta -- and
    // the exact kappa only for warps where the bound cannot rule it out.
    bool singular = false;
    if (!ridge) {
        // lane glane owns the columns l = glane, glane + G, ... (G may be < K)
        double offmax = 0.0, dmin = INFINITY, dmax = 0.0;
#pragma unroll
        for (int l0 = 0; l0 < K; l0 += G) {
            const int l = l0 + glane;
            if (l < K) {
                const double d = fabs(sR[l * K + l]);
                dmin = fmin(dmin, d);
                dmax = fmax(dmax, d);
#pragma unroll
                for (int c = 1; c < K; c++)
                    if (c > l) offmax = fmax(offmax, fabs(sR[l * K + c]));
            }
        }
        offmax = group_max<G>(offmax);
        dmax = group_max<G>(dmax);
        dmin = -group_max<G>(-dmin);
        double growth = 1.0;
        const double ratio = 1.0 + offmax / dmin;
#pragma unroll
        for (int i = 1; i < K; i++) growth *= ratio;
        const double bound = (double)K * fmax(offmax, dmax) * growth / dmin;
        const bool unsure = !(bound < 1e12);  // NaN / inf / large: decide exactly
        if (__any_sync(FM_FULL_MASK, unsure)) {
            double colsum = 0.0, invsum = 0.0;
#pragma unroll
            for (int l0 = 0; l0 < K; l0 += G) {
                const int l = l0 + glane;
                double cs = 0.0, is = 0.0;
                double x[K];
#pragma unroll
                for (int ii = 0; ii < K; ii++) {
                    const int i = K - 1 - ii;
                    double acc = (i == l) ? 1.0 : 0.0;
#pragma unroll
                    for (int c = i + 1; c < K; c++) acc = fma(-sR[i * K + c], x[c], acc);
                    x[i] = (i <= l) ? acc * sIb[i] : 0.0;
                    if (i <= l && l < K) {
                        cs += fabs(sR[i * K + l]);
                        is += fabs(x[i]);
                    }
                }
                colsum = fmax(colsum, cs);
                invsum = fmax(invsum, is);
            }
            const double kappa = group_max<G>(colsum) * group_max<G>(invsum);
            singular = unsure && !(kappa < kSingularKappa);
        }
    }
    const int status = empty ? FM_FIT_EMPTY : (singular ? FM_FIT_SINGULAR : FM_FIT_OK);

    if (SOLVE) {
        // c_scaled = R^-1 (Q^T b), coeffs = c_scaled / s^deg (_ext.pyx:411-412)
        double cs[K];
#pragma unroll
        for (int i = K - 1; i >= 0; i--) {
            double acc = sQ[i];
#pragma unroll
            for (int c = i + 1; c < K; c++) acc = fma(-sR[i * K + c], cs[c], acc);
            cs[i] = acc * sIb[i];
        }
#pragma unroll
        for (int c = 0; c < K; c++) coeffs[c] = __ddiv_rn(cs[c], spow(c));
        if (centering) {
            value = coeffs[0];  // _ext.pyx:413-414
        } else {
            double mono_t[K];
            eval_monos<DIM, DEG>(t, mono_t);
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < K; c++) v = add_rn(v, mul_rn(coeffs[c], mono_t[c]));
            value = v;  // _ext.pyx:415-425
        }
    } else {
        // z = R^-T g
        double g[K];
        if (centering) {
#pragma unroll
            for (int i = 0; i < K; i++) g[i] = i == 0 ? 1.0 : 0.0;
        } else {
            double mono_t[K];
            eval_monos<DIM, DEG>(t, mono_t);
#pragma unroll
            for (int i = 0; i < K; i++) g[i] = __ddiv_rn(mono_t[i], spow(i));
        }
        double z[K];
#pragma unroll
        for (int i = 0; i < K; i++) {
            double acc = g[i];
#pragma unroll
            for (int c = 0; c < i; c++) acc = fma(-sR[c * K + i], z[c], acc);
            z[i] = acc * sIb[i];
        }
        double yy[ROWS];
#pragma unroll
        for (int q = 0; q < ROWS; q++) {
            const int i = q * G + glane;
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < K; c++)
                if (i == c) v = z[c];
            yy[q] = v;
        }
        // y = H_0 H_1 ... H_{K-1} [z; 0]  (static_for: a runtime j would
        // move A into local memory)
        static_for<0, K>([&](auto jj) {
            constexpr int j = K - 1 - decltype(jj)::value;
            const double vj = sV0[j];
            double v[ROWS];
#pragma unroll
            for (int q = 0; q < ROWS; q++)
                v[q] = row_diag<G>(q, j, glane) ? vj : row_below<G>(q, j, glane) ? A[q][j] : 0.0;
            double pl = 0.0;
#pragma unroll
            for (int q = 0; q < ROWS; q++) pl = fma(v[q], yy[q], pl);
            const double td = sGam[j] * group_sum<G>(pl);
#pragma unroll
            for (int q = 0; q < ROWS; q++) yy[q] = fma(-td, v[q], yy[q]);
        });
#pragma unroll
        for (int q = 0; q < ROWS; q++) y[q] = valid[q] ? w[q] * yy[q] : 0.0;
    }
    __syncwarp();
    return status;
}

}  // namespace fm
