// fm_common.cuh -- shared device helpers for the field-mapping kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <math.h>
#include <type_traits>
#include <stdint.h>

#include "../../include/fieldmap.h"

#define FM_FULL_MASK 0xffffffffu

#define FM_CHECK_LAUNCH()                                   \
    do {                                                    \
        if (cudaPeekAtLastError() != cudaSuccess) {         \
            (void)cudaGetLastError();                       \
            return FM_ERR_CUDA;                             \
        }                                                   \
    } while (0)

// Debug builds (-DFM_DEBUG; scripts/build_variant.py debug -DFM_DEBUG) trap on
// out-of-range indices at the path's gathers and scatters -- the bounds
// checks standing in for compute-sanitizer, which this GPU pool does not run.
#ifdef FM_DEBUG
#define FM_DCHECK(cond)                                                                   \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("FM_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define FM_DCHECK(cond) \
    do {                \
    } while (0)
#endif

namespace fm {

constexpr int kMaxDim = FM_MAX_DIM;
constexpr int kSMs = 148;  // B200

// Device copy of fm_grid (unused axes: n = 1).
struct GridDev {
    int64_t n[kMaxDim];
    double lo[kMaxDim];
    double inv_d[kMaxDim];
    double d[kMaxDim];  // 1 / inv_d (only used for conservative window bounds)
};

static inline GridDev to_dev(const fm_grid *g) {
    GridDev d{};
    for (int a = 0; a < kMaxDim; a++) {
        d.n[a] = a < g->dim ? g->n[a] : 1;
        d.lo[a] = a < g->dim ? g->lo[a] : 0.0;
        d.inv_d[a] = a < g->dim ? g->inv_d[a] : 0.0;
        d.d[a] = a < g->dim ? 1.0 / g->inv_d[a] : 0.0;
    }
    return d;
}

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// ---------------------------------------------------------------- IEEE ops
// The search path must reproduce the reference's rounding bit for bit
// (_ext.pyx is compiled with -ffp-contract=off, setup.py:5-12), so every
// product/sum there is an explicit round-to-nearest op that nvcc cannot
// contract into an FMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// squared distance sum_a (p_a - t_a)^2, left to right (_ext.pyx:192-194)
template <int DIM>
__device__ __forceinline__ double dist2_rn(const double *p, const double *t) {
    double dx = sub_rn(p[0], t[0]);
    double acc = mul_rn(dx, dx);
#pragma unroll
    for (int a = 1; a < DIM; a++) {
        dx = sub_rn(p[a], t[a]);
        acc = add_rn(acc, mul_rn(dx, dx));
    }
    return acc;
}

// _ext.pyx:78-85
__device__ __forceinline__ int64_t cell_of(double v, double lo, double inv_d, int64_t n) {
    int64_t c = (int64_t)mul_rn(sub_rn(v, lo), inv_d);
    if (c < 0) return 0;
    if (c >= n) return n - 1;
    return c;
}

// _ext.pyx:35-62, same operation order, no contraction.  exp/log are the
// CUDA libm (<= 1-2 ulp from glibc), so Gaussian/TPS weights can differ from
// the reference in the last bit; neighbour sets and distances cannot.
__device__ __forceinline__ double rbf_one(int kind, double a, double r_c, double r) {
    if (kind == FM_RBF_IDENTITY) return 1.0;
    if (r > r_c) return 0.0;
    const double x = __ddiv_rn(mul_rn(a, r), r_c);
    switch (kind) {
    case FM_RBF_GAUSSIAN: return exp(-mul_rn(x, x));
    case FM_RBF_C4: {
        const double u = __ddiv_rn(r, r_c);
        double poly = add_rn(30.0, mul_rn(u, 5.0));
        poly = add_rn(72.0, mul_rn(u, poly));
        poly = add_rn(82.0, mul_rn(u, poly));
        poly = add_rn(36.0, mul_rn(u, poly));
        poly = add_rn(6.0, mul_rn(u, poly));
        const double q = sub_rn(1.0, u);
        const double q2 = mul_rn(q, q);
        return mul_rn(poly, mul_rn(mul_rn(q2, q2), q2));
    }
    case FM_RBF_CONST: return 1.0;
    case FM_RBF_MULTIQUADRIC: return __dsqrt_rn(add_rn(1.0, mul_rn(x, x)));
    case FM_RBF_INVERSE_MULTIQUADRIC:
        return __ddiv_rn(1.0, __dsqrt_rn(add_rn(1.0, mul_rn(x, x))));
    case FM_RBF_THIN_PLATE_SPLINE: return x > 0.0 ? mul_rn(mul_rn(x, x), log(x)) : 0.0;
    case FM_RBF_CUBIC_SPLINE: return mul_rn(mul_rn(x, x), x);
    }
    return -1.0;
}

// The same weights for the fit path, where they only need ~1 ulp (the fit is
// held to 1e-10): products with 1/r_c instead of IEEE divisions.  The support
// ABI (fm_support_fill, fm_rbf_weights) keeps rbf_one.
__device__ __forceinline__ double rbf_fast(int kind, double a, double r_c, double inv_rc,
                                           double r) {
    if (kind == FM_RBF_IDENTITY) return 1.0;
    if (r > r_c) return 0.0;
    const double u = r * inv_rc;
    const double x = a * u;
    switch (kind) {
    case FM_RBF_GAUSSIAN: return exp(-(x * x));
    case FM_RBF_C4: {
        double poly = fma(u, 5.0, 30.0);
        poly = fma(u, poly, 72.0);
        poly = fma(u, poly, 82.0);
        poly = fma(u, poly, 36.0);
        poly = fma(u, poly, 6.0);
        const double q = 1.0 - u;
        const double q2 = q * q;
        return poly * (q2 * q2 * q2);
    }
    case FM_RBF_CONST: return 1.0;
    case FM_RBF_MULTIQUADRIC: return sqrt(fma(x, x, 1.0));
    case FM_RBF_INVERSE_MULTIQUADRIC: return rsqrt(fma(x, x, 1.0));
    case FM_RBF_THIN_PLATE_SPLINE: return x > 0.0 ? x * x * log(x) : 0.0;
    case FM_RBF_CUBIC_SPLINE: return x * x * x;
    }
    return -1.0;
}

// ------------------------------------------------------------- monomials
// Graded-lex monomials in DIM variables up to DEG (x0 > x1 > ...); for DIM=2
// this is [1, x, y, x^2, xy, y^2] (pointwise.py:44) extended by
// [x^3, x^2y, xy^2, y^3].  Monomial c > 0 equals monomial parent[c] times
// variable var[c]; the parent drops one power of the last variable present,
// so products are formed left to right in variable order (`u * v * w`,
// _ext.pyx:391-393).  Same table as oracle/fb_oracle.c make_monos().
constexpr int binom(int n, int k) {
    int r = 1;
    for (int i = 1; i <= k; i++) r = r * (n - k + i) / i;
    return r;
}

template <int DIM, int DEG>
struct Monos {
    static constexpr int K = binom(DIM + DEG, DEG);
    int parent[K];
    int var[K];
    int deg[K];
    constexpr Monos() : parent(), var(), deg() {
        int exps[K][kMaxDim] = {};
        int k = 0;
        for (int q = 0; q <= DEG; q++) {
            int e[kMaxDim] = {};
            e[0] = q;
            for (;;) {
                for (int a = 0; a < DIM; a++) exps[k][a] = e[a];
                deg[k] = q;
                k++;
                int a = DIM - 2;
                while (a >= 0 && e[a] == 0) a--;
                if (a < 0) break;
                e[a]--;
                int rest = 0;
                for (int b = a + 1; b < DIM; b++) {
                    rest += e[b];
                    e[b] = 0;
                }
                e[a + 1] = rest + 1;
            }
        }
        parent[0] = -1;
        var[0] = -1;
        for (int c = 1; c < K; c++) {
            int v = DIM - 1;
            while (exps[c][v] == 0) v--;
            int pe[kMaxDim] = {};
            for (int a = 0; a < DIM; a++) pe[a] = exps[c][a];
            pe[v]--;
            int p = -1;
            for (int c2 = 0; c2 < c && p < 0; c2++) {
                bool same = true;
                for (int a = 0; a < DIM; a++)
                    if (exps[c2][a] != pe[a]) same = false;
                if (same) p = c2;
            }
            parent[c] = p;
            var[c] = v;
        }
    }
};

// mono[c] for coordinates x (fully unrolled; plain IEEE products as in the
// reference, contraction-free because they are pure products)
template <int DIM, int DEG>
__device__ __forceinline__ void eval_monos(const double *x, double *mono) {
    constexpr Monos<DIM, DEG> M{};
    mono[0] = 1.0;
#pragma unroll
    for (int c = 1; c < M.K; c++) {
        if (M.parent[c] == 0)
            mono[c] = x[M.var[c]];
        else
            mono[c] = mul_rn(mono[M.parent[c]], x[M.var[c]]);
    }
}

// 1/x and 1/sqrt(x) to ~1 ulp: MUFU seed + three Newton steps.  Only the fit
// uses them (held to 1e-10, not bitwise); 0 -> NaN/inf propagates into the
// rank test, which then reports FIT_SINGULAR.
__device__ __forceinline__ double rcp_fast(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int it = 0; it < 3; it++) y = fma(y, fma(-x, y, 1.0), y);
    return y;
}
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int it = 0; it < 3; it++) y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    return y;
}

// Compile-time loop: f(std::integral_constant<int, 0>) ... f(<N-1>).  Used
// where `#pragma unroll` is not honoured and a runtime index would push the
// register-resident matrix into local memory.
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

// ------------------------------------------------------- group collectives
// A "group" is G consecutive, G-aligned lanes of a warp (G = 8, 16 or 32).
// All collectives use the full-warp mask: callers keep control flow
// warp-uniform (loop bounds are reduced over the warp first).
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FM_FULL_MASK, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FM_FULL_MASK, v, o));
    return v;
}
template <int G>
__device__ __forceinline__ int group_sum_int(int v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FM_FULL_MASK, v, o);
    return v;
}
template <int G>
__device__ __forceinline__ int group_max_int(int v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FM_FULL_MASK, v, o));
    return v;
}
// inclusive prefix sum over the group
template <int G>
__device__ __forceinline__ int group_scan_incl(int v, int glane) {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        int u = __shfl_up_sync(FM_FULL_MASK, v, o, G);
        if (glane >= o) v += u;
    }
    return v;
}
template <int G>
__device__ __forceinline__ unsigned group_bits(unsigned ballot, int lane) {
    if constexpr (G == 32) {
        return ballot;
    } else {
        const int base = lane & ~(G - 1);
        return (ballot >> base) & ((1u << G) - 1u);
    }
}

__device__ __forceinline__ int warp_max_int(int v) { return __reduce_max_sync(FM_FULL_MASK, v); }

// --------------------------------------------------- asynchronous copies
// cp.async (global -> shared, bypassing registers); a false predicate
// zero-fills the destination without reading the source.  Completion is per
// thread: cp_async_wait_all() then __syncwarp() before other lanes read.
__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
                 "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src, bool pred) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
                 "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

}  // namespace fm
