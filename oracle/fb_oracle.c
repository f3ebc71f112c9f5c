/*
 * fb_oracle.c -- CPU restatement of the reference field-mapping hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * library in paper_2510_18838_b200/csrc; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  It is never on the product
 * path.
 *
 * What it restates (reference = /root/reference/pkg/src/fieldbridge):
 *   _kernels/_ext.pyx:35-62    _rbf_one        -> orc_rbf
 *   _kernels/_ext.pyx:78-85    _cell_of        -> cell_of
 *   _kernels/_ext.pyx:155-169  _sort_by_id     -> sort_by_id
 *   _kernels/_ext.pyx:172-200  _gather_radius  -> gather_radius
 *   _kernels/_ext.pyx:203-235  fixed_radius_supports    -> orc_fixed_count / orc_fill
 *   _kernels/_ext.pyx:238-288  adaptive_radius_supports -> orc_adaptive_count / orc_fill
 *   _kernels/_ext.pyx:291-426  fit_many        -> orc_fit_many
 *
 * Same operation order as _ext.pyx (compiled with -ffp-contract=off like the
 * reference's setup.py:5-12), and the least-squares solve calls the very
 * same LAPACK dgelsy the reference calls (scipy.linalg.cython_lapack ->
 * scipy-openblas `scipy_dgelsy_`; pointer handed in by oracle/oracle.py).
 * On 2-D inputs with degree <= 2 the outputs are therefore bitwise equal to
 * the reference (pinned by tests/test_oracle.py against tests/golden/).
 *
 * Extensions beyond the reference (unpinned by any reference test; defined
 * here and in DESIGN.md):
 *   - dimension 1..5: cells are linearised with axis 0 fastest (the
 *     reference's `iy * nx + ix`), distances summed left to right
 *     (((dx0*dx0 + dx1*dx1) + dx2*dx2) + ...);
 *   - degree 3: monomials in graded-lex order x0 > x1 > ..., each monomial
 *     built as parent-monomial * coordinate (the reference's `u * u * w`
 *     pattern), column scale s^deg built as s, s*s, (s*s)*s;
 *   - several field components: each column is fitted independently with
 *     the scalar semantics (nrhs = 1 per column).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_DIM 5
#define ORC_MAX_K 56 /* C(5+3,3) */

typedef void (*dgelsy_fn)(const int *m, const int *n, const int *nrhs, double *a,
                          const int *lda, double *b, const int *ldb, int *jpvt,
                          const double *rcond, int *rank, double *work,
                          const int *lwork, int *info);

static dgelsy_fn g_dgelsy = 0;

void orc_set_dgelsy(void *fn) { g_dgelsy = (dgelsy_fn)fn; }

/* ------------------------------------------------------------------ rbf */
/* _ext.pyx:35-62 */
static inline double rbf_one(int kind, double a, double r_c, double r) {
    double x, u, poly, q, q2;
    if (kind == 3) return 1.0;
    if (r > r_c) return 0.0;
    x = a * r / r_c;
    switch (kind) {
    case 0: return exp(-(x * x));
    case 1:
        u = r / r_c;
        poly = 6.0 + u * (36.0 + u * (82.0 + u * (72.0 + u * (30.0 + u * 5.0))));
        q = 1.0 - u;
        q2 = q * q;
        return poly * (q2 * q2 * q2);
    case 2: return 1.0;
    case 4: return sqrt(1.0 + x * x);
    case 5: return 1.0 / sqrt(1.0 + x * x);
    case 6: return x > 0.0 ? x * x * log(x) : 0.0;
    case 7: return x * x * x;
    }
    return -1.0;
}

int orc_rbf(int kind, double a, double r_c, const double *r, int64_t n, double *out) {
    if (kind < 0 || kind > 7) return -1;
    for (int64_t i = 0; i < n; i++) out[i] = rbf_one(kind, a, r_c, r[i]);
    return 0;
}

/* pointwise.py:266-269: rbf_weights of each target's support at that
 * target's own final radius (the adaptive per-target loop, in C). */
int orc_rbf_per_target(int kind, double a, const int64_t *off, int64_t nt,
                       const double *radii, const double *r, double *out) {
    if (kind < 0 || kind > 7) return -1;
    for (int64_t t = 0; t < nt; t++)
        for (int64_t j = off[t]; j < off[t + 1]; j++) out[j] = rbf_one(kind, a, radii[t], r[j]);
    return 0;
}

/* ----------------------------------------------------------------- grid */
typedef struct {
    int dim;
    int64_t n[ORC_MAX_DIM];
    double lo[ORC_MAX_DIM];
    double inv_d[ORC_MAX_DIM];
} orc_grid;

/* _ext.pyx:78-85 */
static inline int64_t cell_of(double v, double lo, double inv_d, int64_t n) {
    int64_t c = (int64_t)((v - lo) * inv_d);
    if (c < 0) return 0;
    if (c >= n) return n - 1;
    return c;
}

/* _ext.pyx:155-169 */
static void sort_by_id(int64_t *ids, double *ds, int64_t n) {
    for (int64_t i = 1; i < n; i++) {
        int64_t id_i = ids[i];
        double d_i = ds[i];
        int64_t j = i - 1;
        while (j >= 0 && ids[j] > id_i) {
            ids[j + 1] = ids[j];
            ds[j + 1] = ds[j];
            j--;
        }
        ids[j + 1] = id_i;
        ds[j + 1] = d_i;
    }
}

static inline double dist_of(int dim, const double *p, const double *t) {
    double acc, dx;
    dx = p[0] - t[0];
    acc = dx * dx;
    for (int a = 1; a < dim; a++) {
        dx = p[a] - t[a];
        acc = acc + dx * dx;
    }
    return sqrt(acc);
}

/* _ext.pyx:172-200, generalised to `dim` axes (axis 0 innermost). */
static int64_t gather_radius(const orc_grid *g, const double *t, double r,
                             const double *pts, const int64_t *cell_off,
                             const int64_t *cell_items, int64_t *out_ids,
                             double *out_ds, int count_only) {
    const int dim = g->dim;
    int64_t lo[ORC_MAX_DIM], hi[ORC_MAX_DIM], cur[ORC_MAX_DIM];
    int64_t m = 0;
    for (int a = 0; a < dim; a++) {
        lo[a] = cell_of(t[a] - r, g->lo[a], g->inv_d[a], g->n[a]);
        hi[a] = cell_of(t[a] + r, g->lo[a], g->inv_d[a], g->n[a]);
        cur[a] = lo[a];
    }
    for (;;) {
        int64_t c = 0, stride = 1;
        for (int a = 0; a < dim; a++) {
            c += cur[a] * stride;
            stride *= g->n[a];
        }
        for (int64_t j = cell_off[c]; j < cell_off[c + 1]; j++) {
            int64_t p = cell_items[j];
            double d = dist_of(dim, pts + p * dim, t);
            if (d < r) {
                if (!count_only) {
                    out_ids[m] = p;
                    out_ds[m] = d;
                }
                m++;
            }
        }
        int a = 0;
        while (a < dim) {
            if (cur[a] < hi[a]) {
                cur[a]++;
                break;
            }
            cur[a] = lo[a];
            a++;
        }
        if (a == dim) break;
    }
    return m;
}

static void fill_grid(orc_grid *g, int dim, const int64_t *n, const double *lo,
                      const double *inv_d) {
    g->dim = dim;
    for (int a = 0; a < dim; a++) {
        g->n[a] = n[a];
        g->lo[a] = lo[a];
        g->inv_d[a] = inv_d[a];
    }
}

/* _ext.pyx:215-220: count pass of fixed_radius_supports */
int orc_fixed_count(int dim, const double *targets, int64_t nt, const double *pts,
                    const int64_t *n, const double *lo, const double *inv_d,
                    const int64_t *cell_off, const int64_t *cell_items, double r_c,
                    int64_t *counts, int nthreads) {
    orc_grid g;
    fill_grid(&g, dim, n, lo, inv_d);
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads)
    for (int64_t i = 0; i < nt; i++)
        counts[i] = gather_radius(&g, targets + i * dim, r_c, pts, cell_off, cell_items,
                                  0, 0, 1);
    return 0;
}

/* _ext.pyx:256-272: radius growth loop of adaptive_radius_supports */
int orc_adaptive_count(int dim, const double *targets, int64_t nt, const double *pts,
                       const int64_t *n, const double *lo, const double *inv_d,
                       const int64_t *cell_off, const int64_t *cell_items,
                       int64_t min_pts, double r0, double growth, double r_max,
                       int64_t *counts, double *radii, uint8_t *status, int nthreads) {
    orc_grid g;
    fill_grid(&g, dim, n, lo, inv_d);
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (int64_t i = 0; i < nt; i++) {
        double r = r0;
        int64_t m;
        status[i] = 0;
        for (;;) {
            m = gather_radius(&g, targets + i * dim, r, pts, cell_off, cell_items, 0, 0, 1);
            if (m >= min_pts) break;
            if (r >= r_max) {
                status[i] = 1;
                break;
            }
            r = r * growth;
            if (r > r_max) r = r_max;
        }
        radii[i] = r;
        counts[i] = m;
    }
    return 0;
}

/* _ext.pyx:225-234 / 277-287: fill pass at a per-target radius (radii may be
 * NULL for a fixed radius r_c), then insertion sort by id. */
int orc_fill(int dim, const double *targets, int64_t nt, const double *pts,
             const int64_t *n, const double *lo, const double *inv_d,
             const int64_t *cell_off, const int64_t *cell_items, double r_c,
             const double *radii, const int64_t *offsets, int64_t *idx, double *dist,
             int nthreads) {
    orc_grid g;
    fill_grid(&g, dim, n, lo, inv_d);
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads)
    for (int64_t i = 0; i < nt; i++) {
        int64_t o = offsets[i], m = offsets[i + 1] - offsets[i];
        if (m == 0) continue;
        double r = radii ? radii[i] : r_c;
        gather_radius(&g, targets + i * dim, r, pts, cell_off, cell_items, idx + o,
                      dist + o, 0);
        if (m > 1) sort_by_id(idx + o, dist + o, m);
    }
    return 0;
}

/* ------------------------------------------------------------ monomials */
/* Graded-lex monomials in `dim` variables up to `degree`; monomial c (c>0) is
 * parent[c] * x[var[c]].  For dim 2 this is [1, x, y, x^2, xy, y^2, x^3,
 * x^2y, xy^2, y^3] -- pointwise.py:44 extended. */
typedef struct {
    int k;
    int deg[ORC_MAX_K];
    int parent[ORC_MAX_K];
    int var[ORC_MAX_K];
} orc_monos;

static int n_monos(int dim, int degree) {
    /* C(dim + degree, degree) */
    long num = 1, den = 1;
    for (int i = 1; i <= degree; i++) {
        num *= dim + i;
        den *= i;
    }
    return (int)(num / den);
}

static void make_monos(int dim, int degree, orc_monos *mo) {
    int exps[ORC_MAX_K][ORC_MAX_DIM];
    int k = 0;
    memset(exps, 0, sizeof(exps));
    for (int q = 0; q <= degree; q++) {
        /* exponent tuples of total degree q in lex-descending order */
        int e[ORC_MAX_DIM];
        memset(e, 0, sizeof(e));
        e[0] = q;
        for (;;) {
            for (int a = 0; a < dim; a++) exps[k][a] = e[a];
            mo->deg[k] = q;
            k++;
            /* next tuple in lex-descending order */
            int a = dim - 2;
            while (a >= 0 && e[a] == 0) a--;
            if (a < 0) break;
            e[a]--;
            int rest = 0;
            for (int b = a + 1; b < dim; b++) {
                rest += e[b];
                e[b] = 0;
            }
            e[a + 1] = rest + 1;
        }
    }
    mo->k = k;
    mo->parent[0] = -1;
    mo->var[0] = -1;
    for (int c = 1; c < k; c++) {
        /* the parent drops one power of the LAST variable with a positive
         * exponent, so the product is built left to right in variable
         * order: x*x*y, matching the reference's `u * v * w`. */
        int v = dim - 1;
        while (exps[c][v] == 0) v--;
        int pe[ORC_MAX_DIM];
        for (int a = 0; a < dim; a++) pe[a] = exps[c][a];
        pe[v]--;
        int p = -1;
        for (int c2 = 0; c2 < c; c2++) {
            int same = 1;
            for (int a = 0; a < dim; a++)
                if (exps[c2][a] != pe[a]) same = 0;
            if (same) {
                p = c2;
                break;
            }
        }
        mo->parent[c] = p;
        mo->var[c] = v;
    }
}

int orc_n_monomials(int dim, int degree) { return n_monos(dim, degree); }

/* exposes the monomial table for the CUDA side's self-check */
int orc_monomial_table(int dim, int degree, int *parent, int *var, int *deg) {
    orc_monos mo;
    make_monos(dim, degree, &mo);
    for (int c = 0; c < mo.k; c++) {
        parent[c] = mo.parent[c];
        var[c] = mo.var[c];
        deg[c] = mo.deg[c];
    }
    return mo.k;
}

static inline void eval_monos(const orc_monos *mo, const double *x, double *out) {
    out[0] = 1.0;
    for (int c = 1; c < mo->k; c++) {
        if (mo->parent[c] == 0)
            out[c] = x[mo->var[c]];
        else
            out[c] = out[mo->parent[c]] * x[mo->var[c]];
    }
}

/* ------------------------------------------------------------------ fit */
/* _ext.pyx:291-426.  `ncomp` columns of src_val (row-major (ns, ncomp)) are
 * fitted one by one; values (nt, ncomp), coeffs (nt, ncomp, k). */
int orc_fit_many(int dim, int degree, double lam, int centering, const double *targets,
                 int64_t nt, const int64_t *sup_off, const int64_t *sup_idx,
                 const double *sup_w, const double *src, const double *src_val,
                 int ncomp, double *values, double *coeffs, uint8_t *status,
                 int nthreads) {
    if (!g_dgelsy) return -2;
    orc_monos mo;
    make_monos(dim, degree, &mo);
    const int k = mo.k;
    const double sqrt_lam = lam > 0 ? sqrt(lam) : 0.0;
    int64_t maxm = 1;
    for (int64_t i = 0; i < nt; i++)
        if (sup_off[i + 1] - sup_off[i] > maxm) maxm = sup_off[i + 1] - sup_off[i];
    const int extra = lam > 0 ? k : 0;
    const int lda = (int)maxm + extra;
    const int ldb = lda > k ? lda : k;
    const double rcond = DBL_EPSILON;
    int lwork;
    {
        int m_q = lda, n_q = k, nrhs = 1, rank = 0, info = 0, lw = -1;
        double wkopt = 0.0;
        double *A = calloc((size_t)lda * k, sizeof(double));
        double *b = calloc((size_t)ldb, sizeof(double));
        int jp[ORC_MAX_K] = {0};
        g_dgelsy(&m_q, &n_q, &nrhs, A, &lda, b, &ldb, jp, &rcond, &rank, &wkopt, &lw, &info);
        free(A);
        free(b);
        lwork = (int)wkopt + 16;
    }
    for (int64_t i = 0; i < nt * ncomp; i++) values[i] = NAN;
    for (int64_t i = 0; i < nt * ncomp * k; i++) coeffs[i] = NAN;

#pragma omp parallel num_threads(nthreads)
    {
        double *A = calloc((size_t)lda * k, sizeof(double));
        double *bvec = calloc((size_t)ldb, sizeof(double));
        double *work = calloc((size_t)lwork, sizeof(double));
        double spow[ORC_MAX_K], mono[ORC_MAX_K], u[ORC_MAX_DIM], dxv[ORC_MAX_DIM];
        int jpvt[ORC_MAX_K];
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < nt; i++) {
            int64_t lo = sup_off[i], hi = sup_off[i + 1], m = hi - lo;
            status[i] = 0;
            if (m == 0) {
                status[i] = 2;
                continue;
            }
            int any_pos = 0;
            for (int64_t j = lo; j < hi; j++)
                if (sup_w[j] > 0.0) {
                    any_pos = 1;
                    break;
                }
            if (!any_pos) {
                status[i] = 2;
                continue;
            }
            const double *t = targets + i * dim;
            double smax = 0.0;
            for (int64_t j = lo; j < hi; j++) {
                const double *p = src + sup_idx[j] * dim;
                double acc;
                for (int a = 0; a < dim; a++) dxv[a] = centering ? p[a] - t[a] : p[a];
                acc = dxv[0] * dxv[0];
                for (int a = 1; a < dim; a++) acc = acc + dxv[a] * dxv[a];
                if (acc > smax) smax = acc;
            }
            double s = sqrt(smax);
            if (s == 0.0) s = 1.0;
            for (int c = 0; c < k; c++) {
                int dg = mo.deg[c];
                spow[c] = dg == 0 ? 1.0 : (dg == 1 ? s : (dg == 2 ? s * s : s * s * s));
            }
            const int mrows = (int)m + extra;
            for (int comp = 0; comp < ncomp; comp++) {
                for (int64_t p = lo; p < hi; p++) {
                    int j = (int)(p - lo);
                    const double *q = src + sup_idx[p] * dim;
                    for (int a = 0; a < dim; a++) {
                        double dx = centering ? q[a] - t[a] : q[a];
                        u[a] = dx / s;
                    }
                    double w = sup_w[p];
                    eval_monos(&mo, u, mono);
                    A[j] = w;
                    for (int c = 1; c < k; c++) A[j + (int64_t)c * lda] = mono[c] * w;
                    bvec[j] = w * src_val[sup_idx[p] * ncomp + comp];
                }
                if (lam > 0) {
                    for (int col = 0; col < k; col++) {
                        for (int j = 0; j < k; j++) A[(m + j) + (int64_t)col * lda] = 0.0;
                        A[(m + col) + (int64_t)col * lda] = sqrt_lam / spow[col];
                        bvec[m + col] = 0.0;
                    }
                }
                for (int col = 0; col < k; col++) jpvt[col] = 0;
                int kk = k, nrhs = 1, rank = 0, info = 0, mr = mrows;
                g_dgelsy(&mr, &kk, &nrhs, A, &lda, bvec, &ldb, jpvt, &rcond, &rank, work,
                         &lwork, &info);
                if (info != 0 || (rank < k && lam == 0.0)) {
                    status[i] = 1;
                    continue;
                }
                double *cf = coeffs + (i * ncomp + comp) * k;
                for (int col = 0; col < k; col++) cf[col] = bvec[col] / spow[col];
                if (centering) {
                    values[i * ncomp + comp] = cf[0];
                } else {
                    eval_monos(&mo, t, mono);
                    double acc = 0.0;
                    for (int col = 0; col < k; col++) acc += cf[col] * mono[col];
                    values[i * ncomp + comp] = acc;
                }
            }
            if (status[i] != 0) {
                for (int comp = 0; comp < ncomp; comp++) {
                    values[i * ncomp + comp] = NAN;
                    for (int col = 0; col < k; col++)
                        coeffs[(i * ncomp + comp) * k + col] = NAN;
                }
            }
        }
        free(A);
        free(bvec);
        free(work);
    }
    return 0;
}

/* ------------------------------------------------------------ locate_batch
 * _ext.pyx:88-152: per point, its cell of the element grid (row-major
 * iy*nx+ix), the cell's candidate elements in stored (ascending id) order,
 * barycentric coordinates with the reference's operation order, first
 * element whose tol-halo contains the point; classification on the lowest
 * dimensional entity within tolerance (2 small -> vertex, 1 -> edge, else
 * element).  Outputs pre-filled by the caller (found 0, ids -1, bary NaN). */
void orc_locate_batch(const double *points, int64_t n, const double *tri_xy,
                      const int64_t *tri_verts, const int64_t *tri_edges,
                      const int64_t *vert_gid, const int64_t *tri_gid, const double *inv2a,
                      const double *epsfac, double gx0, double gy0, double gdx, double gdy,
                      int64_t nx, int64_t ny, const int64_t *cell_off,
                      const int64_t *cell_items, double tol, uint8_t *found, int64_t *elem,
                      int64_t *dim, int64_t *ent, double *bary) {
    const double inv_dx = 1.0 / gdx, inv_dy = 1.0 / gdy;
    for (int64_t i = 0; i < n; i++) {
        const double px = points[2 * i], py = points[2 * i + 1];
        const int64_t c = cell_of(py, gy0, inv_dy, ny) * nx + cell_of(px, gx0, inv_dx, nx);
        for (int64_t j = cell_off[c]; j < cell_off[c + 1]; j++) {
            const int64_t t = cell_items[j];
            const double *P = tri_xy + 6 * t;
            const double b0 = ((P[2] - px) * (P[5] - py) - (P[3] - py) * (P[4] - px)) * inv2a[t];
            const double b1 = ((P[4] - px) * (P[1] - py) - (P[5] - py) * (P[0] - px)) * inv2a[t];
            const double b2 = 1.0 - b0 - b1;
            const double e0 = tol * epsfac[3 * t], e1 = tol * epsfac[3 * t + 1],
                         e2 = tol * epsfac[3 * t + 2];
            if (b0 >= -e0 && b1 >= -e1 && b2 >= -e2) {
                found[i] = 1;
                elem[i] = t;
                bary[3 * i] = b0;
                bary[3 * i + 1] = b1;
                bary[3 * i + 2] = b2;
                const int s0 = b0 <= e0, s1 = b1 <= e1, s2 = b2 <= e2;
                const int nsmall = s0 + s1 + s2;
                if (nsmall == 2) {
                    const int v = !s0 ? 0 : (!s1 ? 1 : 2);
                    dim[i] = 0;
                    ent[i] = vert_gid[tri_verts[3 * t + v]];
                } else if (nsmall == 1) {
                    const int k = s0 ? 0 : (s1 ? 1 : 2);
                    dim[i] = 1;
                    ent[i] = tri_edges[3 * t + k];
                } else {
                    dim[i] = 2;
                    ent[i] = tri_gid[t];
                }
                break;
            }
        }
    }
}
