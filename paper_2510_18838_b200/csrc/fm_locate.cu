// fm_locate.cu -- element point localization with topological
// classification (locate_batch, _ext.pyx:88-152; §8(f) rank 1).
//
// One thread per query point: its cell of the element grid (row-major
// iy*nx + ix, _cell_of of _ext.pyx:78-85), the cell's candidate elements in
// stored (ascending id) order, barycentric coordinates with the reference's
// operation order and rounding (no contraction: _rn intrinsics), the first
// element whose tol-halo contains the point wins; the point is classified on
// the lowest-dimensional entity within tolerance.  Bitwise equal to the
// reference.  The loop is a short data-dependent scan (a few candidates per
// cell), latency bound: points are independent, so the grid is sized for
// many resident warps rather than tiled.
#include <algorithm>

#include "fm_common.cuh"

namespace fm {

__global__ void __launch_bounds__(256)
    k_locate(const double *__restrict__ points, int64_t n, const double *__restrict__ tri_xy,
             const int64_t *__restrict__ tri_verts, const int64_t *__restrict__ tri_edges,
             const int64_t *__restrict__ vert_gid, const int64_t *__restrict__ tri_gid,
             const double *__restrict__ inv2a, const double *__restrict__ epsfac, double gx0,
             double gy0, double inv_dx, double inv_dy, int64_t nx, int64_t ny,
             const int64_t *__restrict__ cell_off, const int64_t *__restrict__ cell_items,
             double tol, uint8_t *__restrict__ found, int64_t *__restrict__ elem,
             int64_t *__restrict__ dim, int64_t *__restrict__ ent, double *__restrict__ bary) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double px = points[2 * i], py = points[2 * i + 1];
        const int64_t c = cell_of(py, gy0, inv_dy, ny) * nx + cell_of(px, gx0, inv_dx, nx);
        uint8_t f = 0;
        int64_t el = -1, dm = -1, en = -1;
        double b0 = NAN, b1 = NAN, b2 = NAN;
        const int64_t j1 = __ldg(cell_off + c + 1);
        for (int64_t j = __ldg(cell_off + c); j < j1; j++) {
            const int64_t t = __ldg(cell_items + j);
            const double *P = tri_xy + 6 * t;
            const double x0 = __ldg(P), y0 = __ldg(P + 1), x1 = __ldg(P + 2), y1 = __ldg(P + 3),
                         x2 = __ldg(P + 4), y2 = __ldg(P + 5), ia = __ldg(inv2a + t);
            const double c0 = mul_rn(sub_rn(mul_rn(sub_rn(x1, px), sub_rn(y2, py)),
                                            mul_rn(sub_rn(y1, py), sub_rn(x2, px))),
                                     ia);
            const double c1 = mul_rn(sub_rn(mul_rn(sub_rn(x2, px), sub_rn(y0, py)),
                                            mul_rn(sub_rn(y2, py), sub_rn(x0, px))),
                                     ia);
            const double c2 = sub_rn(sub_rn(1.0, c0), c1);
            const double e0 = mul_rn(tol, __ldg(epsfac + 3 * t));
            const double e1 = mul_rn(tol, __ldg(epsfac + 3 * t + 1));
            const double e2 = mul_rn(tol, __ldg(epsfac + 3 * t + 2));
            if (c0 >= -e0 && c1 >= -e1 && c2 >= -e2) {
                f = 1;
                el = t;
                b0 = c0;
                b1 = c1;
                b2 = c2;
                const int s0 = c0 <= e0, s1 = c1 <= e1, s2 = c2 <= e2;
                const int nsmall = s0 + s1 + s2;
                if (nsmall == 2) {
                    const int v = !s0 ? 0 : (!s1 ? 1 : 2);
                    dm = 0;
                    en = vert_gid[tri_verts[3 * t + v]];
                } else if (nsmall == 1) {
                    const int k = s0 ? 0 : (s1 ? 1 : 2);
                    dm = 1;
                    en = tri_edges[3 * t + k];
                } else {
                    dm = 2;
                    en = tri_gid[t];
                }
                break;
            }
        }
        found[i] = f;
        elem[i] = el;
        dim[i] = dm;
        ent[i] = en;
        bary[3 * i] = b0;
        bary[3 * i + 1] = b1;
        bary[3 * i + 2] = b2;
    }
}

}  // namespace fm

using namespace fm;

extern "C" int fm_locate_batch(const double *points, int64_t n, const double *tri_xy,
                               const int64_t *tri_verts, const int64_t *tri_edges,
                               const int64_t *vert_gid, const int64_t *tri_gid,
                               const double *inv2a, const double *epsfac, double gx0, double gy0,
                               double gdx, double gdy, int64_t nx, int64_t ny,
                               const int64_t *cell_off, const int64_t *cell_items, double tol,
                               uint8_t *found, int64_t *elem, int64_t *dim, int64_t *ent,
                               double *bary, fm_stream_t stream) {
    if (n < 0 || nx < 1 || ny < 1 || !(tol >= 0.0)) return FM_ERR_ARG;
    if (n == 0) return FM_OK;
    if (!points || !tri_xy || !tri_verts || !tri_edges || !vert_gid || !tri_gid || !inv2a ||
        !epsfac || !cell_off || !cell_items || !found || !elem || !dim || !ent || !bary)
        return FM_ERR_ARG;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, (int64_t)kSMs * 8);
    // 1/gdx as the reference computes it (_ext.pyx:106-107): IEEE division
    k_locate<<<blocks, threads, 0, (cudaStream_t)stream>>>(
        points, n, tri_xy, tri_verts, tri_edges, vert_gid, tri_gid, inv2a, epsfac, gx0, gy0,
        1.0 / gdx, 1.0 / gdy, nx, ny, cell_off, cell_items, tol, found, elem, dim, ent, bary);
    FM_CHECK_LAUNCH();
    return FM_OK;
}
