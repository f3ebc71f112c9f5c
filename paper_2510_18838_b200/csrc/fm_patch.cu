// fm_patch.cu -- element-patch support selection:
// the reference's per-target Python BFS (_PatchTopology.patch_dofs,
// pointwise.py:212-230) as one thread per target.
//
// The patch is the set of elements within `layers` hops of the seed element,
// so the BFS visiting order does not matter: each thread grows its element
// list layer by layer (frontier = the elements appended in the previous
// layer, membership by a linear scan of the short list), sorts it, and either
// emits it (centroid dofs) or merges the elements' three vertices into a
// sorted, de-duplicated list (vertex dofs, np.unique of pointwise.py:229).
// The lists live in per-thread local memory (L1-resident: a 1-layer patch is
// ~13 elements / ~12 vertices); the work is a short dependent scan, latency
// bound, so the grid is sized for many resident warps.  Two passes (count,
// then fill at the scanned offsets) recompute the patch instead of staging
// it, which keeps the output exactly nnz long.
#include <algorithm>

#include "../../include/fieldmap_patch.h"
#include "fm_common.cuh"

namespace fm {

// Patch of target i (elements within `layers` hops of its seed, then the
// sorted distinct dofs) in caller-provided element / dof lists of capacity
// maxe / maxd: per-thread local arrays (k_patch), or global scratch for the
// few targets whose patch exceeds those (k_patch_big).
template <bool FILL>
__device__ __forceinline__ void patch_one(int64_t i, const int64_t *__restrict__ seed,
                                          const int32_t *__restrict__ adj_off,
                                          const int32_t *__restrict__ adj,
                                          const int32_t *__restrict__ tris, int32_t layers,
                                          int32_t centroids, int64_t ne, int32_t *el, int maxe,
                                          int32_t *dof, int maxd, int64_t *__restrict__ counts,
                                          const int64_t *__restrict__ off,
                                          int64_t *__restrict__ idx) {
    int n = 1;
    bool overflow = false;
    const int64_t sd = __ldg(seed + i);
    if (sd < 0 || sd >= ne) {  // not located (-1) or not an element: no patch
        if (!FILL) counts[i] = -2;
        return;
    }
    el[0] = (int32_t)sd;
    int fs = 0, fe = 1;  // frontier [fs, fe)
    for (int layer = 0; layer < layers && !overflow && fs < fe; layer++) {
        for (int f = fs; f < fe && !overflow; f++) {
            const int32_t t = el[f];
            const int32_t a1 = __ldg(adj_off + t + 1);
            for (int32_t a = __ldg(adj_off + t); a < a1; a++) {
                const int32_t nb = __ldg(adj + a);
                bool seen = false;
                for (int q = 0; q < n; q++) seen |= (el[q] == nb);
                if (seen) continue;
                if (n == maxe) {
                    overflow = true;
                    break;
                }
                el[n++] = nb;
            }
        }
        fs = fe;
        fe = n;
    }
    if (overflow) {
        if (!FILL) counts[i] = -1;
        return;
    }
    // sorted(seen) (pointwise.py:226): insertion sort of a short list
    for (int a = 1; a < n; a++) {
        const int32_t v = el[a];
        int b = a - 1;
        while (b >= 0 && el[b] > v) {
            el[b + 1] = el[b];
            b--;
        }
        el[b + 1] = v;
    }
    if (centroids) {
        if (FILL) {
            int64_t *o = idx + off[i];
            for (int a = 0; a < n; a++) o[a] = el[a];
        } else {
            counts[i] = n;
        }
        return;
    }
    // np.unique(tris[elems]) (pointwise.py:229): sorted insert with dedup
    int m = 0;
    for (int a = 0; a < n && !overflow; a++) {
        const int32_t *tv = tris + 3 * (int64_t)el[a];
        for (int c = 0; c < 3; c++) {
            const int32_t v = __ldg(tv + c);
            int b = m - 1;
            while (b >= 0 && dof[b] > v) b--;
            if (b >= 0 && dof[b] == v) continue;
            if (m == maxd) {
                overflow = true;
                break;
            }
            for (int q = m; q > b + 1; q--) dof[q] = dof[q - 1];
            dof[b + 1] = v;
            m++;
        }
    }
    if (FILL) {
        if (!overflow) {
            int64_t *o = idx + off[i];
            for (int a = 0; a < m; a++) o[a] = dof[a];
        }
    } else {
        counts[i] = overflow ? -1 : m;
    }
}

template <bool FILL>
__global__ void __launch_bounds__(128)
    k_patch(const int64_t *__restrict__ seed, int64_t nt, const int64_t *__restrict__ order,
            const int32_t *__restrict__ adj_off, const int32_t *__restrict__ adj,
            const int32_t *__restrict__ tris, int32_t layers,
            int32_t centroids, int64_t ne, int64_t *__restrict__ counts,
            const int64_t *__restrict__ off, int64_t *__restrict__ idx) {
    int32_t el[FM_PATCH_MAX_ELEMS];
    int32_t dof[FM_PATCH_MAX_DOFS];
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nt;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = order ? __ldg(order + p) : p;
        patch_one<FILL>(i, seed, adj_off, adj, tris, layers, centroids, ne, el,
                        FM_PATCH_MAX_ELEMS, dof, FM_PATCH_MAX_DOFS, counts, off, idx);
    }
}

// targets list[0..nlist) with patches beyond the local bounds: element / dof
// lists in global scratch (maxe + maxd int32 per target slot)
template <bool FILL>
__global__ void __launch_bounds__(128)
    k_patch_big(const int64_t *__restrict__ seed, const int64_t *__restrict__ list, int64_t nlist,
                const int32_t *__restrict__ adj_off, const int32_t *__restrict__ adj,
                const int32_t *__restrict__ tris, int32_t layers, int32_t centroids, int64_t ne,
                int32_t maxe, int32_t maxd, int32_t *__restrict__ scratch,
                int64_t *__restrict__ counts, const int64_t *__restrict__ off,
                int64_t *__restrict__ idx) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int32_t *el = scratch + slot * (int64_t)(maxe + maxd);
    for (int64_t p = slot; p < nlist; p += stride)
        patch_one<FILL>(list[p], seed, adj_off, adj, tris, layers, centroids, ne, el, maxe,
                        el + maxe, maxd, counts, off, idx);
}

static int launch_patch(bool fill, const int64_t *seed, int64_t nt, const int64_t *order,
                        const int32_t *adj_off, const int32_t *adj, const int32_t *tris,
                        int64_t ne, int32_t layers,
                        int32_t centroids, int64_t *counts, const int64_t *off, int64_t *idx,
                        cudaStream_t stream) {
    if (nt < 0 || ne < 1 || layers < 1 || ne > INT32_MAX) return FM_ERR_ARG;
    if (nt == 0) return FM_OK;
    if (!seed || !adj_off || !adj || (!centroids && !tris)) return FM_ERR_ARG;
    if (fill ? (!off || !idx) : !counts) return FM_ERR_ARG;
    const int threads = 128;
    const int blocks = (int)std::min<int64_t>((nt + threads - 1) / threads, (int64_t)kSMs * 16);
    if (fill)
        k_patch<true><<<blocks, threads, 0, stream>>>(seed, nt, order, adj_off, adj, tris,
                                                      layers, centroids, ne, nullptr, off, idx);
    else
        k_patch<false><<<blocks, threads, 0, stream>>>(seed, nt, order, adj_off, adj, tris,
                                                       layers, centroids, ne, counts, nullptr,
                                                       nullptr);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

}  // namespace fm

extern "C" int fm_patch_count(const int64_t *seed, int64_t nt, const int64_t *order,
                              const int32_t *adj_off, const int32_t *adj, const int32_t *tris,
                              int64_t ne, int32_t layers, int32_t centroids, int64_t *counts,
                              fm_stream_t stream) {
    return fm::launch_patch(false, seed, nt, order, adj_off, adj, tris, ne, layers, centroids, counts,
                            nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int fm_patch_fill(const int64_t *seed, int64_t nt, const int64_t *order,
                             const int32_t *adj_off, const int32_t *adj, const int32_t *tris,
                             int64_t ne, int32_t layers, int32_t centroids, const int64_t *off,
                             int64_t *idx, fm_stream_t stream) {
    return fm::launch_patch(true, seed, nt, order, adj_off, adj, tris, ne, layers, centroids, nullptr,
                            off, idx, (cudaStream_t)stream);
}

// scratch slots = threads launched (a multiple of 128, at most 148 x 128)
static int64_t patch_big_slots(int64_t nlist) {
    const int64_t n = nlist < (int64_t)fm::kSMs * 128 ? nlist : (int64_t)fm::kSMs * 128;
    return ((n > 0 ? n : 1) + 127) / 128 * 128;
}

extern "C" size_t fm_patch_big_workspace(int64_t nlist, int32_t max_elems, int32_t max_dofs) {
    return (size_t)patch_big_slots(nlist) * (size_t)(max_elems + max_dofs) * sizeof(int32_t);
}

static int launch_patch_big(bool fill, const int64_t *seed, const int64_t *list, int64_t nlist,
                            const int32_t *adj_off, const int32_t *adj, const int32_t *tris,
                            int64_t ne, int32_t layers, int32_t centroids, int32_t max_elems,
                            int32_t max_dofs, void *workspace, size_t workspace_bytes,
                            int64_t *counts, const int64_t *off, int64_t *idx,
                            cudaStream_t st) {
    if (nlist < 0 || ne < 1 || layers < 1 || max_elems < 1 || max_dofs < 1 || !seed || !list ||
        !adj_off || !adj || (!centroids && !tris) || (fill ? (!off || !idx) : !counts))
        return FM_ERR_ARG;
    if (nlist == 0) return FM_OK;
    if (workspace_bytes < fm_patch_big_workspace(nlist, max_elems, max_dofs))
        return FM_ERR_WORKSPACE;
    const int blocks = (int)(patch_big_slots(nlist) / 128);  // slot = global thread index
    int32_t *scratch = reinterpret_cast<int32_t *>(workspace);
    if (fill)
        fm::k_patch_big<true><<<blocks, 128, 0, st>>>(seed, list, nlist, adj_off, adj, tris, layers,
                                                      centroids, ne, max_elems, max_dofs, scratch,
                                                      nullptr, off, idx);
    else
        fm::k_patch_big<false><<<blocks, 128, 0, st>>>(seed, list, nlist, adj_off, adj, tris,
                                                       layers, centroids, ne, max_elems, max_dofs,
                                                       scratch, counts, nullptr, nullptr);
    if (cudaPeekAtLastError() != cudaSuccess) {
        (void)cudaGetLastError();
        return FM_ERR_CUDA;
    }
    return FM_OK;
}

extern "C" int fm_patch_count_big(const int64_t *seed, const int64_t *list, int64_t nlist,
                                  const int32_t *adj_off, const int32_t *adj,
                                  const int32_t *tris, int64_t ne, int32_t layers,
                                  int32_t centroids, int32_t max_elems, int32_t max_dofs,
                                  void *workspace, size_t workspace_bytes, int64_t *counts,
                                  fm_stream_t stream) {
    return launch_patch_big(false, seed, list, nlist, adj_off, adj, tris, ne, layers, centroids,
                            max_elems, max_dofs, workspace, workspace_bytes, counts, nullptr,
                            nullptr, (cudaStream_t)stream);
}

extern "C" int fm_patch_fill_big(const int64_t *seed, const int64_t *list, int64_t nlist,
                                 const int32_t *adj_off, const int32_t *adj, const int32_t *tris,
                                 int64_t ne, int32_t layers, int32_t centroids, int32_t max_elems,
                                 int32_t max_dofs, void *workspace, size_t workspace_bytes,
                                 const int64_t *off, int64_t *idx, fm_stream_t stream) {
    return launch_patch_big(true, seed, list, nlist, adj_off, adj, tris, ne, layers, centroids,
                            max_elems, max_dofs, workspace, workspace_bytes, nullptr, off, idx,
                            (cudaStream_t)stream);
}
