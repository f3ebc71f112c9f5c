/* fieldmap_patch.h -- element-patch support selection.
 *
 * Replaces the per-target Python BFS of the reference's ElementPatch branch:
 * `_PatchTopology.neighbors` / `patch_dofs` (pointwise.py:190-230) as called
 * from `_select_batch` (pointwise.py:271-296).  Same conventions as
 * fieldmap.h: device pointers, sizes and a stream; FM_OK or a negative
 * FM_ERR_* code; no global state.
 */
#ifndef FIELDMAP_PATCH_H
#define FIELDMAP_PATCH_H

#include "fieldmap.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Largest patch one target can hold: elements reached within `layers`
 * edge-adjacency hops, and distinct vertex dofs of those elements.  A larger
 * patch reports count -1 for that target (Python: FieldmapError). */
#define FM_PATCH_MAX_ELEMS 128
#define FM_PATCH_MAX_DOFS 256

/* Per target i with containing element seed[i] (locate_batch's `elem`,
 * int64, >= 0): the elements within `layers` hops over the element
 * adjacency CSR (adj_off int32 (ne+1), adj int32 -- each interior edge
 * contributes both directions, pointwise.py:195-200), sorted ascending
 * (pointwise.py:226); dofs = those element ids when `centroids` != 0, else
 * the sorted distinct vertex ids of tris[elems] (tris int32 (ne, 3),
 * pointwise.py:229).  The topology is int32 (the Python shim converts the
 * reference's int64 arrays once) so it stays L2-resident.  `order` (int64
 * permutation of 0..nt-1, or NULL) is the processing order -- e.g. targets
 * sorted by seed element, for L2 locality; outputs stay at each target's own
 * position, so results never depend on it.
 *   fm_patch_count: counts int64 (nt); -1 when the patch exceeds the bounds
 *                   above, -2 when seed[i] is not an element id (e.g. -1, the
 *                   not-found value of fm_locate_batch).  A caller must stop on
 *                   any negative count (Python raises FieldmapError /
 *                   InsufficientSourcesError) before scanning the counts.
 *   fm_patch_fill:  idx int64 at off[i] .. off[i+1] (off = exclusive scan of
 *                   the counts, int64 (nt+1)); targets with a negative count
 *                   write nothing.  Bitwise equal to the reference. */
int fm_patch_count(const int64_t *seed, int64_t nt, const int64_t *order, const int32_t *adj_off,
                   const int32_t *adj, const int32_t *tris, int64_t ne, int32_t layers,
                   int32_t centroids, int64_t *counts, fm_stream_t stream);
int fm_patch_fill(const int64_t *seed, int64_t nt, const int64_t *order, const int32_t *adj_off,
                  const int32_t *adj, const int32_t *tris, int64_t ne, int32_t layers,
                  int32_t centroids, const int64_t *off, int64_t *idx, fm_stream_t stream);

/* Targets whose patch exceeds the bounds above (count -1) have no size limit
 * the reference lacks: the same patch with element / dof lists of capacity
 * max_elems / max_dofs in caller scratch (fm_patch_big_workspace bytes), for
 * the targets list[0..nlist) only; counts[list[p]] is overwritten (still -1
 * if even these capacities are exceeded), fill writes at off[list[p]]. */
size_t fm_patch_big_workspace(int64_t nlist, int32_t max_elems, int32_t max_dofs);
int fm_patch_count_big(const int64_t *seed, const int64_t *list, int64_t nlist,
                       const int32_t *adj_off, const int32_t *adj, const int32_t *tris, int64_t ne,
                       int32_t layers, int32_t centroids, int32_t max_elems, int32_t max_dofs,
                       void *workspace, size_t workspace_bytes, int64_t *counts,
                       fm_stream_t stream);
int fm_patch_fill_big(const int64_t *seed, const int64_t *list, int64_t nlist,
                      const int32_t *adj_off, const int32_t *adj, const int32_t *tris, int64_t ne,
                      int32_t layers, int32_t centroids, int32_t max_elems, int32_t max_dofs,
                      void *workspace, size_t workspace_bytes, const int64_t *off, int64_t *idx,
                      fm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FIELDMAP_PATCH_H */
