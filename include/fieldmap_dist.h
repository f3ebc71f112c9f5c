/*
 * fieldmap_dist.h -- multi-GPU delivery of the target field (libfieldmap.so).
 *
 * targets sharded across the GPUs of one node, the source
 * cloud replicated; the full target field is delivered to every rank while
 * the operator is still being built.  The reference's sharded caller is
 * rendezvous._coupled_pointwise (rendezvous.py:452-495), which routes every
 * target's value back through host messages; here the values move GPU to GPU
 * over NVLink as copy-engine transfers into peer memory (CUDA IPC).
 *
 * Allocation/IPC helpers are the only calls of the library that allocate
 * device memory (the receive buffers peers write into).
 */
#ifndef FIELDMAP_DIST_H
#define FIELDMAP_DIST_H

#include <stddef.h>
#include <stdint.h>

#include "fieldmap.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FM_MAX_PEERS 63

int fm_ipc_handle_size(void);
int fm_device_alloc(size_t bytes, void **ptr);
int fm_device_free(void *ptr);
/* handle: fm_ipc_handle_size() bytes (cudaIpcMemHandle_t) of the allocation
 * starting at `base` (an fm_device_alloc pointer). */
int fm_ipc_export(void *base, void *handle);
int fm_ipc_open(const void *handle, void **ptr);
int fm_ipc_close(void *ptr);

/* Operator build + apply of one rank's targets in nblocks target blocks
 * (perm from fm_target_order_blocked(..., nblocks, ...); the positions of
 * block b are [nt*b/nblocks, nt*(b+1)/nblocks)), with each block's rows of Y
 * (nt x ncomp, this rank's slot of the receive buffer) pushed into every
 * peer's copy of that slot (peer_Y[q], IPC pointers) on stream `comm` as soon
 * as the block is applied.  Same arguments as fm_build_operator (lists from
 * fm_select_supports / fm_offsets_ordered, its host bucket_count naming the
 * non-empty buckets) plus scratch: bucket_list (FM_NBUCKETS x max block),
 * bucket_count (device int32[FM_NBUCKETS]), stats (device int32[2*nblocks]:
 * per block fm_build_operator's fit stats).  Completion on the peers is the
 * caller's to establish (e.g. a collective on `comm` after this call). */
int fm_build_apply_blocks(const fm_grid *grid, const int32_t *cell_start,
                          const double *sorted_pts, const int32_t *sorted_ids,
                          const double *targets, int64_t nt, const int32_t *perm,
                          const fm_select *sel, const double *radii, const fm_lists *lists,
                          const int64_t *offsets, int32_t max_count, const fm_rbf *rbf,
                          const fm_fit *fit, int32_t *col, double *val, uint8_t *status,
                          int32_t *bucket_list, int32_t *bucket_count, int32_t *stats,
                          int32_t nblocks, const double *X, int32_t ncomp, double *Y,
                          int32_t npeers, void *const *peer_Y, fm_stream_t stream,
                          fm_stream_t comm);

/* Push `bytes` at device `src` (this GPU) to offset dst_offset of every
 * peer buffer peer_bases[q] (IPC pointers): one copy-engine transfer per peer
 * on its own stream, after the work already queued on `stream`; `comm` waits
 * for all of them (close the exchange with a collective on `comm`). */
int fm_push_rows(const void *src, size_t bytes, size_t dst_offset, int32_t npeers,
                 void *const *peer_bases, fm_stream_t stream, fm_stream_t comm);

#ifdef __cplusplus
}
#endif
#endif /* FIELDMAP_DIST_H */
