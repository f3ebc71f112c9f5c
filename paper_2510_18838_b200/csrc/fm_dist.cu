// fm_dist.cu -- §8(e): the target field of a target-sharded transfer
// delivered to every rank over NVLink peer memory, overlapped with the build.
//
// The reference shards targets across ranks with a replicated source cloud
// (rendezvous.py:452-495; per-target work is independent and bitwise
// chunk-invariant).  When every rank needs the full target field, the B200
// path does not append an all-gather after the compute: each rank builds its
// operator rows block by block (fm_target_order_blocked makes a target block
// a contiguous range of processing positions), applies each block as soon as
// it is built, and pushes the block's rows straight into every peer's
// receive buffer with copy-engine transfers over NVLink (CUDA IPC peer
// pointers) on a second stream -- no SMs spent on communication, and block
// b's transfer runs under block b+1's build.  The host loop issuing all of
// it is here, in C++, so the per-block launches cost no interpreter time.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "../../include/fieldmap.h"
#include "../../include/fieldmap_dist.h"

namespace {
// one stream per peer: the pushes of a block to different peers run on
// different copy engines concurrently (one stream would serialise them)
struct PeerStreams {
    cudaStream_t s[FM_MAX_PEERS];
    cudaEvent_t join[FM_MAX_PEERS];
    int n = 0;
};

PeerStreams *peer_streams(int npeers) {
    static PeerStreams pool[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    PeerStreams &p = pool[dev];
    while (p.n < npeers) {
        if (cudaStreamCreateWithFlags(&p.s[p.n], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&p.join[p.n], cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
        p.n++;
    }
    return &p;
}
}  // namespace

extern "C" {

int fm_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int fm_device_alloc(size_t bytes, void **ptr) {
    if (!ptr) return FM_ERR_ARG;
    *ptr = nullptr;
    return cudaMalloc(ptr, bytes ? bytes : 1) == cudaSuccess ? FM_OK : FM_ERR_CUDA;
}

int fm_device_free(void *ptr) { return cudaFree(ptr) == cudaSuccess ? FM_OK : FM_ERR_CUDA; }

int fm_ipc_export(void *base, void *handle) {
    if (!base || !handle) return FM_ERR_ARG;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return FM_ERR_CUDA;
    memcpy(handle, &h, sizeof h);
    return FM_OK;
}

int fm_ipc_open(const void *handle, void **ptr) {
    if (!handle || !ptr) return FM_ERR_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess
               ? FM_OK
               : FM_ERR_CUDA;
}

int fm_ipc_close(void *ptr) {
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? FM_OK : FM_ERR_CUDA;
}

int fm_build_apply_blocks(const fm_grid *grid, const int32_t *cell_start,
                          const double *sorted_pts, const int32_t *sorted_ids,
                          const double *targets, int64_t nt, const int32_t *perm,
                          const fm_select *sel, const double *radii, const fm_lists *lists,
                          const int64_t *offsets, int32_t max_count, const fm_rbf *rbf,
                          const fm_fit *fit, int32_t *col, double *val, uint8_t *status,
                          int32_t *bucket_list, int32_t *bucket_count, int32_t *stats,
                          int32_t nblocks, const double *X, int32_t ncomp, double *Y,
                          int32_t npeers, void *const *peer_Y, fm_stream_t stream,
                          fm_stream_t comm) {
    if (!lists || !bucket_list || !bucket_count || !stats || nblocks < 1 || npeers < 0 ||
        npeers > FM_MAX_PEERS || (npeers > 0 && (!peer_Y || !comm)) || ncomp < 1 || nt < 0)
        return FM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream, cs = (cudaStream_t)comm;
    int64_t stride = 0;
    for (int b = 0; b < nblocks; b++) {
        const int64_t w = nt * (b + 1) / nblocks - nt * b / nblocks;
        if (w > stride) stride = w;
    }
    int mask = 0;
    for (int b = 0; b < FM_NBUCKETS; b++)
        if (lists->bucket_count[b] > 0) mask |= 1 << b;
    std::vector<cudaEvent_t> evs;
    int rc = FM_OK;
    for (int b = 0; b < nblocks && rc == FM_OK; b++) {
        const int64_t lo = nt * b / nblocks, hi = nt * (b + 1) / nblocks;
        if (hi == lo) continue;
        rc = fm_bucket_positions(lists->counts, perm, lo, hi, lists->slot_cap, bucket_list,
                                 stride, bucket_count, stream);
        if (rc) break;
        fm_lists L = *lists;
        L.bucket_list = bucket_list;
        L.bucket_stride = stride;
        L.bucket_count_dev = bucket_count;
        L.bucket_mask = mask;
        L.skip_overflow = b > 0;  // overflowing supports: all rebuilt with block 0
        rc = fm_build_operator(grid, cell_start, sorted_pts, sorted_ids, targets, nt, perm, sel,
                               radii, &L, offsets, max_count, rbf, fit, col, val, status,
                               stats + 2 * b, stream);
        if (rc) break;
        rc = fm_apply(hi - lo, offsets + lo, col, val, perm + lo, X, ncomp, Y, stream);
        if (rc) break;
        if (npeers > 0) {
            cudaEvent_t ev;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
                rc = FM_ERR_CUDA;
                break;
            }
            evs.push_back(ev);
            cudaEventRecord(ev, st);
            PeerStreams *ps = peer_streams(npeers);
            const size_t bytes = (size_t)(hi - lo) * ncomp * sizeof(double);
            for (int q = 0; q < npeers; q++) {
                cudaStream_t sq = ps ? ps->s[q] : cs;
                cudaStreamWaitEvent(sq, ev, 0);
                double *dst = reinterpret_cast<double *>(peer_Y[q]) + lo * ncomp;
                if (cudaMemcpyAsync(dst, Y + lo * ncomp, bytes, cudaMemcpyDeviceToDevice, sq) !=
                    cudaSuccess) {
                    rc = FM_ERR_CUDA;
                    break;
                }
                if (ps) {
                    cudaEventRecord(ps->join[q], sq);
                    cudaStreamWaitEvent(cs, ps->join[q], 0);
                }
            }
        }
    }
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);  // released once the streams pass them
    return rc;
}

int fm_push_rows(const void *src, size_t bytes, size_t dst_offset, int32_t npeers,
                 void *const *peer_bases, fm_stream_t stream, fm_stream_t comm) {
    if (npeers < 0 || npeers > FM_MAX_PEERS || (npeers > 0 && (!src || !peer_bases || !comm)))
        return FM_ERR_ARG;
    if (npeers == 0 || bytes == 0) return FM_OK;
    cudaStream_t st = (cudaStream_t)stream, cs = (cudaStream_t)comm;
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return FM_ERR_CUDA;
    cudaEventRecord(ev, st);
    PeerStreams *ps = peer_streams(npeers);
    int rc = FM_OK;
    for (int q = 0; q < npeers && rc == FM_OK; q++) {
        cudaStream_t sq = ps ? ps->s[q] : cs;
        cudaStreamWaitEvent(sq, ev, 0);
        char *dst = reinterpret_cast<char *>(peer_bases[q]) + dst_offset;
        if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, sq) != cudaSuccess)
            rc = FM_ERR_CUDA;
        if (ps) {
            cudaEventRecord(ps->join[q], sq);
            cudaStreamWaitEvent(cs, ps->join[q], 0);
        }
    }
    cudaEventDestroy(ev);
    return rc;
}

}  // extern "C"
