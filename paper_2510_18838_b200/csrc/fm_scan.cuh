// fm_scan.cuh -- exclusive prefix sum in ONE pass (decoupled look-back).
//
// out[0] = 0, out[i+1] = out[i] + in[i] for i < n  (n+1 outputs).
// Used for the grid's cell_start (locate.py:82-84 `add.at` + `cumsum`), the
// target order, and the support CSR offsets (_ext.pyx:220, 272).
//
// Tiles of kScanTile elements are claimed in order through an atomic tile
// counter; each tile publishes its aggregate, then looks back over its
// predecessors (32 at a time, one warp) for the running prefix and publishes
// the inclusive value.  Status words pack a 2-bit flag with a 62-bit value,
// so one 64-bit store publishes both.  One memset + one launch per scan.
#pragma once

#include "fm_common.cuh"

namespace fm {

// Large tiles: a tile's look-back walks its predecessors 32 per round until
// it meets an inclusive prefix, and the inclusive frontier advances ~32 tiles
// per round, so the scan's critical path grows with the tile COUNT (2048-
// element tiles: 489 tiles and ~14 us for 1M elements).
constexpr int kScanThreads = 512;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

#define FM_SCAN_AGG (1ull << 62)
#define FM_SCAN_INCL (2ull << 62)
#define FM_SCAN_VAL_MASK ((1ull << 62) - 1)

inline int64_t scan_blocks(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
// status words (one per tile) + the tile counter
inline size_t scan_workspace_bytes(int64_t n) {
    return (size_t)(scan_blocks(n) + 1) * sizeof(unsigned long long) + 256;
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(
    const TIn *__restrict__ in, int64_t n, TOut *__restrict__ out,
    unsigned long long *__restrict__ status, unsigned int *__restrict__ tile_counter) {
    __shared__ long long warp_tot[kScanThreads / 32];
    __shared__ long long s_prefix;
    __shared__ unsigned int s_tile;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    long long v[kScanItems];
    long long local = 0;
    // full tiles of a 16-byte aligned int32 input: 16-byte loads
    const bool vec = sizeof(TIn) == 4 && (tile + 1) * kScanTile <= n &&
                     ((uintptr_t)in & 15) == 0;
    if (vec) {
#pragma unroll
        for (int k = 0; k < kScanItems; k += 4) {
            const int4 q = __ldg(reinterpret_cast<const int4 *>(in + base + k));
            v[k] = q.x;
            v[k + 1] = q.y;
            v[k + 2] = q.z;
            v[k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const int64_t i = base + k;
            v[k] = i < n ? (long long)in[i] : 0;
        }
    }
#pragma unroll
    for (int k = 0; k < kScanItems; k++) local += v[k];
    long long x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(FM_FULL_MASK, x, o);
        if (lane >= o) x += u;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        long long t = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(FM_FULL_MASK, t, o);
            if (lane >= o) t += u;
        }
        if (lane < kScanThreads / 32) warp_tot[lane] = t;
        const long long agg = __shfl_sync(FM_FULL_MASK, t, kScanThreads / 32 - 1);
        volatile unsigned long long *vs = status;
        if (tile == 0) {
            if (lane == 0) {
                vs[0] = FM_SCAN_INCL | (unsigned long long)agg;
                s_prefix = 0;
            }
        } else {
            if (lane == 0) vs[tile] = FM_SCAN_AGG | (unsigned long long)agg;
            // look back: lane l inspects tile idx - l
            long long prefix = 0;
            int64_t idx = tile - 1;
            for (;;) {
                const int64_t j = idx - lane;
                unsigned long long w = j >= 0 ? vs[j] : FM_SCAN_INCL;  // before tile 0: prefix 0
                while (__any_sync(FM_FULL_MASK, (w >> 62) == 0)) {
                    if ((w >> 62) == 0) w = vs[j];
                }
                const unsigned incl = __ballot_sync(FM_FULL_MASK, (w >> 62) == 2);
                const int stop = incl ? __ffs(incl) - 1 : 32;  // nearest inclusive predecessor
                long long mine = (lane <= stop) ? (long long)(w & FM_SCAN_VAL_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(FM_FULL_MASK, mine, o);
                prefix += mine;
                if (incl) break;
                idx -= 32;
            }
            if (lane == 0) {
                vs[tile] = FM_SCAN_INCL | (unsigned long long)(prefix + agg);
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    long long run = s_prefix + (x - local) + (wid > 0 ? warp_tot[wid - 1] : 0);
    if (vec && ((uintptr_t)out & 15) == 0) {  // full tile: 16-byte stores
        TOut o[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            o[k] = (TOut)run;
            run += v[k];
        }
        if constexpr (sizeof(TOut) == 4) {
#pragma unroll
            for (int k = 0; k < kScanItems; k += 4)
                *reinterpret_cast<int4 *>(out + base + k) =
                    make_int4((int)o[k], (int)o[k + 1], (int)o[k + 2], (int)o[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < kScanItems; k += 2)
                *reinterpret_cast<longlong2 *>(out + base + k) =
                    make_longlong2((long long)o[k], (long long)o[k + 1]);
        }
        if (base + kScanItems == n) out[n] = (TOut)run;
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const int64_t i = base + k;
            if (i < n) out[i] = (TOut)run;
            run += v[k];
            if (i == n - 1) out[n] = (TOut)run;
        }
    }
}

// host helper: one memset (status + counter) and one launch on `stream`
template <typename TIn, typename TOut>
inline int exclusive_scan(const TIn *in, int64_t n, TOut *out, void *ws, size_t ws_bytes,
                          cudaStream_t stream) {
    if (n < 0) return FM_ERR_ARG;
    if (ws_bytes < scan_workspace_bytes(n)) return FM_ERR_WORKSPACE;
    const int64_t nb = scan_blocks(n);
    if (nb == 0) {
        cudaMemsetAsync(out, 0, sizeof(TOut), stream);
        FM_CHECK_LAUNCH();
        return FM_OK;
    }
    unsigned long long *status = reinterpret_cast<unsigned long long *>(ws);
    unsigned int *counter = reinterpret_cast<unsigned int *>(status + nb);
    if (cudaMemsetAsync(ws, 0, (size_t)(nb + 1) * sizeof(unsigned long long), stream) !=
        cudaSuccess)
        return FM_ERR_CUDA;
    k_scan_lookback<TIn, TOut><<<(unsigned)nb, kScanThreads, 0, stream>>>(in, n, out, status,
                                                                          counter);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

}  // namespace fm
