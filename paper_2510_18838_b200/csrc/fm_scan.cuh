// fm_scan.cuh -- exclusive prefix sum (reduce-then-scan, 3 launches).
//
// out[0] = 0, out[i+1] = out[i] + in[i] for i < n  (n+1 outputs).
// Used for the grid's cell_start (locate.py:82-84 `add.at` + `cumsum`) and for
// the support CSR offsets (_ext.pyx:220, 272).
#pragma once

#include "fm_common.cuh"

namespace fm {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

inline int64_t scan_blocks(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
inline size_t scan_workspace_bytes(int64_t n) {
    return (size_t)(scan_blocks(n) + 1) * sizeof(long long) + 256;
}

template <typename TIn>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const TIn *__restrict__ in,
                                                               int64_t n,
                                                               long long *__restrict__ sums) {
    __shared__ long long warp_part[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    long long acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
        if (i < n) acc += (long long)in[i];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FM_FULL_MASK, acc, o);
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int w = 0; w < kScanThreads / 32; w++) s += warp_part[w];
        sums[blockIdx.x] = s;
    }
}

// exclusive scan of the block sums in place (one block, chunked)
static __global__ void __launch_bounds__(1024) k_scan_sums(long long *__restrict__ sums, int64_t nb) {
    __shared__ long long warp_tot[32];
    __shared__ long long carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < nb; base += 1024) {
        const int64_t i = base + threadIdx.x;
        long long v = i < nb ? sums[i] : 0;
        long long x = v;
        for (int o = 1; o < 32; o <<= 1) {
            long long u = __shfl_up_sync(FM_FULL_MASK, x, o);
            if (lane >= o) x += u;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            long long t = warp_tot[lane];
            for (int o = 1; o < 32; o <<= 1) {
                long long u = __shfl_up_sync(FM_FULL_MASK, t, o);
                if (lane >= o) t += u;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        const long long carry = carry_s;
        const long long incl = x + (wid > 0 ? warp_tot[wid - 1] : 0) + carry;
        if (i < nb) sums[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[nb] = carry_s;
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const TIn *__restrict__ in,
                                                              int64_t n,
                                                              const long long *__restrict__ sums,
                                                              int64_t nb, TOut *__restrict__ out) {
    __shared__ long long warp_tot[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // each thread owns kScanItems consecutive elements
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    long long v[kScanItems];
    long long local = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const int64_t i = base + k;
        v[k] = i < n ? (long long)in[i] : 0;
        local += v[k];
    }
    long long x = local;
    for (int o = 1; o < 32; o <<= 1) {
        long long u = __shfl_up_sync(FM_FULL_MASK, x, o);
        if (lane >= o) x += u;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        long long t = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            long long u = __shfl_up_sync(FM_FULL_MASK, t, o);
            if (lane >= o) t += u;
        }
        if (lane < kScanThreads / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    long long run = sums[blockIdx.x] + (x - local) + (wid > 0 ? warp_tot[wid - 1] : 0);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const int64_t i = base + k;
        if (i < n) out[i] = (TOut)run;
        run += v[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = (TOut)sums[nb];
}

// host helper: launches the three kernels on `stream`
template <typename TIn, typename TOut>
inline int exclusive_scan(const TIn *in, int64_t n, TOut *out, void *ws, size_t ws_bytes,
                          cudaStream_t stream) {
    if (n < 0) return FM_ERR_ARG;
    if (ws_bytes < scan_workspace_bytes(n)) return FM_ERR_WORKSPACE;
    long long *sums = reinterpret_cast<long long *>(ws);
    const int64_t nb = scan_blocks(n);
    if (nb == 0) {
        cudaMemsetAsync(out, 0, sizeof(TOut), stream);
        FM_CHECK_LAUNCH();
        return FM_OK;
    }
    k_scan_reduce<TIn><<<(unsigned)nb, kScanThreads, 0, stream>>>(in, n, sums);
    k_scan_sums<<<1, 1024, 0, stream>>>(sums, nb);
    k_scan_apply<TIn, TOut><<<(unsigned)nb, kScanThreads, 0, stream>>>(in, n, sums, nb, out);
    FM_CHECK_LAUNCH();
    return FM_OK;
}

}  // namespace fm
