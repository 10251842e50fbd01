// scan.cu -- device-wide exclusive scans used by the aggregate numbering
// (Alg. 3: ids "in ascending vertex order", reading Q18) and by the coarse
// CSR row pointers.  Three passes: per-tile reduce, single-block scan of the
// tile sums, per-tile scan + write.  Integer only, so order of combination
// never changes the result.
#include "common.cuh"
#include "internal.h"

namespace mis2k {

constexpr int kScanThreads = 256;
constexpr int kScanItems8 = 16;  // uint8 flags per thread
constexpr int kTile8 = kScanThreads * kScanItems8;
constexpr int kScanItems64 = 4;  // int64 counts per thread
constexpr int kTile64 = kScanThreads * kScanItems64;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T x, T* s_warp, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        T y = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = (lane < (int)(blockDim.x >> 5)) ? s_warp[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            T y = __shfl_up_sync(kFull, wi, off);
            if (lane >= off) wi += y;
        }
        if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    T res = s_warp[warp] + inc - x;
    if (total) *total = s_warp[32];
    __syncthreads();
    return res;
}

__device__ __forceinline__ int64_t eff_n(int64_t n, const int32_t* d_n) {
    if (!d_n) return n;
    const int64_t m = *d_n;
    return m < n ? m : n;
}

__global__ void k_tile_count8(const uint8_t* __restrict__ f, int64_t n, int64_t* __restrict__ tsum,
                              const int32_t* __restrict__ d_n) {
    __shared__ int64_t s[33];
    n = eff_n(n, d_n);
    const int64_t base = (int64_t)blockIdx.x * kTile8 + (int64_t)threadIdx.x * kScanItems8;
    int64_t c = 0;
#pragma unroll
    for (int i = 0; i < kScanItems8; i++)
        if (base + i < n) c += f[base + i] != 0;
    int64_t tot;
    block_exclusive_scan<int64_t>(c, s, &tot);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

// exclusive scan of tile sums in one block; out[k] = offset of tile k; *total
__global__ void k_scan_tiles(int64_t* __restrict__ tsum, int64_t ntiles, int64_t* __restrict__ total) {
    __shared__ int64_t s[33];
    int64_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int64_t x = i < ntiles ? tsum[i] : 0;
        int64_t tot;
        int64_t ex = block_exclusive_scan<int64_t>(x, s, &tot);
        if (i < ntiles) tsum[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

// prefix[i] (if non-null) = number of set flags before i; list[prefix[i]] =
// (map ? map[i] : i) for every set flag (if non-null): the ordered compaction
__global__ void k_tile_write8(const uint8_t* __restrict__ f, int64_t n, const int64_t* __restrict__ toff,
                              int32_t* __restrict__ prefix, int32_t* __restrict__ list,
                              const int32_t* __restrict__ map, const int32_t* __restrict__ d_n) {
    __shared__ int64_t s[33];
    n = eff_n(n, d_n);
    const int64_t base = (int64_t)blockIdx.x * kTile8 + (int64_t)threadIdx.x * kScanItems8;
    uint8_t v[kScanItems8];
    int64_t c = 0;
#pragma unroll
    for (int i = 0; i < kScanItems8; i++) {
        v[i] = (base + i < n) ? (f[base + i] != 0) : 0;
        c += v[i];
    }
    int64_t run = toff[blockIdx.x] + block_exclusive_scan<int64_t>(c, s, nullptr);
#pragma unroll
    for (int i = 0; i < kScanItems8; i++) {
        if (base + i < n) {
            if (prefix) prefix[base + i] = (int32_t)run;
            if (list && v[i]) list[run] = map ? map[base + i] : (int32_t)(base + i);
        }
        run += v[i];
    }
}

__global__ void k_total_to_i32(const int64_t* t64, int32_t* t32) { *t32 = (int32_t)*t64; }

__global__ void k_tile_sum64(const int64_t* __restrict__ x, int64_t n, int64_t* __restrict__ tsum) {
    __shared__ int64_t s[33];
    const int64_t base = (int64_t)blockIdx.x * kTile64 + (int64_t)threadIdx.x * kScanItems64;
    int64_t c = 0;
#pragma unroll
    for (int i = 0; i < kScanItems64; i++)
        if (base + i < n) c += x[base + i];
    int64_t tot;
    block_exclusive_scan<int64_t>(c, s, &tot);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

__global__ void k_tile_write64(const int64_t* __restrict__ x, int64_t n, const int64_t* __restrict__ toff,
                               int64_t* __restrict__ out, const int64_t* __restrict__ total) {
    __shared__ int64_t s[33];
    const int64_t base = (int64_t)blockIdx.x * kTile64 + (int64_t)threadIdx.x * kScanItems64;
    int64_t v[kScanItems64];
    int64_t c = 0;
#pragma unroll
    for (int i = 0; i < kScanItems64; i++) {
        v[i] = (base + i < n) ? x[base + i] : 0;
        c += v[i];
    }
    int64_t run = toff[blockIdx.x] + block_exclusive_scan<int64_t>(c, s, nullptr);
#pragma unroll
    for (int i = 0; i < kScanItems64; i++) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = *total;
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

size_t scan_ws_bytes(int64_t n) {
    const int64_t tiles = (n + kTile8 - 1) / kTile8 + 1;
    return (size_t)(tiles + 2) * sizeof(int64_t) + 256;
}

int scan_flags(const uint8_t* flags, int64_t n, int32_t* prefix, int32_t* d_total, void* tmp, cudaStream_t s) {
    return scan_flags_list(flags, n, nullptr, prefix, nullptr, nullptr, d_total, tmp, s);
}

int scan_flags_list(const uint8_t* flags, int64_t n, const int32_t* d_n, int32_t* prefix, int32_t* list,
                    const int32_t* map, int32_t* d_total, void* tmp, cudaStream_t s) {
    const int64_t tiles = (n + kTile8 - 1) / kTile8;
    int64_t* tsum = (int64_t*)tmp;
    int64_t* tot = tsum + tiles + 1;
    if (tiles > 0) {
        k_tile_count8<<<(unsigned)tiles, kScanThreads, 0, s>>>(flags, n, tsum, d_n);
        count_launch();
    }
    k_scan_tiles<<<1, 1024, 0, s>>>(tsum, tiles, tot);
    count_launch();
    if (tiles > 0) {
        k_tile_write8<<<(unsigned)tiles, kScanThreads, 0, s>>>(flags, n, tsum, prefix, list, map, d_n);
        count_launch();
    }
    k_total_to_i32<<<1, 1, 0, s>>>(tot, d_total);
    count_launch();
    MIS2_CUDA_TRY(cudaGetLastError());
    return MIS2_OK;
}

size_t scan64_ws_bytes(int64_t n) {
    const int64_t tiles = (n + kTile64 - 1) / kTile64 + 1;
    return (size_t)(tiles + 2) * sizeof(int64_t) + 256;
}

int scan_counts64(const int64_t* counts, int64_t n, int64_t* out, void* tmp, cudaStream_t s) {
    const int64_t tiles = (n + kTile64 - 1) / kTile64;
    int64_t* tsum = (int64_t*)tmp;
    int64_t* tot = tsum + tiles + 1;
    if (tiles > 0) {
        k_tile_sum64<<<(unsigned)tiles, kScanThreads, 0, s>>>(counts, n, tsum);
        count_launch();
    }
    k_scan_tiles<<<1, 1024, 0, s>>>(tsum, tiles, tot);
    count_launch();
    if (tiles > 0) {
        k_tile_write64<<<(unsigned)tiles, kScanThreads, 0, s>>>(counts, n, tsum, out, tot);
        count_launch();
    } else {
        MIS2_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    }
    MIS2_CUDA_TRY(cudaGetLastError());
    return MIS2_OK;
}

}  // namespace mis2h
