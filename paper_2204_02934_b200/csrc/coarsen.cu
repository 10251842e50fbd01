// coarsen.cu -- coarse graph A_c <- coarsen(A) (Alg. 4 setup): the
// quotient graph over the aggregates, rows sorted and deduplicated, no
// self-loops (reading Q21).
//
// Device pipeline (no global sort of all nnz keys):
//   1. seglen[a] = sum of stored row lengths of a's members
//   2. sptr = exclusive scan(seglen)
//   3. every fine row u appends the distinct labels of adj(u) other than its
//      own (per-lane register lists) into its aggregate's segment at an
//      atomically reserved offset
//   4. per segment: shared-memory hash set of the distinct labels, then the
//      uniques in sorted order (warp per segment up to 4096 entries / 255
//      distinct; else a block per segment up to 2047 distinct); segments with
//      more distinct labels use an na-bit bitmap (ordered compaction = sorted unique)
//   5. c_rowptr = exclusive scan(unique counts); copy out.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace mis2k {

constexpr int32_t kSent = 0x7fffffff;

__global__ void k_check_labels(int64_t n, const int32_t* __restrict__ labels, int64_t na, int* err) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = labels[v];
        if (a < 0 || a >= na) atomicOr(err, 1);
    }
}

__global__ void k_seglen(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ labels,
                         int64_t na, unsigned long long* __restrict__ seglen) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = rowptr[v + 1] - rowptr[v];
        const int32_t a = labels[v];
        // out-of-range labels are skipped here and in k_fill (k_check_labels
        // flags them; the call returns MIS2_EINVAL without touching memory
        // outside the workspace)
        if (d && a >= 0 && a < na) atomicAdd(&seglen[a], (unsigned long long)d);
    }
}

// Each lane keeps the distinct labels (!= own) of its entries in a register
// list of kFillList; a full list is flushed to the segment at an atomically
// reserved offset.  Typical rows touch 2-4 aggregates, so the segments hold a
// few entries per fine row instead of its degree (duplicates across lanes and
// flushes remain; step 4 removes them).  A segment's used length is
// cursor[a] - sptr[a] <= its capacity seglen[a].
#ifndef MIS2_FILL_LIST
#define MIS2_FILL_LIST 6
#endif
// list size measured (coarsen ms, C5 / C2 / C3): 4 -> 2.69 / 0.284 / 4.33,
// 6 -> 2.70 / 0.275 / 4.31, 8 -> ~2.9 / 0.275 / 4.38, 12 -> 3.72 / 0.300 / 4.49
constexpr int kFillList = MIS2_FILL_LIST;
template <int G>
__global__ void k_fill(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                       const int32_t* __restrict__ labels, int64_t na, unsigned long long* __restrict__ cursor,
                       int32_t* __restrict__ buf) {
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & 31, grp = lane / G, sub = lane % G;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = gwarp * RPW; base < n; base += nwarps * RPW) {
        const int64_t v = base + grp;
        const bool valid = v < n;
        int32_t lst[kFillList];
        int cnt = 0;
        int32_t a = 0;
        if (valid) a = labels[v];
        if (valid && a >= 0 && a < na) {
            const int64_t s = rowptr[v], e = rowptr[v + 1];
            row_batched<G, 8>(s, e, sub, colinds, [&](int32_t w) { return labels[w]; }, [&](int32_t, int32_t b) {
                if (b == a || b < 0 || b >= na) return;
                bool found = false;
#pragma unroll
                for (int k = 0; k < kFillList; k++) found |= (k < cnt) && lst[k] == b;
                if (found) return;
                if (cnt == kFillList) {
                    const unsigned long long pos = atomicAdd(&cursor[a], (unsigned long long)kFillList);
#pragma unroll
                    for (int k = 0; k < kFillList; k++) buf[pos + k] = lst[k];
                    cnt = 0;
                }
#pragma unroll
                for (int k = 0; k < kFillList; k++)
                    if (k == cnt) lst[k] = b;
                cnt++;
            });
        }
        // one reservation per row for the lanes' final lists
        int incl = cnt;
#pragma unroll
        for (int off = 1; off < G; off <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, off, G);
            if (sub >= off) incl += y;
        }
        const int tot = __shfl_sync(kFull, incl, G - 1, G);
        unsigned long long pos = 0;
        if (sub == G - 1 && tot > 0) pos = atomicAdd(&cursor[a], (unsigned long long)tot);
        pos = __shfl_sync(kFull, pos, G - 1, G) + (unsigned long long)(incl - cnt);
#pragma unroll
        for (int k = 0; k < kFillList; k++)
            if (k < cnt) buf[pos + k] = lst[k];
    }
}

// in-place bitonic sort of x[0..P) (P power of two) by `nthreads` threads
__device__ __forceinline__ void bitonic(int32_t* x, int P, int tid, int nthreads, bool warp_only) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P / 2; i += nthreads) {
                const int lo = 2 * i - (i & (j - 1));
                const int hi = lo + j;
                const bool up = (lo & k) == 0;
                const int32_t a = x[lo], b = x[hi];
                if ((a > b) == up) { x[lo] = b; x[hi] = a; }
            }
            if (warp_only) __syncwarp(); else __syncthreads();
        }
    }
}

// warp per segment: the distinct labels go through a per-warp shared-memory
// hash set (a coarse row of a stencil graph has ~27 distinct neighbours
// against ~60-100 segment entries), then each unique is placed by its rank
// among the uniques (O(u) broadcast reads per unique).  Segments longer than
// kWarpSegMax entries or with kWarpUniq or more distinct labels are marked
// ucnt = -1 for the block kernel.
constexpr int kWarpHash = 512;
constexpr int kWarpUniq = 256;
constexpr int64_t kWarpSegMax = 4096;
__global__ void k_dedupe_warp(int64_t na, const int64_t* __restrict__ sptr, const unsigned long long* __restrict__ send,
                              int32_t* __restrict__ buf, int64_t* __restrict__ ucnt) {
    __shared__ int32_t hs[kWarpsPerBlock][kWarpHash];
    __shared__ int32_t uqs[kWarpsPerBlock][kWarpUniq];
    __shared__ int s_cnt[kWarpsPerBlock];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t* h = hs[warp];
    int32_t* uq = uqs[warp];
    const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
    for (int64_t a = (int64_t)blockIdx.x * kWarpsPerBlock + warp; a < na; a += nwarps) {
        const int64_t s = sptr[a], len = (int64_t)send[a] - s;
        if (len > kWarpSegMax) {
            if (lane == 0) ucnt[a] = -1;
            continue;
        }
        for (int i = lane; i < kWarpHash; i += 32) h[i] = -1;
        if (lane == 0) s_cnt[warp] = 0;
        __syncwarp();
        for (int64_t j0 = 0; j0 < len; j0 += 32) {
            if (__any_sync(kFull, *(volatile int*)&s_cnt[warp] >= kWarpUniq)) break;  // overflow: block path
            const int64_t j = j0 + lane;
            const int32_t b = j < len ? buf[s + j] : -1;
            // one lane per distinct value of the chunk inserts it
            const unsigned m = __match_any_sync(kFull, b);
            if (b < 0 || (m & lanemask_lt())) continue;
            uint32_t slot = ((uint32_t)b * 2654435761u) >> 23;  // 9-bit hash
            for (;;) {
                const int32_t cur = ((volatile int32_t*)h)[slot];
                if (cur == b) break;
                if (cur != -1) {
                    slot = (slot + 1) & (kWarpHash - 1);
                    continue;
                }
                const int32_t prev = atomicCAS(&h[slot], -1, b);
                if (prev == -1) {
                    const int k = atomicAdd(&s_cnt[warp], 1);
                    if (k < kWarpUniq) uq[k] = b;
                    break;
                }
                if (prev == b) break;
                slot = (slot + 1) & (kWarpHash - 1);
            }
        }
        __syncwarp();
        const int cnt = *(volatile int*)&s_cnt[warp];
        if (cnt >= kWarpUniq) {
            if (lane == 0) ucnt[a] = -1;
            __syncwarp();
            continue;
        }
        for (int i = lane; i < cnt; i += 32) {
            const int32_t x = uq[i];
            int r = 0;
            for (int k = 0; k < cnt; k++) r += uq[k] < x;
            buf[s + r] = x;
        }
        if (lane == 0) ucnt[a] = cnt;
        __syncwarp();
    }
}

// block per segment the warp kernel marked (ucnt = -1): the distinct labels are collected
// in a shared-memory hash set (coarse rows have few distinct neighbours, e.g.
// ~17 per aggregate on the elasticity graph against ~5.7K entries), then only
// the uniques are sorted.  Segments with more than kMaxUniq distinct labels go
// to `big` (bitmap path).
constexpr int kHashCap = 4096;
constexpr int kMaxUniq = 2048;
__global__ void k_dedupe_block(int64_t na, const int64_t* __restrict__ sptr, const unsigned long long* __restrict__ send,
                               int32_t* __restrict__ buf,
                               int64_t* __restrict__ ucnt, int32_t* __restrict__ big, int* big_cnt) {
    __shared__ int32_t keys[kHashCap];
    __shared__ int32_t uq[kMaxUniq];
    __shared__ int s_cnt;
    for (int64_t a = blockIdx.x; a < na; a += gridDim.x) {
        if (ucnt[a] >= 0) continue;
        const int64_t s = sptr[a], len = (int64_t)send[a] - s;
        for (int i = threadIdx.x; i < kHashCap; i += blockDim.x) keys[i] = -1;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int64_t j = s + threadIdx.x; j < s + len; j += blockDim.x) {
            const int32_t b = buf[j];
            if (*(volatile int*)&s_cnt >= kMaxUniq) break;  // overflow: bitmap path below
            uint32_t slot = ((uint32_t)b * 2654435761u) >> 20;  // 12-bit hash
            for (;;) {
                const int32_t prev = atomicCAS(&keys[slot], -1, b);
                if (prev == -1) {
                    const int k = atomicAdd(&s_cnt, 1);
                    if (k < kMaxUniq) uq[k] = b;
                    break;
                }
                if (prev == b) break;
                slot = (slot + 1) & (kHashCap - 1);
            }
        }
        __syncthreads();
        const int cnt = s_cnt;
        if (cnt > kMaxUniq || (cnt == kMaxUniq)) {
            if (threadIdx.x == 0) big[atomicAdd(big_cnt, 1)] = (int32_t)a;
            __syncthreads();
            continue;
        }
        int P = 1;
        while (P < cnt) P <<= 1;
        for (int i = cnt + threadIdx.x; i < P; i += blockDim.x) uq[i] = kSent;
        __syncthreads();
        bitonic(uq, P, threadIdx.x, blockDim.x, false);
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) buf[s + i] = uq[i];
        if (threadIdx.x == 0) ucnt[a] = cnt;
        __syncthreads();
    }
}

// one block handles one long segment via an na-bit bitmap
__global__ void k_bitmap_segment(const int32_t* __restrict__ big, int idx, const int64_t* __restrict__ sptr,
                                 const unsigned long long* __restrict__ send,
                                 int32_t* __restrict__ buf, int64_t* __restrict__ ucnt, unsigned* __restrict__ bm,
                                 int64_t na) {
    __shared__ int s_w[32 + 1];
    const int64_t a = big[idx];
    const int64_t s = sptr[a], e = (int64_t)send[a];
    const int64_t words = (na + 31) / 32;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int64_t j = s + threadIdx.x; j < e; j += blockDim.x) {
        const int32_t b = buf[j];
        atomicOr(&bm[b >> 5], 1u << (b & 31));
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    int64_t carry = 0;
    for (int64_t base = 0; base < words; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const unsigned wbits = i < words ? bm[i] : 0u;
        int c = __popc(wbits);
        int inc = c;
        for (int off = 1; off < 32; off <<= 1) {
            int y = __shfl_up_sync(kFull, inc, off);
            if (lane >= off) inc += y;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        int64_t off = carry;
        for (int w = 0; w < warp; w++) off += s_w[w];
        off += inc - c;
        unsigned bits = wbits;
        while (bits) {
            const int t = __ffs(bits) - 1;
            buf[s + off++] = (int32_t)(i * 32 + t);
            bits &= bits - 1;
        }
        int tot = 0;
        for (int w = 0; w < nw; w++) tot += s_w[w];
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) ucnt[a] = carry;
}

// warp per aggregate: copy uniques to the output CSR
__global__ void k_copy_out(int64_t na, const int64_t* __restrict__ sptr, const int32_t* __restrict__ buf,
                           const int64_t* __restrict__ crow, int32_t* __restrict__ ccol) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
    for (int64_t a = (int64_t)blockIdx.x * kWarpsPerBlock + warp; a < na; a += nwarps) {
        const int64_t s = sptr[a], o = crow[a], len = crow[a + 1] - o;
        for (int64_t i = lane; i < len; i += 32) ccol[o + i] = buf[s + i];
    }
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

int run_coarsen(const mis2_graph& g, const int32_t* labels, int64_t na, int64_t* c_rowptr, int32_t* c_colinds,
                int64_t cap, int64_t* c_nnz, void* ws, size_t ws_bytes, cudaStream_t s, size_t* bytes_needed) {
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    const int64_t n = g.n;
    // sizing uses the bound na <= n (the partitioned driver sizes with n = max(rows, na))
    const int64_t nab = bytes_needed ? n : na;
    Carve c(ws, ws_bytes);
    unsigned long long* seglen = c.take<unsigned long long>((size_t)nab + 1);
    int64_t* sptr = c.take<int64_t>((size_t)nab + 2);
    unsigned long long* cursor = c.take<unsigned long long>((size_t)nab + 1);
    int64_t* ucnt = c.take<int64_t>((size_t)nab + 1);
    int32_t* big = c.take<int32_t>((size_t)nab + 1);
    unsigned* bm = c.take<unsigned>((size_t)(nab + 31) / 32 + 1);
    int32_t* buf = c.take<int32_t>((size_t)g.nnz + 1);
    void* tmp = c.take<char>(scan64_ws_bytes(nab + 1));
    int* scal = c.take<int>(16);
    if (bytes_needed) { *bytes_needed = c.off; return MIS2_OK; }
    if (!c.ok()) { set_error("workspace too small: need %zu bytes", c.off); return MIS2_ENOMEM; }
    if (na < 0 || na > nab || (n > 0 && na == 0)) { set_error("num_aggs out of range"); return MIS2_EINVAL; }

    // lanes per row of the fill: a quarter of the MIS-2 kernels' group for
    // long rows -- each lane's distinct-label list then sees more of its
    // row (C5, G = 1 / 2 / 4 / 8 / 32: 2.17 / 2.37 / 2.79 / 3.49 / 6.21 ms;
    // C3 at 1 / 2 / 4: 4.23 / 4.56 / 5.15 ms; C2 0.273 / 0.288 ms)
    int G = choose_group(g.n, g.nnz, 0);
    if (G >= 4) G /= 4;
    if (const char* e = getenv("MIS2_COARSEN_G")) G = atoi(e);  // measurement knob (1..32, power of 2)
    int64_t blocks = (n + kBlock - 1) / kBlock;
    if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
    if (blocks < 1) blocks = 1;

    MIS2_CUDA_TRY(cudaMemsetAsync(scal, 0, 16 * sizeof(int), s));
    MIS2_CUDA_TRY(cudaMemsetAsync(seglen, 0, sizeof(unsigned long long) * ((size_t)na + 1), s));
    count_launch(2);
    k_check_labels<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, na, &scal[0]);
    k_seglen<<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, labels, na, seglen);
    count_launch(2);
    MIS2_TRY(scan_counts64((const int64_t*)seglen, na, sptr, tmp, s));
    MIS2_CUDA_TRY(cudaMemcpyAsync(cursor, sptr, sizeof(int64_t) * (size_t)na, cudaMemcpyDeviceToDevice, s));
    {
        const int64_t rows_per_block = (int64_t)(kBlock / 32) * (32 / G);
        int64_t fb = (n + rows_per_block - 1) / rows_per_block;
        if (fb > (int64_t)di.sms * 16) fb = (int64_t)di.sms * 16;
        if (fb < 1) fb = 1;
        switch (G) {
            case 1: k_fill<1><<<(unsigned)fb, kBlock, 0, s>>>(n, g.rowptr, g.colinds, labels, na, cursor, buf); break;
            case 2: k_fill<2><<<(unsigned)fb, kBlock, 0, s>>>(n, g.rowptr, g.colinds, labels, na, cursor, buf); break;
            case 4: k_fill<4><<<(unsigned)fb, kBlock, 0, s>>>(n, g.rowptr, g.colinds, labels, na, cursor, buf); break;
            case 8: k_fill<8><<<(unsigned)fb, kBlock, 0, s>>>(n, g.rowptr, g.colinds, labels, na, cursor, buf); break;
            case 16: k_fill<16><<<(unsigned)fb, kBlock, 0, s>>>(n, g.rowptr, g.colinds, labels, na, cursor, buf); break;
            default: k_fill<32><<<(unsigned)fb, kBlock, 0, s>>>(n, g.rowptr, g.colinds, labels, na, cursor, buf); break;
        }
        count_launch();
    }
    {
        int64_t wb = (na + kWarpsPerBlock - 1) / kWarpsPerBlock;
        if (wb > (int64_t)di.sms * 32) wb = (int64_t)di.sms * 32;
        if (wb < 1) wb = 1;
        k_dedupe_warp<<<(unsigned)wb, kBlock, 0, s>>>(na, sptr, cursor, buf, ucnt);
        int64_t bb = na < (int64_t)di.sms * 8 ? na : (int64_t)di.sms * 8;
        if (bb < 1) bb = 1;
        k_dedupe_block<<<(unsigned)bb, kBlock, 0, s>>>(na, sptr, cursor, buf, ucnt, big, &scal[1]);
        count_launch(2);
    }
    int hs[16];
    MIS2_CUDA_TRY(cudaMemcpyAsync(hs, scal, sizeof(hs), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    if (hs[0]) { set_error("labels out of [0, num_aggs)"); return MIS2_EINVAL; }
    for (int i = 0; i < hs[1]; i++) {
        k_bitmap_segment<<<1, 1024, 0, s>>>(big, i, sptr, cursor, buf, ucnt, bm, na);
        count_launch();
    }
    MIS2_TRY(scan_counts64(ucnt, na, c_rowptr, tmp, s));
    int64_t total = 0;
    MIS2_CUDA_TRY(cudaMemcpyAsync(&total, c_rowptr + na, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    *c_nnz = total;
    if (c_colinds == nullptr || cap < total) return MIS2_ERANGE;
    {
        int64_t wb = (na + kWarpsPerBlock - 1) / kWarpsPerBlock;
        if (wb > (int64_t)di.sms * 32) wb = (int64_t)di.sms * 32;
        if (wb < 1) wb = 1;
        k_copy_out<<<(unsigned)wb, kBlock, 0, s>>>(na, sptr, buf, c_rowptr, c_colinds);
        count_launch();
    }
    MIS2_CUDA_TRY(cudaGetLastError());
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    return MIS2_OK;
}

}  // namespace mis2h
