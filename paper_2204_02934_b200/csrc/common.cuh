// common.cuh -- device helpers shared by the sm_100a kernels of libmis2.so.
//
// Product code (no oracle/ dependency).  "P:n" = PAPER.md line n; "Qk" =
// DESIGN.md reading k.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mis2.h"

namespace mis2k {

// §V-C compressed status words: IN = 0, OUT = UINT_MAX (64-bit, Q6).
constexpr uint64_t kIN = 0ull;
constexpr uint64_t kOUT = ~0ull;
constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = 32 * kWarpsPerBlock;
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- priorities
// §V-A: h(iter, v) = f(f(iter) ^ f(v)); Xor*: f = xorshift64*
// (xorshift (13,7,17) then * 0x2545F4914F6CDD1D, reading Q3); seed mixed
// into the iteration term (Q4); the priority is the HIGH 64-b bits (Q5).
__device__ __forceinline__ uint64_t xs64(uint64_t x) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}
__device__ __forceinline__ uint64_t xs64star(uint64_t x) { return xs64(x) * 0x2545F4914F6CDD1Dull; }

struct Prio {
    int scheme;
    int b;
    uint64_t seed;
    uint64_t hi_mask;           // ~(2^b - 1)
    int hshift;                 // 0: W = 64; 32: W = 32, priority from the high half of h (Q32)
    int64_t n;
    const uint64_t* override_;  // test-only (Fig. 1 replay)
    int override_iters;

    // per-iteration constant part of h
    __device__ __forceinline__ uint64_t iter_term(int it) const {
        if (scheme == MIS2_SCHEME_XOR) return xs64((uint64_t)it ^ seed);
        return xs64star((uint64_t)it ^ seed);
    }
    // packed undecided word (priority << b) | (v + 1)
    __device__ __forceinline__ uint64_t word(int it, uint64_t fi, int64_t v) const {
        if (override_ != nullptr && it < override_iters)
            return (override_[(int64_t)it * n + v] << b) | (uint64_t)(v + 1);
        uint64_t h;
        if (scheme == MIS2_SCHEME_FIXED) h = xs64star(seed ^ xs64star((uint64_t)v));
        else if (scheme == MIS2_SCHEME_XOR) h = xs64(fi ^ xs64((uint64_t)v));
        else h = xs64star(fi ^ xs64star((uint64_t)v));
        return ((h >> hshift) & hi_mask) | (uint64_t)(v + 1);
    }
};

// ------------------------------------------------------------- warp helpers
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int G>
__device__ __forceinline__ uint64_t group_min(uint64_t x) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        uint64_t y = __shfl_xor_sync(kFull, x, off);
        x = y < x ? y : x;
    }
    return x;
}
template <int G>
__device__ __forceinline__ int group_or(int x) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) x |= __shfl_xor_sync(kFull, x, off);
    return x;
}
template <int G>
__device__ __forceinline__ int group_and(int x) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) x &= __shfl_xor_sync(kFull, x, off);
    return x;
}
template <int G>
__device__ __forceinline__ int group_sum(int x) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) x += __shfl_xor_sync(kFull, x, off);
    return x;
}

__device__ __forceinline__ long long warp_sum_ll(long long x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(kFull, x, off);
    return x;
}

// -------------------------------------------------------------- grid barrier
// Sense-flip grid barrier for a cooperatively launched (co-resident) grid:
// block 0 adds 0x80000000 - (nblocks - 1), every other block adds 1, so the
// top bit flips exactly when all blocks have arrived.  Release on arrival;
// the spin uses RELAXED loads with a short sleep (an acquire load compiles to
// LD.STRONG + CCTL.IVALL, and invalidating L1 on every poll would wipe the
// cache of co-resident blocks that are still gathering); one acquire fence
// after the flip makes every block's prior writes visible.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, int mode = 0) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int nb = (blockIdx.x == 0) ? (0x80000000u - (gridDim.x - 1)) : 1u;
        unsigned int old;
        asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
        unsigned int cur;
        if (mode == 2) {  // acquire polling (as cooperative_groups)
            for (;;) {
                asm volatile("ld.acquire.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
                if ((old ^ cur) & 0x80000000u) break;
            }
        } else {
            for (;;) {
                asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
                if ((old ^ cur) & 0x80000000u) break;
                if (mode == 0) __nanosleep(32);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    __syncthreads();
}

// Grid barrier that also sums one value per block (the loop condition
// |worklist_1|, and the active count), so no extra L2 round trip
// follows the barrier.  One 64-bit counter per barrier parity (ctr[0] and
// ctr[kSumStride], separate lines): bits [0, 40) accumulate the values, bits
// [40, 63) count arrivals, bit 63 flips when the last block arrives (block 0
// adds 2^63 - (B-1) 2^40, every other block 2^40).  A block reaches barrier
// k + 2 -- the same counter -- only after every block has left barrier k + 1,
// hence after every block has read barrier k's final value, so that value
// minus the one seen at barrier k - 2 is barrier k's sum.  Thread 0 keeps
// the previous totals; every thread gets the sum.
constexpr int kSumStride = 16;  // 128 bytes
struct SumBarrier {
    unsigned long long last[2];
    unsigned int k;
};
// Split phase: grid_arrive_sum (after the block's writes; thread 0's atomic
// returns the pre-arrival value `old`), independent work (the next phase's
// prologue: it only reads static data and the block's own rows), then
// grid_wait_sum.
// sb lives in shared memory (only thread 0 touches it; fewer registers)
__device__ __forceinline__ unsigned long long grid_arrive_sum(unsigned long long* ctr, const SumBarrier& sb,
                                                              unsigned long long val,
                                                              unsigned long long* side = nullptr,
                                                              unsigned long long side_val = 0ull) {
    __syncthreads();
    unsigned long long old = 0;
    if (threadIdx.x == 0) {
        // an extra per-block value accumulated beside the barrier (visible to
        // every block once the barrier completes: the arrival is a release)
        if (side && side_val) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(side), "l"(side_val) : "memory");
        unsigned long long* c = ctr + (sb.k & 1u) * kSumStride;
        const unsigned long long add =
            (blockIdx.x == 0 ? (1ull << 63) - ((unsigned long long)(gridDim.x - 1) << 40) : (1ull << 40)) + val;
        asm volatile("atom.add.release.gpu.u64 %0,[%1],%2;" : "=l"(old) : "l"(c), "l"(add) : "memory");
    }
    return old;
}
__device__ __forceinline__ unsigned long long grid_wait_sum(unsigned long long* ctr, SumBarrier& sb,
                                                            unsigned long long old, unsigned long long* s_out) {
    constexpr unsigned long long kSumMask = (1ull << 40) - 1ull;
    if (threadIdx.x == 0) {
        unsigned long long* c = ctr + (sb.k & 1u) * kSumStride;
        unsigned long long cur;
        for (;;) {
            asm volatile("ld.relaxed.gpu.u64 %0,[%1];" : "=l"(cur) : "l"(c) : "memory");
            if ((old ^ cur) >> 63) break;
            __nanosleep(32);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const unsigned long long tot = cur & kSumMask;
        *s_out = (tot - sb.last[sb.k & 1u]) & kSumMask;
        sb.last[sb.k & 1u] = tot;
        sb.k++;
    }
    __syncthreads();
    return *(volatile unsigned long long*)s_out;
}
__device__ __forceinline__ unsigned long long grid_sync_sum(unsigned long long* ctr, SumBarrier& sb,
                                                            unsigned long long val, unsigned long long* s_out) {
    const unsigned long long old = grid_arrive_sum(ctr, sb, val);
    return grid_wait_sum(ctr, sb, old, s_out);
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.u64 %0,[%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// block-wide sum of one value per warp (lane 0 holds it); result in thread 0
__device__ __forceinline__ long long block_sum_warps(long long warp_val, long long* s_tmp) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) s_tmp[warp] = warp_val;
    __syncthreads();
    long long s = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += s_tmp[w];
    __syncthreads();
    return s;
}

// Visits the entries j = s + sub, s + sub + G, ... < e of a row with U column
// loads, then U gathers ld(w), in flight per batch; use(w, ld(w)) in order.
template <int G, int U, class Load, class Use>
__device__ __forceinline__ void row_batched(int64_t s, int64_t e, int sub, const int32_t* __restrict__ colinds,
                                            Load ld, Use use) {
    for (int64_t j0 = s + sub; j0 < e; j0 += (int64_t)U * G) {
        int32_t w[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t j = j0 + (int64_t)u * G;
            w[u] = j < e ? colinds[j] : -1;
        }
        decltype(ld(0)) x[U];
#pragma unroll
        for (int u = 0; u < U; u++) x[u] = w[u] >= 0 ? ld(w[u]) : decltype(ld(0))();
#pragma unroll
        for (int u = 0; u < U; u++)
            if (w[u] >= 0) use(w[u], x[u]);
    }
}

}  // namespace mis2k
