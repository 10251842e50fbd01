// mis2_kernel.cuh -- device code of Alg. 1 (MIS-2, §III-A): the
// single-GPU persistent kernel and the partitioned persistent kernel (one
// per GPU), both cooperatively launched sm_100a kernels.  Included by
// mis2_core.cu (host side, types only) and instantiated per lane-group width
// G in mis2_g<G>.cu (parallel build).
#pragma once
//
// Design:
//  * Each thread block owns runs of at most 256/G consecutive rows (Rows:
//    cyclic 256/G-row chunks b, b + B, ... on one GPU) and works through them
//    in steps of one run, G lanes per CSR row (§V-D "SIMD parallelism",
//    P:452-457, with a tunable group width).
//  * worklist_1 / worklist_2 (§V-B) live in the block's segment of
//    int32[n] arrays, double buffered (in -> out) and compacted with warp
//    ballots + one shared-memory atomic per warp: no global scan, no global
//    atomics, no block barrier per step.  The order inside a segment is
//    free (reading Q11): every phase is a per-vertex function of the
//    previous phase's arrays.
//  * Dense phases (iteration 0, and any block whose worklist still covers
//    >= 3/8 of its rows) walk its runs; the colinds of the next run are
//    streamed into shared memory by the Blackwell bulk-copy engine
//    (cp.async.bulk + mbarrier complete_tx), double buffered, while the
//    current run gathers T / M.  Worklist membership is read from the
//    status words (M_v != OUT for worklist_2, T_v undecided for worklist_1).
//  * Sparse phases read the block's compacted worklist; each row group
//    leader bulk-copies its row into a shared-memory slot one step ahead.
//    Rows longer than heavy_len<G>() (skewed graphs: one gather batch of
//    the lane group) are deferred to warps, rows longer than kHugeRow to the
//    whole block.
//  * Neighbour loops issue batches of independent gathers (indices clamped
//    to the row's last entry: min / exists / forall are idempotent).
//  * Phases are separated by a split-phase grid barrier that also sums the
//    loop condition |worklist_1|, so one call is 1 memset + 1 kernel
//    launch; each phase's prologue (first tile's bulk copy, first rows'
//    bounds and own status) is issued between the block's arrival and its
//    wait (PhaseState).  The IN decisions write the output mask directly and
//    their count rides beside the barrier.
//  * Refresh Row of iteration i+1 is fused into Decide of
//    iteration i; iteration 0's refresh is the init phase.
//  * 64-bit status words (Eq. 1, reading Q6): a min is one compare.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace mis2k {

// Warps per block: 8, four co-resident blocks per SM (shared memory and
// registers limit it to four).  Measured against 2 x 16 and 1 x 32 warps per
// SM with full-size tiles (C2 440 / 399 us against 371, profiles/
// r02a_experiments.md): the co-resident blocks of one SM are not scheduled
// fairly, but one large block synchronises more warps per step.
#ifndef MIS2_WARPS
#define MIS2_WARPS 8
#endif
constexpr int kMW = MIS2_WARPS;
constexpr int kMB = 32 * kMW;
constexpr int kMinBlocksPerSM = kMW >= 16 ? 1 : 32 / kMW;  // 32 warps per SM at 64 registers
// int32 colinds per staging buffer: a dense step of 27-entry rows
#ifndef MIS2_TILE_ROWS
#define MIS2_TILE_ROWS (kMB >= 512 ? kMB / 2 : kMB)
#endif
constexpr int kTileCap = (MIS2_TILE_ROWS) * 27;
// rows longer than 8 gather batches of their lane group are deferred and
// reduced by the whole block (flattened over all deferred rows of the block)
// independent gathers per lane per batch of the row loops
// issue each phase's prologue between the barrier arrival and wait (1) or
// after the wait (0, measurement knob)
#ifndef MIS2_HOIST
#define MIS2_HOIST 1
#endif
// 32-bit column keys with one minimum and a tie flag (1) or two 64-bit
// minima (0)
#ifndef MIS2_K32
#define MIS2_K32 1  // C4 31.0 -> 30.7 ms; the stencils keep 64-bit words (keys there: C2 342 -> 381 us)
#endif
#ifndef MIS2_B1
#define MIS2_B1 9  // measured: 9 is best on C2 (27 entries = 3 batches, 373 us vs 388 at 16) and near-best on C3
#endif
#ifndef MIS2_B4
#define MIS2_B4 11  // measured on C5 (81-entry rows over 4 lanes = 2 batches): 7.95 ms vs 8.24 at 8
#endif
template <int G>
__host__ __device__ constexpr int gather_batch() {
    return G == 1 ? MIS2_B1 : (G == 2 ? 16 : (G == 4 ? MIS2_B4 : 4));
}
#ifndef MIS2_HEAVY_BATCHES
#define MIS2_HEAVY_BATCHES 8
#endif
template <int G>
__host__ __device__ constexpr int heavy_len() {
    return MIS2_HEAVY_BATCHES * G * gather_batch<G>();
}
constexpr int kDenseNum = 3, kDenseDen = 8;
// lanes per row of the sparse (worklist) phases: GS = min(G * kSparseMul, 32)
#ifndef MIS2_SPARSE_MUL
#define MIS2_SPARSE_MUL 2
#endif
constexpr int kSparseMul = MIS2_SPARSE_MUL;
template <int G>
__host__ __device__ constexpr int sparse_group() {
    return G * kSparseMul <= 32 ? G * kSparseMul : 32;
}  // dense if |worklist segment| >= 3/8 of the range (pull phases)
// M_v is only ever compared against T_v (Decide: "M_w = T_v", "M_w = OUT").
// By Eq. 1 the low b bits of an undecided word are id+1, unique per vertex,
// never 0 and never all ones (2^b - 1 > |V|), and M_w is always a
// word of the CURRENT iteration (worklist_2 vertices are recomputed every
// iteration, the others hold OUT).  Hence M_w = T_v  <=>  id(M_w) = v + 1 and
// M_w = OUT <=> id(M_w) = all ones, so M is stored as a uint32 id field:
//   kM_OUT   : M_v = OUT
//   0        : inactive vertex (phase 2, reading Q15) -- ignored by Decide
//   a + 1    : M_v = T_a (a = argmin of T over N[v])
constexpr uint32_t kM_OUT = 0xffffffffu;
constexpr uint32_t kPending = 1u;  // M of an active vertex before its first column pass

struct MisParams {
    int64_t n;       // rows processed (all of them, or the owned rows of a partition)
    int64_t gbase;   // global id of local row 0 (0 on one GPU): hashes and ids use gbase + v
    // an induced subgraph (the masked MIS-2 of Alg. 3 phase 2, run on the
    // unaggregated vertices only): row v is vertex gid[v] of the whole graph,
    // whose id the hash and the packed words use (reading Q15: original ids);
    // inv maps those ids back to rows (push form).  Null: gbase + v.
    const int32_t* gid;
    const int32_t* inv;
    int64_t nnz;
    const int64_t* __restrict__ rowptr;
    const int32_t* __restrict__ colinds;
    const int32_t* __restrict__ labels;  // phase-2 mask (active iff labels[v] < 0) or null
    uint64_t* T;                         // row status T_v (64-bit packed word, Eq. 1)
    uint32_t* M;                         // column status M_v, stored as its id field (see below)
    uint32_t* K;                         // 32-bit column keys of T (kkey), maintained when non-null
    int keys_mode;                       // K non-null: 1 = use the keys, 0 = use them iff the degrees are skewed
    uint32_t id_mask;                    // 2^b - 1
    int32_t* L1[2];                      // worklist_1, double buffered, per-block segments
    int32_t* L2[2];                      // worklist_2
    unsigned long long* ctrl;
    int32_t* heavy;       // [n] deferred long rows, per-block segments at Rows::seg
    uint8_t* oflag;       // push-form Decide: some w in N[v] got M_w = OUT this iteration
    uint32_t* cnt;        // push-form Decide: |{w in N[v] : M_w = T_v}| this iteration
    uint32_t* degc;       // |N[v] ∩ active| (closed), written by the column pass of iteration 0
    unsigned int* mark;   // stats only
    long long* dstats;    // stats only
    long long* timeline;  // MIS2_FLAG_TIMELINE only
    float l2_keep;        // fraction of each block's colinds span kept in L2 (evict_last)
    int cyclic;           // row ownership: 0 = one contiguous range per block, 1 = cyclic chunks (Rows)
    int gather_keep;      // 1: key / M gathers carry an L2 evict_last hint (skewed graphs)
    int32_t* gq;          // MIS2_GQ kernels: global queue of deferred rows (int32[n]), null = off
    int heavy_batches;    // > 0: rows longer than heavy_batches gather batches of their lane group are
                          // deferred to warps (0: MIS2_HEAVY_BATCHES)
    int push_iters;       // PUSH kernels: iterations it < push_iters use the push-form Decide
    int dbg_it, dbg_ph;   // MIS2_FLAG_TIMELINE: sparse phase instrumented into `mark`
    Prio prio;
    int max_iters;
    uint8_t* in_set;
    int64_t* d_count;
    int32_t* d_iters;
    int32_t* d_status;
};

__device__ __forceinline__ int64_t gid_of(const MisParams& p, int64_t v) {
    return p.gid ? (int64_t)p.gid[v] : p.gbase + v;
}
__device__ __forceinline__ int64_t row_of_id(const MisParams& p, int64_t id) {
    return p.inv ? (int64_t)p.inv[id] : id - p.gbase;
}

// ------------------------------------------------------------ row ownership
// The rows of block b as "runs" of at most rpb consecutive rows (rpb = the
// rows of one dense step, kMB / G).
//  * contiguous (partitioned driver): the range [n*b/B, n*(b+1)/B) cut into
//    runs of rpb rows;
//  * cyclic (single GPU): the graph's rpb-row chunks c = b, b + B, b + 2B, ...
//    Vertices still undecided late in the loop cluster in space, so a block
//    owning one contiguous range can hold several times the mean worklist
//    of a phase (C2 iteration 5: 483 rows on average, 1689 on the largest)
//    and the grid barrier waits for it; chunks dealt round-robin give every
//    block a sample of the whole graph.
// The block's worklist / deferred-row segment is [seg, seg + count) of the
// int32[n] list arrays (segments of different blocks are disjoint).
struct Rows {
    int64_t n, B, b, rpb;
    bool cyclic;
    int64_t lo, hi;  // contiguous range (cyclic: unused)
    int64_t nruns, count, seg;
    __device__ __forceinline__ int64_t run_lo(int64_t k) const { return cyclic ? (b + k * B) * rpb : lo + k * rpb; }
    __device__ __forceinline__ int64_t run_hi(int64_t k) const {
        const int64_t e = run_lo(k) + rpb, lim = cyclic ? n : hi;
        return e < lim ? e : lim;
    }
    __device__ __forceinline__ int64_t row_at(int64_t i) const { return run_lo(i / rpb) + i % rpb; }
};
__device__ __forceinline__ Rows make_rows(int64_t n, int64_t B, int64_t b, int64_t rpb, bool cyclic) {
    Rows r;
    r.n = n;
    r.B = B;
    r.b = b;
    r.rpb = rpb;
    r.cyclic = cyclic;
    if (!cyclic) {
        r.lo = n * b / B;
        r.hi = n * (b + 1) / B;
        r.count = r.hi - r.lo;
        r.nruns = (r.count + rpb - 1) / rpb;
        r.seg = r.lo;
        return r;
    }
    r.lo = r.hi = 0;
    const int64_t nch = (n + rpb - 1) / rpb;         // chunks of the graph; chunk c -> block c mod B
    const int64_t tail = nch * rpb - n;              // rows missing from the last chunk
    const int64_t last_owner = nch > 0 ? (nch - 1) % B : -1;
    r.nruns = b < nch ? (nch - b + B - 1) / B : 0;
    r.count = r.nruns * rpb - (b == last_owner ? tail : 0);
    const int64_t before = (nch / B) * b + (b < nch % B ? b : nch % B);  // chunks of blocks < b
    r.seg = before * rpb - (last_owner >= 0 && last_owner < b ? tail : 0);
    return r;
}

// per block: the column passes use the 32-bit keys (decided once per call,
// after the init phase; see the kernel)
__shared__ int s_use_keys;
// per block: this iteration's phases use the global deferred-row queue
// (decided from the global |worklist_1|, so every block agrees)
__shared__ int s_gq_on;

struct __align__(16) TileSmem {
    int32_t buf[2][kTileCap + 8];
    unsigned long long mbar[2];   // dense tiles: one arrival (thread 0)
    unsigned long long mbarS[2];  // sparse tiles: one arrival per row group
    int64_t sal[2];  // 16-byte aligned colinds start of the staged span
    int32_t fits[2];
    uint64_t pol;    // L2 policy of this block's colinds span
    int cnt;         // survivors written this phase
    int hcount;
    int hnext;       // deferred rows: next row for a warp
    int nhuge;       // deferred rows too long for a warp
    int64_t nx_s, nx_e;  // dense phase, thread 0: colinds span of the step after the next
    int pending;         // a phase prologue was issued and not yet run (PhaseState)
    int gen0;            // buf[0] written by the generic proxy (push_halo's scan)
    uint64_t red64[kMW];
    int wred[kMW];
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// Blackwell bulk-copy engine: global -> shared, completion on an mbarrier
// with an L2 eviction-priority policy (see l2_policy)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* b,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
        : "memory");
}
// L2 residency of the CSR stream.  Every phase re-streams colinds; C2's
// 106 MB fits the 126 MB L2 but, with T, M, rowptr and the worklists also
// cycling through it, a plain LRU-like replacement of a cyclic scan larger
// than the cache keeps almost none of it between passes.  Each block marks
// the first `keep` fraction of its own colinds span evict_last and the rest
// evict_first, so a fixed, evenly spread part of the stream stays resident
// from phase to phase (all blocks see the same hit rate).  The span is
// demoted back to evict_normal when the call ends (l2_release).
__device__ __forceinline__ uint64_t l2_policy_range(const MisParams& p, int64_t s0, int64_t s1) {
    const char* base = reinterpret_cast<const char*>(p.colinds + s0);
    int64_t tot = (s1 - s0) * 4 + 128;
    if (tot > 0x7fffff00ll) tot = 0x7fffff00ll;
    const int64_t prim = (int64_t)((double)tot * (double)p.l2_keep) & ~(int64_t)127;
    uint64_t pol;
    if (p.l2_keep <= 0.f) {
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        return pol;
    }
    asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
                 : "=l"(pol)
                 : "l"(base), "r"((uint32_t)prim), "r"((uint32_t)tot));
    return pol;
}
// contiguous ownership: the first l2_keep of the block's own colinds span;
// cyclic ownership: the first l2_keep of the whole colinds array (= the first
// l2_keep of every block's chunks, since chunk c belongs to block c mod B)
__device__ __forceinline__ uint64_t l2_policy(const MisParams& p, const Rows& r) {
    if (r.cyclic) return l2_policy_range(p, 0, p.nnz);
    return l2_policy_range(p, p.rowptr[r.lo] & ~(int64_t)31, p.rowptr[r.hi]);
}
__device__ __forceinline__ void l2_release(const MisParams& p, const Rows& r) {
    if (p.l2_keep <= 0.f) return;
    const int64_t s0 = r.cyclic ? 0 : (p.rowptr[r.lo] & ~(int64_t)31), s1 = r.cyclic ? p.nnz : p.rowptr[r.hi];
    int64_t tot = (s1 - s0) * 4 + 128;
    if (tot > 0x7fffff00ll) tot = 0x7fffff00ll;
    const int64_t prim = (int64_t)((double)tot * (double)p.l2_keep);
    const char* base = reinterpret_cast<const char*>(p.colinds + s0);
    // cyclic: the blocks split the kept range; contiguous: each block its own
    const int64_t lines = (prim + 127) / 128;
    const int64_t l0 = r.cyclic ? lines * r.b / r.B : 0, l1 = r.cyclic ? lines * (r.b + 1) / r.B : lines;
    for (int64_t l = l0 + threadIdx.x; l < l1; l += blockDim.x)
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(base + l * 128) : "memory");
}
// gather of a 32-bit status word with an L2 eviction-priority hint (skewed
// graphs: the keys / M ids are the reuse targets; the CSR stream goes by)
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* a, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__shared__ uint64_t s_keep_pol;  // evict_last when p.gather_keep, else evict_normal
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ block helpers
// Warp-aggregated append of the group leaders' survivors to out[base + ...]
// (one shared atomic per warp; order inside the segment is free, Q11).
__device__ __forceinline__ void append(TileSmem& sm, bool keep, int32_t v, int32_t* out, int64_t base) {
    const unsigned ball = __ballot_sync(kFull, keep);
    if (ball == 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ball) - 1;
    int pos = 0;
    if (lane == leader) pos = atomicAdd(&sm.cnt, __popc(ball));
    pos = __shfl_sync(kFull, pos, leader);
    if (keep) out[base + pos + __popc(ball & lanemask_lt())] = v;
}

__device__ __forceinline__ uint64_t block_min_u64(TileSmem& sm, uint64_t x) {
    x = group_min<32>(x);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sm.red64[warp] = x;
    __syncthreads();
    uint64_t r = sm.red64[0];
#pragma unroll
    for (int w = 1; w < kMW; w++) r = sm.red64[w] < r ? sm.red64[w] : r;
    __syncthreads();
    return r;
}

__device__ __forceinline__ long long block_sum_int(TileSmem& sm, int x) {
    x = group_sum<32>(x);
    if ((threadIdx.x & 31) == 0) sm.wred[threadIdx.x >> 5] = x;
    __syncthreads();
    long long s = 0;
#pragma unroll
    for (int w = 0; w < kMW; w++) s += sm.wred[w];
    __syncthreads();
    return s;
}

// ------------------------------------------------------------ statistics
struct Stat {
    long long r = 0, e = 0, d = 0;
};
template <bool STATS>
__device__ __forceinline__ void stat_row(const MisParams& p, unsigned tag, int64_t v, bool leader, int64_t deg,
                                         Stat& st) {
    if (STATS && leader) {
        st.r++;
        st.e += deg;
        if (atomicMax(&p.mark[v], tag) < tag) st.d++;
    }
}
template <bool STATS>
__device__ __forceinline__ void stat_nbrs(const MisParams& p, unsigned tag, const int32_t* x, int64_t len, int sub,
                                          int stride, Stat& st) {
    if (STATS)
        for (int64_t j = sub; j < len; j += stride)
            if (atomicMax(&p.mark[x[j]], tag) < tag) st.d++;
}
template <bool STATS>
__device__ __forceinline__ void stats_flush(const MisParams& p, int it, int slot0, Stat st) {
    if (!STATS) return;
    st.r = warp_sum_ll(st.r);
    st.e = warp_sum_ll(st.e);
    st.d = warp_sum_ll(st.d);
    if ((threadIdx.x & 31) == 0) {
        long long* o = p.dstats + 6 * it;
        if (st.r) atomicAdd((unsigned long long*)&o[slot0], (unsigned long long)st.r);
        if (st.e) atomicAdd((unsigned long long*)&o[slot0 + 2], (unsigned long long)st.e);
        if (st.d) atomicAdd((unsigned long long*)&o[slot0 + 4], (unsigned long long)st.d);
    }
}

// ------------------------------------------------------------ row kernels
// Refresh Column of one row: min of T over the row's entries x[0..len)
// (x is shared memory or global; generic addressing), lanes sub, sub+G, ...
// Indices past the row end are clamped to its last entry: min / exists /
// forall are idempotent, so a repeated entry never changes the result and the
// loads need no predicate.
template <int G>
__device__ __forceinline__ uint64_t row_min(const uint64_t* __restrict__ T, const int32_t* x, int len, int sub,
                                            uint64_t m) {
    constexpr int B = gather_batch<G>();
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint64_t tt[B];
#pragma unroll
        for (int q = 0; q < B; q++) tt[q] = T[x[min(j + q * G, last)]];
#pragma unroll
        for (int q = 0; q < B; q++) m = tt[q] < m ? tt[q] : m;
        if (m == kIN) break;  // IN is the least word: the row's M is OUT whatever follows
    }
    return m;
}

// The same, also telling whether the row holds its own vertex (a stored
// diagonal, Q23): |N[v]| = len + 1 - self for the push-form Decide of an
// unmasked call (one compare per entry; counting T_w != OUT as below costs
// more: C2 column pass 0 ~8 us)
template <int G>
__device__ __forceinline__ uint64_t row_min_self(const uint64_t* __restrict__ T, const int32_t* x, int len, int sub,
                                                 uint64_t m, int32_t self, int& has) {
    constexpr int B = gather_batch<G>();
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint64_t tt[B];
        int32_t ww[B];
#pragma unroll
        for (int q = 0; q < B; q++) {
            ww[q] = x[min(j + q * G, last)];
            tt[q] = T[ww[q]];
        }
#pragma unroll
        for (int q = 0; q < B; q++) {
            m = tt[q] < m ? tt[q] : m;
            has |= ww[q] == self;
        }
    }
    return m;
}

// The same, also counting the entries w != self with T_w != OUT (iteration 0:
// exactly the active neighbours) for the push-form Decide.  Clamped repeats
// are not counted.
template <int G>
__device__ __forceinline__ uint64_t row_min_deg(const uint64_t* __restrict__ T, const int32_t* x, int len, int sub,
                                                uint64_t m, int64_t self, int& dc) {
    constexpr int B = gather_batch<G>();
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint64_t tt[B];
        int ww[B];
#pragma unroll
        for (int q = 0; q < B; q++) {
            ww[q] = x[min(j + q * G, last)];
            tt[q] = T[ww[q]];
        }
#pragma unroll
        for (int q = 0; q < B; q++) {
            m = tt[q] < m ? tt[q] : m;
            dc += (j + q * G <= last) & (tt[q] != kOUT) & ((int64_t)ww[q] != self);
        }
    }
    return m;
}

// Refresh Column on 32-bit keys (KEYS: p.K != null): the gathers read
// K_w = kkey(T_w) -- half the bytes of T, so K of a 16.7M-vertex graph stays
// L2-resident where T does not.  Two minima are kept: of (K_w, w) and of
// (K_w, ~w); their key parts are the least key, their id parts the least and
// the greatest id holding it.  Different ids = a tie in the key class, which
// the caller resolves on the full words.
__device__ __forceinline__ uint64_t key_lo(uint32_t k, uint32_t w) { return ((uint64_t)k << 32) | w; }
__device__ __forceinline__ uint64_t key_hi(uint32_t k, uint32_t w) { return ((uint64_t)k << 32) | (~w); }
template <int G>
__device__ __forceinline__ void row_min_keys(const uint32_t* __restrict__ K, const int32_t* x, int len, int sub,
                                             uint64_t& k1, uint64_t& k2, int32_t self = -1, int* has = nullptr) {
    constexpr int B = gather_batch<G>();
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint32_t kk[B];
        int32_t ww[B];
#pragma unroll
        for (int q = 0; q < B; q++) {
            ww[q] = x[min(j + q * G, last)];
            kk[q] = ld_keep(K + ww[q], s_keep_pol);
        }
#pragma unroll
        for (int q = 0; q < B; q++) {
            const uint64_t a = key_lo(kk[q], (uint32_t)ww[q]), b = key_hi(kk[q], (uint32_t)ww[q]);
            k1 = a < k1 ? a : k1;
            k2 = b < k2 ? b : k2;
            if (has) *has |= ww[q] == self;
        }
        if (!has && (k1 >> 32) == 0u) break;  // an IN neighbour: M is OUT (no IN in iteration 0 anyway)
    }
}

// Refresh Column on 32-bit keys, one minimum: (km, am) = the least key and
// the entry holding it; tie = another vertex holds the same key (resolved by
// the caller on the full words).  Cheaper than the two 64-bit minima of
// row_min_keys.
template <int G>
__device__ __forceinline__ void row_min_k32(const uint32_t* __restrict__ K, const int32_t* x, int len, int sub,
                                            uint32_t& km, int32_t& am, int& tie, int32_t self = -1,
                                            int* has = nullptr) {
    constexpr int B = gather_batch<G>();
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint32_t kk[B];
        int32_t ww[B];
#pragma unroll
        for (int q = 0; q < B; q++) {
            ww[q] = x[min(j + q * G, last)];
            kk[q] = ld_keep(K + ww[q], s_keep_pol);
        }
#pragma unroll
        for (int q = 0; q < B; q++) {
            const bool lt = kk[q] < km;
            const int eq = (kk[q] == km) & (ww[q] != am);
            tie = lt ? 0 : (tie | eq);
            am = lt ? ww[q] : am;
            km = lt ? kk[q] : km;
            if (has) *has |= ww[q] == self;
        }
        if (!has && km == 0u) break;  // an IN neighbour: M is OUT
    }
}
template <int G>
__device__ __forceinline__ void group_min_k32(uint32_t& km, int32_t& am, int& tie) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        const uint32_t k2 = __shfl_xor_sync(kFull, km, off);
        const int32_t a2 = __shfl_xor_sync(kFull, am, off);
        const int t2 = __shfl_xor_sync(kFull, tie, off);
        if (k2 < km) {
            km = k2;
            am = a2;
            tie = t2;
        } else if (k2 == km) {
            tie = tie | t2 | (a2 != am);
            am = a2 < am ? a2 : am;
        }
    }
}

// Decide of one row on id fields: exists M_w = OUT / forall
// M_w = T_v (id v+1); M_w = 0 (inactive, reading Q15) is ignored.
__device__ __forceinline__ void decide_acc(uint32_t m, uint32_t vid1, int& any_out, int& all_eq) {
    any_out |= (m == kM_OUT);
    all_eq &= (m == vid1) | (m == 0u);
}
template <int G>
__device__ __forceinline__ void row_decide(const uint32_t* __restrict__ M, const int32_t* x, int len, int sub,
                                           uint32_t vid1, int& any_out, int& all_eq) {
    constexpr int B = gather_batch<G>();
    const int last = len - 1;
    for (int j = sub; j < len; j += B * G) {
        uint32_t mm[B];
#pragma unroll
        for (int q = 0; q < B; q++) mm[q] = ld_keep(M + x[min(j + q * G, last)], s_keep_pol);
#pragma unroll
        for (int q = 0; q < B; q++) decide_acc(mm[q], vid1, any_out, all_eq);
        if (any_out) break;  // the row is OUT whatever follows
    }
}

// M_v from the column minimum m (IN -> OUT)
__device__ __forceinline__ uint32_t m_field(uint64_t m, uint32_t id_mask) {
    return (m == kIN || m == kOUT) ? kM_OUT : (uint32_t)m & id_mask;
}

// 32-bit column key of a status word (KEYS kernels): IN -> 0, OUT -> all
// ones, an undecided word -> its top 32 bits clamped to [1, 2^32 - 2].  The
// key order agrees with the word order except inside a class of equal keys,
// which the column pass detects and resolves on the full words (row_min_keys).
__device__ __forceinline__ uint32_t kkey(uint64_t t) {
    if (t == kIN) return 0u;
    if (t == kOUT) return 0xffffffffu;
    const uint32_t k = (uint32_t)(t >> 32);
    return k == 0u ? 1u : (k == 0xffffffffu ? 0xfffffffeu : k);
}
__device__ __forceinline__ void set_T(const MisParams& p, int64_t v, uint64_t t) {
    p.T[v] = t;
    if (p.K) p.K[v] = kkey(t);
}
// v decided IN: the output mask is written at the decision
// (init cleared it) and counted per block, so no pass over T follows the loop
__shared__ int s_nin;
__device__ __forceinline__ void set_IN(const MisParams& p, int64_t v) {
    set_T(p, v, kIN);
    p.in_set[v] = 1;
    atomicAdd(&s_nin, 1);
}

__device__ __forceinline__ bool decide_write(const MisParams& p, int64_t v, int any_out, int all_eq, int it,
                                             uint64_t fi_next) {
    if (any_out) {
        set_T(p, v, kOUT);
        return false;
    }
    if (all_eq) {
        set_IN(p, v);
        return false;
    }
    set_T(p, v, p.prio.word(it + 1, fi_next, gid_of(p, v)));  // fused Refresh Row
    return true;
}

// issue the bulk copy of colinds[s, e) (16-byte aligned hull) into buffer `slot`
__device__ __forceinline__ void stage_tile(TileSmem& sm, const MisParams& p, int slot, int64_t s, int64_t e) {
    const int64_t sal = s & ~(int64_t)3;
    const int64_t nnz4 = p.nnz & ~(int64_t)3;
    const int64_t ecp = (e + 3) & ~(int64_t)3;
    const bool fits = (ecp - sal) <= kTileCap && ecp <= nnz4;
    sm.sal[slot] = sal;
    sm.fits[slot] = fits;
    // no proxy fence: the buffer was only READ by the generic proxy before the
    // __syncthreads that precedes this call (write-after-read needs no
    // fence.proxy.async, which would also drain this thread's global stores)
    if (fits && ecp > sal) {
        mbar_expect_tx(&sm.mbar[slot], (uint32_t)((ecp - sal) * 4));
        bulk_g2s(sm.buf[slot], p.colinds + sal, (uint32_t)((ecp - sal) * 4), &sm.mbar[slot], sm.pol);
    } else {
        mbar_expect_tx(&sm.mbar[slot], 0u);
    }
}

// One row, GG lanes: Refresh Column (PH 0) or Decide (PH 1).  Returns the
// survivor flag in the group leader.  Must be called by all lanes.
// PUSH (single GPU): the column pass also does the edge work of Decide.
// A row whose M_w becomes OUT marks every w' in N[w] (oflag: "some
// neighbour has M = OUT", the first test of P:98-100); otherwise it counts
// itself for its argmin a (cnt[a]; "forall w: M_w = T_a" of P:101-103 holds
// iff cnt[a] = |N[a] ∩ active|).  Sound because a vertex still undecided at
// iteration i has every active neighbour in worklist_2 (a neighbour that
// left it earlier had M = OUT and made the vertex OUT then), so every
// neighbour's M of iteration i is either pushed or counted.  Decide then
// touches no edges (decide_push).
__device__ __forceinline__ void push_out(const MisParams& p, const int32_t* x, int len, int sub, int stride) {
    for (int j = sub; j < len; j += stride) p.oflag[x[j]] = 1;
}

template <int GG, int PH, bool PUSH>
__device__ __forceinline__ bool process_row(const MisParams& p, bool act, int sub, int64_t v, const int32_t* x,
                                            int len, uint64_t tv, int it, uint64_t fi_next) {
    bool keep = false;
    if (PH == 0) {
        uint32_t mf;
        int dc = 0;
#if MIS2_K32
        if (p.K && s_use_keys && !(PUSH && it == 0 && p.labels)) {
            // keys (single GPU: local ids are global ids)
            uint32_t km = 0xffffffffu;
            int32_t am = -1;
            int tie = 0;
            if (act && sub == 0) {  // closed neighbourhood (Q1)
                km = kkey(tv);
                am = (int32_t)v;
            }
            if (act && len > 0) {
                if (PUSH && it == 0) row_min_k32<GG>(p.K, x, len, sub, km, am, tie, (int32_t)v, &dc);
                else row_min_k32<GG>(p.K, x, len, sub, km, am, tie);
            }
            group_min_k32<GG>(km, am, tie);
            const bool decided = km == 0u || km == 0xffffffffu;
            const bool tie_real = act && tie && !decided;
            mf = decided ? kM_OUT : (uint32_t)am + 1u;
            if (__any_sync(kFull, tie_real)) {  // equal keys: the full words decide
                uint64_t m = (tie_real && sub == 0) ? tv : kOUT;
                if (tie_real && len > 0) m = row_min<GG>(p.T, x, len, sub, m);
                m = group_min<GG>(m);
                if (tie_real) mf = m_field(m, p.id_mask);
            }
        } else
#endif
        if (p.K && s_use_keys && !(PUSH && it == 0 && p.labels)) {
            // keys (single GPU: local ids are global ids)
            uint64_t k1 = ~0ull, k2 = ~0ull;
            if (act && sub == 0) {  // closed neighbourhood (Q1)
                k1 = key_lo(kkey(tv), (uint32_t)v);
                k2 = key_hi(kkey(tv), (uint32_t)v);
            }
            if (act && len > 0) {
                if (PUSH && it == 0) row_min_keys<GG>(p.K, x, len, sub, k1, k2, (int32_t)v, &dc);  // [v in its row]
                else row_min_keys<GG>(p.K, x, len, sub, k1, k2);
            }
            k1 = group_min<GG>(k1);
            k2 = group_min<GG>(k2);
            const uint32_t kmin = (uint32_t)(k1 >> 32);
            const bool tie = act && kmin != 0u && kmin != 0xffffffffu && (uint32_t)k1 != ~(uint32_t)k2;
            mf = (kmin == 0u || kmin == 0xffffffffu) ? kM_OUT : (uint32_t)k1 + 1u;
            if (__any_sync(kFull, tie)) {  // equal keys: the full words decide
                uint64_t m = (tie && sub == 0) ? tv : kOUT;
                if (tie && len > 0) m = row_min<GG>(p.T, x, len, sub, m);
                m = group_min<GG>(m);
                if (tie) mf = m_field(m, p.id_mask);
            }
        } else {
            uint64_t m = (act && sub == 0) ? tv : kOUT;  // closed neighbourhood (Q1)
            if (act && len > 0) {
                if (PUSH && it == 0 && p.labels) {  // also |N[v] ∩ active| for the push-form Decide
                    m = row_min_deg<GG>(p.T, x, len, sub, m, v, dc);  // self = this row (local index)
                } else if (PUSH && it == 0) {       // |N[v]| = len + 1 - [v in its own row]
                    m = row_min_self<GG>(p.T, x, len, sub, m, (int32_t)v, dc);
                } else {
                    m = row_min<GG>(p.T, x, len, sub, m);
                }
            }
            m = group_min<GG>(m);
            mf = m_field(m, p.id_mask);
        }
        if (PUSH) {
            // the warp pushes its OUT rows one after another, 32 entries at a time
            const int lane = threadIdx.x & 31;
            unsigned bal = __ballot_sync(kFull, act && sub == 0 && mf == kM_OUT);
            while (bal) {
                const int l = __ffs(bal) - 1;
                bal &= bal - 1;
                const int32_t* xr = reinterpret_cast<const int32_t*>(
                    __shfl_sync(kFull, reinterpret_cast<unsigned long long>(x), l));
                const int lr = __shfl_sync(kFull, len, l);
                push_out(p, xr, lr, lane, 32);
                if (lane == l) p.oflag[v] = 1;
            }
            // count for the argmin; rows of a warp sharing one argmin add together
            const bool cnt_me = act && sub == 0 && mf != kM_OUT;
            const uint32_t key = cnt_me ? mf - 1u : (0x80000000u | (threadIdx.x & 31));
            const unsigned grp = __match_any_sync(kFull, key);
            if (cnt_me && (threadIdx.x & 31) == __ffs(grp) - 1)
                atomicAdd(&p.cnt[row_of_id(p, (int64_t)key)], (uint32_t)__popc(grp));
            if (it == 0) {  // |N[v] ∩ active| (closed; masked: counted, unmasked: from the row length)
                if (p.labels) {
                    dc = group_sum<GG>(dc);
                    if (act && sub == 0) p.degc[v] = (uint32_t)dc + 1u;
                } else {
                    dc = group_or<GG>(dc);
                    if (act && sub == 0) p.degc[v] = (uint32_t)(len + 1 - (dc ? 1 : 0));
                }
            }
        }
        if (act && sub == 0) {
            p.M[v] = mf;
            keep = (mf != kM_OUT);
        }
    } else {
        int any_out = 0, all_eq = 1;
        const uint32_t vid1 = (uint32_t)gid_of(p, v) + 1u;
        if (act) {
            if (sub == 0) decide_acc(p.M[v], vid1, any_out, all_eq);
            if (len > 0) row_decide<GG>(p.M, x, len, sub, vid1, any_out, all_eq);
        }
        any_out = group_or<GG>(any_out);
        all_eq = group_and<GG>(all_eq);
        if (act && sub == 0) keep = decide_write(p, v, any_out, all_eq, it, fi_next);
    }
    return keep;
}

// defer a long row to whole-block processing (group leader decides, group agrees)
#ifndef MIS2_HUGE_ROW
#define MIS2_HUGE_ROW 32768
#endif
constexpr int kHugeRow = MIS2_HUGE_ROW;
// Global queue of deferred rows (MIS2_GQ, skewed graphs, p.gq): the rows a
// block defers are published to one queue after its steps and drained by
// every warp (rows for a whole block by whole blocks, first), so the long
// rows of a power-law graph no longer pile up on the blocks that own them
// (C4: deferred entries per block 1.03 M median, 1.53 M max).  Two extra
// grid barriers per phase; the owner appends its survivors afterwards.
#ifndef MIS2_GQ
#define MIS2_GQ 0
#endif
#ifndef MIS2_GQ_CHUNK
#define MIS2_GQ_CHUNK 4  // C4, rows per grab 1 / 2 / 4 / 8 / 16 / 64: 29.8 / 28.4 / 28.3 / 28.4 / 28.5 / 29.3 ms
#endif
constexpr int kGqChunk = MIS2_GQ_CHUNK;  // rows per warp grab
template <int GG>
__device__ __forceinline__ bool defer_long(TileSmem& sm, const MisParams& p, int64_t seg, bool act, int sub,
                                           int64_t v, int64_t len, bool gq_phase = false) {
    bool defer = false;
    if (act && sub == 0 && len > (p.heavy_batches > 0 ? p.heavy_batches * GG * gather_batch<GG>() : heavy_len<GG>())) {
        const int h = atomicAdd(&sm.hcount, 1);
        // at most one entry per row of the block's segment; with the global
        // queue (MIS2_GQ) rows for a whole block are marked ~v
        p.heavy[seg + h] = (MIS2_GQ && gq_phase && p.gq && s_gq_on && len > kHugeRow) ? ~(int32_t)v : (int32_t)v;
        defer = true;
    }
    return __shfl_sync(kFull, defer, (threadIdx.x & 31) & ~(GG - 1));
}

// Deferred long rows, stats flush, survivor count.  The block reduces all its
// deferred rows together: up to 256 rows per round, their entries flattened
// (prefix of the row lengths), 8 independent gathers per thread per pass,
// combined per row with shared-memory atomics (min is exact in any order;
// exists / forall likewise).
// One deferred (long) row reduced by NT cooperating threads -- a warp
// (NT = 32) or the whole block (NT = kMB) -- each issuing 8 independent,
// coalesced colinds loads and 8 gathers per pass (indices clamped to the
// row's last entry: min / exists / forall are idempotent).  Writes the row's
// result like process_row; returns the survivor flag (valid in thread 0 of
// the group).  All NT threads must call it.
template <int NT>
__device__ __forceinline__ uint64_t nt_min(TileSmem& sm, uint64_t x) {
    if (NT == 32) return group_min<32>(x);
    return block_min_u64(sm, x);
}
template <int NT>
__device__ __forceinline__ int nt_sum(TileSmem& sm, int x) {
    if (NT == 32) return group_sum<32>(x);
    return (int)block_sum_int(sm, x);
}
template <int NT, bool STATS, int PH, bool PUSH>
__device__ bool heavy_row(TileSmem& sm, const MisParams& p, int it, uint64_t fi_next, int64_t v, Stat& st,
                          unsigned tag) {
    const int tid = NT == 32 ? (threadIdx.x & 31) : threadIdx.x;
    const int64_t s = p.rowptr[v], len = p.rowptr[v + 1] - s;
    const int32_t* x = p.colinds + s;
    const int64_t last = len - 1;
    bool keep = false;
    if (STATS) {
        stat_row<STATS>(p, tag, v, tid == 0, len, st);
        stat_nbrs<STATS>(p, tag, x, len, tid, NT, st);
    }
    if (PH == 0) {
        const uint64_t tv = p.T[v];
        const bool count_deg = PUSH && it == 0 && p.labels;  // |N[v] ∩ active| (masked)
        const bool self_chk = PUSH && it == 0 && !p.labels;  // [v in its own row]: |N[v]| = len + 1 - it
        const bool keys = p.K && s_use_keys && !count_deg;
        uint32_t mf;
        int dc = 0, has = 0;
        bool exact = !keys;
        if (keys) {
            uint64_t k1 = tid == 0 ? key_lo(kkey(tv), (uint32_t)v) : ~0ull;
            uint64_t k2 = tid == 0 ? key_hi(kkey(tv), (uint32_t)v) : ~0ull;
            for (int64_t j = tid; j < len; j += (int64_t)NT * 8) {
                int32_t ww[8];
                uint32_t kk[8];
#pragma unroll
                for (int u = 0; u < 8; u++) ww[u] = x[min(j + (int64_t)u * NT, last)];
#pragma unroll
                for (int u = 0; u < 8; u++) kk[u] = ld_keep(p.K + ww[u], s_keep_pol);
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const uint64_t a = key_lo(kk[u], (uint32_t)ww[u]), b = key_hi(kk[u], (uint32_t)ww[u]);
                    k1 = a < k1 ? a : k1;
                    k2 = b < k2 ? b : k2;
                    if (self_chk) has |= (int64_t)ww[u] == v;
                }
            }
            k1 = nt_min<NT>(sm, k1);
            k2 = nt_min<NT>(sm, k2);
            const uint32_t kmin = (uint32_t)(k1 >> 32);
            mf = (kmin == 0u || kmin == 0xffffffffu) ? kM_OUT : (uint32_t)k1 + 1u;
            exact = kmin != 0u && kmin != 0xffffffffu && (uint32_t)k1 != ~(uint32_t)k2;  // a key tie
        }
        if (exact) {
            uint64_t m = tid == 0 ? tv : kOUT;  // closed neighbourhood (Q1)
            for (int64_t j = tid; j < len; j += (int64_t)NT * 8) {
                int32_t ww[8];
                uint64_t tt[8];
#pragma unroll
                for (int u = 0; u < 8; u++) ww[u] = x[min(j + (int64_t)u * NT, last)];
#pragma unroll
                for (int u = 0; u < 8; u++) tt[u] = p.T[ww[u]];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    m = tt[u] < m ? tt[u] : m;
                    if (count_deg) dc += (j + (int64_t)u * NT <= last) & (tt[u] != kOUT) & ((int64_t)ww[u] != v);
                    if (self_chk) has |= (int64_t)ww[u] == v;
                }
            }
            m = nt_min<NT>(sm, m);
            mf = m_field(m, p.id_mask);
            if (count_deg) dc = nt_sum<NT>(sm, dc);
        }
        if (PUSH) {
            if (mf == kM_OUT) {  // mark N[v] (push-form Decide)
                for (int64_t j = tid; j < len; j += NT) p.oflag[x[j]] = 1;
                if (tid == 0) p.oflag[v] = 1;
            } else if (tid == 0) {
                atomicAdd(&p.cnt[row_of_id(p, (int64_t)(mf - 1u))], 1u);
            }
            if (self_chk) has = nt_sum<NT>(sm, has) > 0;
            if (count_deg && tid == 0) p.degc[v] = (uint32_t)dc + 1u;
            if (self_chk && tid == 0) p.degc[v] = (uint32_t)(len + 1 - has);
        }
        if (tid == 0) {
            p.M[v] = mf;
            keep = mf != kM_OUT;
        }
    } else {
        const uint32_t vid1 = (uint32_t)gid_of(p, v) + 1u;
        int any_out = 0, all_eq = 1;
        if (tid == 0) decide_acc(p.M[v], vid1, any_out, all_eq);
        for (int64_t j = tid; j < len; j += (int64_t)NT * 8) {
            uint32_t mm[8];
#pragma unroll
            for (int u = 0; u < 8; u++) mm[u] = ld_keep(p.M + x[min(j + (int64_t)u * NT, last)], s_keep_pol);
#pragma unroll
            for (int u = 0; u < 8; u++) decide_acc(mm[u], vid1, any_out, all_eq);
            if (any_out) break;  // the row is OUT whatever follows
        }
        any_out = nt_sum<NT>(sm, any_out) > 0;
        all_eq = nt_sum<NT>(sm, !all_eq) == 0;
        if (tid == 0) keep = decide_write(p, v, any_out, all_eq, it, fi_next);
    }
    return keep;
}

// Deferred long rows, stats flush, survivor count.  Warps take deferred rows
// from a shared counter and reduce one row each; rows longer than
// kHugeRow are reduced afterwards by the whole block, one at a time.

template <bool STATS, int PH, bool PUSH>
__device__ int finish_phase(TileSmem& sm, const MisParams& p, int it, int64_t seg, int32_t* lout, uint64_t fi_next,
                            Stat& st) {
    const int t = threadIdx.x, lane = t & 31;
    const unsigned tag = 2u * (unsigned)it + 1u + (unsigned)PH;
    __syncthreads();
    const int nh = sm.hcount;
    const bool dbg = p.timeline && it == p.dbg_it && PH == p.dbg_ph && t == 0;
    long long* dbuf = reinterpret_cast<long long*>(p.mark) + (int64_t)blockIdx.x * 64;
    if (dbg) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        dbuf[60] = (long long)ns;
        dbuf[61] = nh;
    }
    int32_t* huge = sm.buf[0];  // rows for the whole block (<= nh <= the buffer)
#if MIS2_GQ
    // column passes only: a Decide's deferred rows mostly stop at their first
    // OUT neighbour, and their grabs cost more than the balance saves (C4
    // Decide 3: 1.09 -> 1.12 ms with the queue)
    if (!STATS && PH == 0 && p.gq && s_gq_on) {  // (s_gq_on is 0 in STATS kernels: defer_long marks no row)
        unsigned long long* qc = p.ctrl + 64;  // [0] rows, [1] warp head, [2] whole-block rows, [3] block head
        unsigned int* gbar = (unsigned int*)&p.ctrl[0];
        // publish: counts of the two kinds, one reservation each
        int nhb = 0;
        for (int i = t; i < nh; i += kMB) nhb += p.heavy[seg + i] < 0;
        const int nhuge_blk = (int)block_sum_int(sm, nhb);
        __shared__ unsigned long long s_base[2];
        if (t == 0) {
            s_base[0] = nh - nhuge_blk ? atomicAdd(&qc[0], (unsigned long long)(nh - nhuge_blk)) : 0ull;
            s_base[1] = nhuge_blk ? atomicAdd(&qc[2], (unsigned long long)nhuge_blk) : 0ull;
            sm.hnext = 0;
            sm.nhuge = 0;
        }
        __syncthreads();
        for (int i = t; i < nh; i += kMB) {
            const int32_t x = p.heavy[seg + i];
            if (x >= 0) p.gq[s_base[0] + atomicAdd(&sm.hnext, 1)] = x;
            else p.gq[p.n - 1 - (int64_t)(s_base[1] + atomicAdd(&sm.nhuge, 1))] = ~x;  // from the end
        }
        grid_barrier(gbar);  // every block's deferred rows are in the queue
        const int64_t nq = (int64_t)*(volatile unsigned long long*)&qc[0];
        const int64_t nqh = (int64_t)*(volatile unsigned long long*)&qc[2];
        // whole-block rows first, a block at a time
        __shared__ long long s_k;
        for (;;) {
            if (t == 0) s_k = (long long)atomicAdd(&qc[3], 1ull);
            __syncthreads();
            const int64_t k = s_k;
            __syncthreads();
            if (k >= nqh) break;
            const int64_t v = p.gq[p.n - 1 - k];
            heavy_row<kMB, STATS, PH, PUSH>(sm, p, it, fi_next, v, st, tag);
        }
        // the rest, a warp per row, kGqChunk rows per grab
        for (;;) {
            long long k0 = 0;
            if (lane == 0) k0 = (long long)atomicAdd(&qc[1], (unsigned long long)kGqChunk);
            k0 = __shfl_sync(kFull, k0, 0);
            if (k0 >= nq) break;
            const int64_t k1 = k0 + kGqChunk < nq ? k0 + kGqChunk : nq;
            for (int64_t k = k0; k < k1; k++) heavy_row<32, STATS, PH, PUSH>(sm, p, it, fi_next, p.gq[k], st, tag);
        }
        grid_barrier(gbar);  // every deferred row has its result
        // the owner keeps its survivors: M_v != OUT (column) / T_v undecided (Decide)
        for (int base = 0; base < nh; base += kMB) {
            const int i = base + t;
            bool keep = false;
            int32_t v = 0;
            if (i < nh) {
                const int32_t x = p.heavy[seg + i];
                v = x < 0 ? ~x : x;
                if (PH == 0) keep = p.M[v] != kM_OUT;
                else {
                    const uint64_t tv = p.T[v];
                    keep = tv != kIN && tv != kOUT;
                }
            }
            append(sm, keep, v, lout, seg);
        }
        if (blockIdx.x == 0 && t == 0) {  // the queue is empty for the next phase (after its barrier)
            qc[0] = qc[1] = qc[2] = qc[3] = 0ull;
        }
    } else
#endif
    if (nh > 0) {
        if (t == 0) {
            sm.hnext = 0;
            sm.nhuge = 0;
        }
        __syncthreads();
        for (;;) {
            int i = 0;
            if (lane == 0) i = atomicAdd(&sm.hnext, 1);
            i = __shfl_sync(kFull, i, 0);
            if (i >= nh) break;
            const int64_t v = p.heavy[seg + i];
            const int64_t len = p.rowptr[v + 1] - p.rowptr[v];
            if (len > kHugeRow && nh <= 2 * kTileCap) {
                if (lane == 0) huge[atomicAdd(&sm.nhuge, 1)] = (int32_t)v;
                continue;
            }
            const bool keep = heavy_row<32, STATS, PH, PUSH>(sm, p, it, fi_next, v, st, tag);
            append(sm, keep && lane == 0, (int32_t)v, lout, seg);
        }
        __syncthreads();
        const int nb = sm.nhuge;
        for (int k = 0; k < nb; k++) {
            const int64_t v = huge[k];
            const bool keep = heavy_row<kMB, STATS, PH, PUSH>(sm, p, it, fi_next, v, st, tag);
            append(sm, keep && t == 0, (int32_t)v, lout, seg);
        }
    }
    stats_flush<STATS>(p, it, PH == 0 ? 1 : 0, st);
    if (dbg) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        dbuf[62] = (long long)ns;
        long long e = 0;
        for (int i = 0; i < nh; i++) {
            const int64_t v = p.heavy[seg + i];
            e += p.rowptr[v + 1] - p.rowptr[v];
        }
        dbuf[63] = e;
    }
    __syncthreads();
    // no trailing barrier: every caller's next step is a barrier (grid or
    // partition sync, halo push) before sm.cnt is written again
    const int out = sm.cnt;
    return out;
}

// ------------------------------------------------------------ dense phase
// Consecutive rows of the block range, RPB = kMB/G per step; the step's
// colinds span is bulk-copied into shared memory one step ahead.
// PH = 0: Refresh Column over worklist_2 (M_v != OUT, active)
// PH = 1: Decide over worklist_1 (T_v undecided)
//
// Every phase is split into a prologue (*_begin: the first tile's bulk copy,
// the first rows' bounds and own status words) and the steps (*_run).  The
// prologue reads only static CSR data and words of the block's OWN rows,
// which only this block writes, so the persistent kernel issues it between
// its arrival at the grid barrier that precedes the phase and its wait
// (grid_arrive_sum / grid_wait_sum): the copy and the loads land while the
// block waits for the others, and the phase's first step starts with its
// data in shared memory instead of after three dependent memory round trips
// (C2 356 -> 348 us).
// The state is parked in the idle second staging buffer (buf[1], written
// by the copy of step 1 only after the run's first __syncthreads), so no
// register stays live across the barrier; thread 0's bounds of the dense
// step after next live in TileSmem.
struct PhaseState {
    int64_t s;    // rowptr of the row: dense, this thread's row of step 0; sparse, the leader's row of tile 1
    uint64_t tv;  // its T_v
    int32_t len;  // its length
    int32_t x;    // dense: its M_v (id field); sparse: the row of tile 1 (-1: none)
    int32_t y;    // sparse: the leader's row of tile 2 (-1: none)
    int32_t pending;  // 0 none, 1 dense tile 0 issued, 2 sparse tile 0 issued
};

__device__ __forceinline__ PhaseState* park(TileSmem& sm) {
    return reinterpret_cast<PhaseState*>(sm.buf[1]) + threadIdx.x;
}
static_assert(sizeof(PhaseState) * kMB <= sizeof(int32_t) * kTileCap, "PhaseState park");

// fresh: the first Refresh Column of an unmasked call (M not initialised,
// every row active)
template <int G, int PH>
__device__ __forceinline__ void dense_begin(TileSmem& sm, const MisParams& p, const Rows& rows, bool fresh = false) {
    PhaseState ps;
    const int t = threadIdx.x, g = t / G;
    if (t == 0) {
        // buf[0] held the huge-row list or the halo scan (generic writes)
        // before the bulk copy refills it
        if (sm.nhuge || sm.gen0) fence_proxy_async();
        sm.nhuge = 0;
        sm.gen0 = 0;
        sm.cnt = 0;
        sm.hcount = 0;
    }
    const int64_t nsteps = rows.nruns;
    if (t == 0 && nsteps > 0) {
        int64_t nx_s = 0, nx_e = 0;
        if (nsteps > 1) {
            nx_s = p.rowptr[rows.run_lo(1)];
            nx_e = p.rowptr[rows.run_hi(1)];
        }
        sm.nx_s = nx_s;
        sm.nx_e = nx_e;
        stage_tile(sm, p, 0, p.rowptr[rows.run_lo(0)], p.rowptr[rows.run_hi(0)]);
    }
    ps.s = 0;
    ps.len = 0;
    ps.tv = kOUT;
    ps.x = (int32_t)kM_OUT;
    ps.y = -1;
    if (nsteps > 0 && rows.run_lo(0) + g < rows.run_hi(0)) {
        const int64_t v0 = rows.run_lo(0) + g;
        ps.s = p.rowptr[v0];
        ps.len = (int32_t)(p.rowptr[v0 + 1] - ps.s);
        ps.tv = p.T[v0];
        if (PH == 0) ps.x = fresh ? (int32_t)kPending : (int32_t)p.M[v0];
    }
    ps.pending = nsteps > 0 ? 1 : 0;
    if (t == 0) sm.pending = ps.pending;
    *park(sm) = ps;
}

template <int G, bool STATS, int PH, bool PUSH = false>
__device__ int dense_run(TileSmem& sm, const MisParams& p, int it, const Rows& rows, int32_t* lout, uint32_t& ph,
                         uint64_t fi_next, bool fresh = false) {
    const PhaseState ps = *park(sm);  // before the first __syncthreads (step 1's copy refills buf[1])
    const int t = threadIdx.x, g = t / G, sub = t % G;
    const unsigned tag = 2u * (unsigned)it + 1u + (unsigned)PH;
    Stat st;
    const int64_t nsteps = rows.nruns;  // step k = run k of the block's rows (<= kMB / G rows)
    int64_t nx_s = 0, nx_e = 0;  // bounds of the next tile (thread 0), prefetched a step ahead
    if (t == 0) {
        nx_s = sm.nx_s;
        nx_e = sm.nx_e;
    }
    const bool dbg = p.timeline && it == p.dbg_it && PH == p.dbg_ph && threadIdx.x == 0;
    long long* dbuf = reinterpret_cast<long long*>(p.mark) + (int64_t)blockIdx.x * 64;
    auto gt = []() {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        return (long long)ns;
    };
    if (dbg) {
        dbuf[0] = gt();
        dbuf[1] = nsteps;
        dbuf[2] = rows.count;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        dbuf[59] = smid;
    }
    // prefetched row bounds / status of the next tile (this thread's row)
    int64_t ns0 = ps.s, ne0 = ps.s + ps.len;
    uint64_t ntv = ps.tv;
    uint32_t nmv = (uint32_t)ps.x;
    for (int64_t k = 0; k < nsteps; k++) {
        const int slot = (int)(k & 1);
        if (dbg && k < 12) dbuf[4 + 5 * k] = gt();
        __syncthreads();  // tile k-1 consumed: its buffer may be refilled
        if (dbg && k < 12) dbuf[4 + 5 * k + 1] = gt();
        if (t == 0 && k + 1 < nsteps) {
            const int64_t s1 = nx_s, e1 = nx_e;
            if (k + 2 < nsteps) {
                nx_s = p.rowptr[rows.run_lo(k + 2)];
                nx_e = p.rowptr[rows.run_hi(k + 2)];
            }
            stage_tile(sm, p, slot ^ 1, s1, e1);
        }
        // this tile's row bounds and status were loaded one step ahead; load
        // the next tile's now (a phase writes only rows of the tile it is
        // processing, so the prefetched words are current)
        const int64_t v = rows.run_lo(k) + g;
        const bool valid = v < rows.run_hi(k);
        const int64_t s = ns0, e = ne0;
        const uint64_t tv = ntv;
        bool act = false;
        if (valid) act = PH == 0 ? (nmv != kM_OUT && nmv != 0u) : (tv != kIN && tv != kOUT);
        if (k + 1 < nsteps) {
            const int64_t vn = rows.run_lo(k + 1) + g;
            if (vn < rows.run_hi(k + 1)) {
                ns0 = p.rowptr[vn];
                ne0 = p.rowptr[vn + 1];
                ntv = p.T[vn];
                if (PH == 0) nmv = fresh ? kPending : p.M[vn];
            }
        }
        const int64_t len = e - s;
        if (defer_long<G>(sm, p, rows.seg, act, sub, v, len, PH == 0)) act = false;
        if (dbg && k < 12) dbuf[4 + 5 * k + 2] = gt();
        mbar_wait(&sm.mbar[slot], (ph >> slot) & 1u);
        ph ^= 1u << slot;
        if (dbg && k < 12) dbuf[4 + 5 * k + 3] = gt();
        const int32_t* x = sm.fits[slot] ? sm.buf[slot] + (s - sm.sal[slot]) : p.colinds + s;
        const bool keep = process_row<G, PH, PUSH>(p, act, sub, v, x, (int)len, tv, it, fi_next);
        if (dbg && k < 12) dbuf[4 + 5 * k + 4] = gt();
        if (STATS && act) {
            stat_row<STATS>(p, tag, v, sub == 0, len, st);
            stat_nbrs<STATS>(p, tag, x, len, sub, G, st);
        }
        append(sm, keep, (int32_t)v, lout, rows.seg);
    }
    if (dbg) dbuf[3] = gt();
    return finish_phase<STATS, PH, PUSH>(sm, p, it, rows.seg, lout, fi_next, st);
}

template <int G, bool STATS, int PH, bool PUSH = false>
__device__ int dense_phase(TileSmem& sm, const MisParams& p, int it, const Rows& rows, int32_t* lout,
                           uint32_t& ph, uint64_t fi_next) {
    dense_begin<G, PH>(sm, p, rows);
    return dense_run<G, STATS, PH, PUSH>(sm, p, it, rows, lout, ph, fi_next);
}

// ------------------------------------------------------------ sparse phase
// Rows of the block's compacted worklist, RPBS = kMB/GS per step with
// GS = 2G lanes per row.  Each group leader bulk-copies its own row into a
// fixed shared-memory slot (16-byte aligned hull, <= SLOT entries) one step
// ahead; rows that do not fit are read from global memory.
struct __align__(16) SMeta {
    int64_t s;    // rowptr[v]
    int32_t v;    // vertex (-1: no row)
    int32_t len;  // row length; bit 30 set: staged in the slot
};
// sparse step layout of a staging buffer: row slots | SMeta per row | T_v per row
constexpr int kMaxRowsS = kMB / 2;                    // rows per sparse step (GS >= 2)
constexpr int kTvOff = kTileCap - 2 * kMaxRowsS;      // uint64 T_v per row
constexpr int kSlotRegion = kTvOff - 4 * kMaxRowsS;   // entries used for row slots; SMeta after
static_assert(kSlotRegion > 0 && (kSlotRegion % 4) == 0, "sparse layout");

// the leader of row group gs of a sparse step: its SMeta, T_v and (when the
// row fits the group's slot) the bulk copy of its colinds hull into `slot`
template <int G>
__device__ __forceinline__ void sparse_issue(TileSmem& sm, const MisParams& p, int slot, int gs, int64_t v,
                                             int64_t s, int64_t e, uint64_t tv) {
    constexpr int GS = sparse_group<G>();
    constexpr int RPBS = kMB / GS;
    constexpr int SLOT = (kSlotRegion / RPBS) & ~3;
    constexpr int kStaged = 1 << 30;
    const int64_t nnz4 = p.nnz & ~(int64_t)3;
    SMeta* meta = reinterpret_cast<SMeta*>(sm.buf[slot] + kSlotRegion);
    SMeta m;
    m.v = -1;
    m.s = 0;
    m.len = 0;
    uint32_t bytes = 0;
    int64_t sal = 0;
    if (v >= 0) {
        sal = s & ~(int64_t)3;
        const int64_t ecp = (e + 3) & ~(int64_t)3;
        const bool fits = (ecp - sal) <= SLOT && ecp <= nnz4;
        m.v = (int32_t)v;
        m.s = s;
        m.len = (int32_t)(e - s) | (fits ? kStaged : 0);
        if (fits && ecp > sal) bytes = (uint32_t)((ecp - sal) * 4);
    }
    meta[gs] = m;
    reinterpret_cast<uint64_t*>(sm.buf[slot] + kTvOff)[gs] = tv;
    mbar_expect_tx(&sm.mbarS[slot], bytes);
    if (bytes) bulk_g2s(sm.buf[slot] + gs * SLOT, p.colinds + sal, bytes, &sm.mbarS[slot], sm.pol);
}

// Leaders pipeline the row metadata: worklist entry of tile j+3, row bounds
// of tile j+2 and T_v of tile j+1 are loaded while tile j is processed, so
// the copy of tile j+1 is issued without waiting on loads.  The prologue
// (tile 0 issued, tiles 1 / 2 loaded) is sparse_begin.
template <int G>
__device__ __forceinline__ void sparse_begin(TileSmem& sm, const MisParams& p, int64_t seg, const int32_t* lin,
                                             int nin) {
    PhaseState ps;
    constexpr int GS = sparse_group<G>();
    constexpr int RPBS = kMB / GS;
    const int t = threadIdx.x, gs = t / GS, sub = t % GS;
    if (t == 0) {
        // buf[0] held the huge-row list or the halo scan (generic writes)
        // before the bulk copy refills it
        if (sm.nhuge || sm.gen0) fence_proxy_async();
        sm.nhuge = 0;
        sm.gen0 = 0;
        sm.cnt = 0;
        sm.hcount = 0;
    }
    const int nsteps = (nin + RPBS - 1) / RPBS;
    auto row_of = [&](int j) -> int64_t {
        const int idx = j * RPBS + gs;
        return (sub == 0 && j < nsteps && idx < nin) ? (int64_t)lin[seg + idx] : -1;
    };
    ps.x = ps.y = -1;
    ps.s = 0;
    ps.len = 0;
    ps.tv = kOUT;
    ps.pending = 0;
    if (nsteps > 0) {
        const int64_t v0 = row_of(0);
        const int64_t v1 = row_of(1);
        ps.x = (int32_t)v1;
        ps.y = (int32_t)row_of(2);
        int64_t s0 = 0, e0 = 0;
        if (v0 >= 0) {
            s0 = p.rowptr[v0];
            e0 = p.rowptr[v0 + 1];
        }
        if (v1 >= 0) {
            ps.s = p.rowptr[v1];
            ps.len = (int32_t)(p.rowptr[v1 + 1] - ps.s);
        }
        const uint64_t tv0 = v0 >= 0 ? p.T[v0] : kOUT;
        ps.tv = v1 >= 0 ? p.T[v1] : kOUT;
        if (sub == 0) sparse_issue<G>(sm, p, 0, gs, v0, s0, e0, tv0);
        ps.pending = 2;
    }
    if (t == 0) sm.pending = ps.pending;
    *park(sm) = ps;
}

template <int G, bool STATS, int PH, bool PUSH = false>
__device__ int sparse_run(TileSmem& sm, const MisParams& p, int it, int64_t seg, const int32_t* lin, int nin,
                          int32_t* lout, uint32_t& ph, uint64_t fi_next) {
    const PhaseState ps = *park(sm);  // before the first __syncthreads (tile 1's copy refills buf[1])
    constexpr int GS = sparse_group<G>();
    constexpr int RPBS = kMB / GS;
    constexpr int SLOT = (kSlotRegion / RPBS) & ~3;
    static_assert(RPBS * sizeof(SMeta) <= (kTileCap - kSlotRegion) * 4, "SMeta region too small");
    constexpr int kStaged = 1 << 30;
    const int t = threadIdx.x, gs = t / GS, sub = t % GS;
    const unsigned tag = 2u * (unsigned)it + 1u + (unsigned)PH;
    Stat st;
    const int nsteps = (nin + RPBS - 1) / RPBS;
    auto row_of = [&](int j) -> int64_t {
        const int idx = j * RPBS + gs;
        return (sub == 0 && j < nsteps && idx < nin) ? (int64_t)lin[seg + idx] : -1;
    };
    auto bounds = [&](int64_t v, int64_t& s, int64_t& e) {
        s = 0;
        e = 0;
        if (v >= 0) {
            s = p.rowptr[v];
            e = p.rowptr[v + 1];
        }
    };

    int64_t v1 = ps.x, s1 = ps.s, e1 = ps.s + ps.len, v2 = ps.y, s2 = 0, e2 = 0, v3 = -1;
    uint64_t tv1 = ps.tv, tv2 = kOUT;
    const bool dbg = p.timeline && it == p.dbg_it && PH == p.dbg_ph && threadIdx.x == 0;
    long long* dbuf = reinterpret_cast<long long*>(p.mark) + (int64_t)blockIdx.x * 64;
    auto gt = []() {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        return (long long)ns;
    };
    if (dbg) {
        dbuf[0] = gt();
        dbuf[1] = nsteps;
        dbuf[2] = nin;
    }
    for (int k = 0; k < nsteps; k++) {
        const int slot = k & 1;
        if (dbg && k < 12) dbuf[4 + 5 * k] = gt();
        __syncthreads();  // metadata of tile k visible; buffer of tile k-1 free
        if (dbg && k < 12) dbuf[4 + 5 * k + 1] = gt();
        if (k + 1 < nsteps && sub == 0) sparse_issue<G>(sm, p, slot ^ 1, gs, v1, s1, e1, tv1);  // no proxy fence needed (see stage_tile)
        bounds(v2, s2, e2);     // prefetch for tile k+2
        tv2 = v2 >= 0 ? p.T[v2] : kOUT;
        v3 = row_of(k + 3);     // prefetch for tile k+3
        const SMeta m = reinterpret_cast<const SMeta*>(sm.buf[slot] + kSlotRegion)[gs];
        const bool valid = m.v >= 0;
        const int64_t v = valid ? m.v : 0;
        const int len = m.len & ~kStaged;
        const uint64_t tv = reinterpret_cast<const uint64_t*>(sm.buf[slot] + kTvOff)[gs];
        bool act = valid;
        if (defer_long<GS>(sm, p, seg, act, sub, v, len, PH == 0)) act = false;
        if (dbg && k < 12) dbuf[4 + 5 * k + 2] = gt();
        mbar_wait(&sm.mbarS[slot], (ph >> (2 + slot)) & 1u);
        ph ^= 1u << (2 + slot);
        if (dbg && k < 12) dbuf[4 + 5 * k + 3] = gt();
        const int32_t* x = (m.len & kStaged) ? sm.buf[slot] + gs * SLOT + (m.s - (m.s & ~(int64_t)3))
                                             : p.colinds + m.s;
        const bool keep = process_row<GS, PH, PUSH>(p, act, sub, v, x, len, tv, it, fi_next);
        if (dbg && k < 12) dbuf[4 + 5 * k + 4] = gt();
        if (STATS && act) {
            stat_row<STATS>(p, tag, v, sub == 0, len, st);
            stat_nbrs<STATS>(p, tag, x, len, sub, GS, st);
        }
        append(sm, keep, (int32_t)v, lout, seg);
        v1 = v2;
        s1 = s2;
        e1 = e2;
        tv1 = tv2;
        v2 = v3;
    }
    if (dbg) dbuf[3] = gt();
    return finish_phase<STATS, PH, PUSH>(sm, p, it, seg, lout, fi_next, st);
}

template <int G, bool STATS, int PH, bool PUSH = false>
__device__ int sparse_phase(TileSmem& sm, const MisParams& p, int it, int64_t seg, const int32_t* lin, int nin,
                            int32_t* lout, uint32_t& ph, uint64_t fi_next) {
    sparse_begin<G>(sm, p, seg, lin, nin);
    return sparse_run<G, STATS, PH, PUSH>(sm, p, it, seg, lin, nin, lout, ph, fi_next);
}

// A prologue issued ahead of a phase that does not run (the loop ended):
// its bulk copy must land before the block exits.
__device__ __forceinline__ void drain_pending(TileSmem& sm, uint32_t& ph) {
    const int pending = sm.pending;
    if (pending == 1) {
        mbar_wait(&sm.mbar[0], ph & 1u);
        ph ^= 1u;
    } else if (pending == 2) {
        mbar_wait(&sm.mbarS[0], (ph >> 2) & 1u);
        ph ^= 1u << 2;
    }
}

// ------------------------------------------------------------ push-form Decide
// Decide over worklist_1 when the column pass has already done its
// edge work (process_row, PUSH): v is OUT iff some M_w = OUT for w in N[v]
// (oflag[v]); else IN iff every active w in N[v] has M_w = T_v
// (cnt[v] = degc[v]); else it stays undecided and gets its word of iteration
// it + 1 (fused Refresh Row).  No neighbour is read.  Dense: all
// rows of the block range, membership from T_v; sparse: the worklist.
template <bool STATS>
__device__ int decide_push(TileSmem& sm, const MisParams& p, int it, const Rows& rows, const int32_t* lin,
                           int nin, bool dense, int32_t* lout, uint64_t fi_next) {
    const int t = threadIdx.x;
    const unsigned tag = 2u * (unsigned)it + 2u;
    Stat st;
    if (t == 0) sm.cnt = 0;
    __syncthreads();
    const int64_t total = dense ? rows.count : (int64_t)nin;
    const bool dbg = p.timeline && it == p.dbg_it && 1 == p.dbg_ph && t == 0;
    long long* dbuf = reinterpret_cast<long long*>(p.mark) + (int64_t)blockIdx.x * 64;
    auto gt = []() {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        return (long long)ns;
    };
    if (dbg) {
        dbuf[0] = gt();
        dbuf[1] = total;
    }
    // U rows per thread per round, loads batched by dependency level.  v is
    // IN iff every active w in N[v] counted v as its argmin: cnt[v] =
    // |N[v] ∩ active| = degc[v], counted by the push-form column pass of
    // iteration 0 (closed neighbourhood; Q23: a stored diagonal is not
    // counted twice) -- no row is read here.
#ifndef MIS2_DPU
#define MIS2_DPU 2  // rows per thread per round: measured 2 / 4 / 8 / 16 -> C2 334 / 336 / 340 / 365 us (the unrolled code is fetched cold every phase)
#endif
    constexpr int U = MIS2_DPU;
    for (int64_t base = 0; base < total; base += (int64_t)kMB * U) {
        int32_t vv[U];
        uint64_t tv[U];
        uint32_t c[U], dg[U];
        uint8_t fl[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t idx = base + u * kMB + t;
            vv[u] = idx < total ? (int32_t)(dense ? rows.row_at(idx) : (int64_t)lin[rows.seg + idx]) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            tv[u] = kIN;
            fl[u] = 0;
            c[u] = 0;
            dg[u] = 0;
            if (vv[u] >= 0) {
                tv[u] = p.T[vv[u]];
                fl[u] = p.oflag[vv[u]];
                c[u] = p.cnt[vv[u]];
                dg[u] = p.degc[vv[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t v = vv[u];
            bool keep = false;
            if (v >= 0 && tv[u] != kIN && tv[u] != kOUT) {
                if (c[u]) p.cnt[v] = 0u;
                if (fl[u]) set_T(p, v, kOUT);
                else if (c[u] == dg[u]) set_IN(p, v);
                else {
#ifdef MIS2_DP_NOHASH
                    set_T(p, v, ((uint64_t)(it + 5) << 40) | (uint64_t)(v + 1));
#else
                    set_T(p, v, p.prio.word(it + 1, fi_next, gid_of(p, v)));
#endif
                    keep = true;
                }
                if (STATS) {
                    const int64_t s = p.rowptr[v], e = p.rowptr[v + 1];
                    stat_row<STATS>(p, tag, v, true, e - s, st);
                    stat_nbrs<STATS>(p, tag, p.colinds + s, e - s, 0, 1, st);
                }
            }
            append(sm, keep, (int32_t)(v < 0 ? 0 : v), lout, rows.seg);
        }
    }
    if (dbg) {
        dbuf[2] = dbuf[3] = dbuf[5] = gt();
        dbuf[4] = 0;
    }
    stats_flush<STATS>(p, it, 0, st);
    __syncthreads();
    // no trailing barrier: every caller's next step is a barrier (grid or
    // partition sync, halo push) before sm.cnt is written again
    const int out = sm.cnt;
    return out;
}

__device__ __forceinline__ void stamp(const MisParams& p, int slot) {
    if (p.timeline && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        p.timeline[slot] = (long long)ns;
    }
}

// ------------------------------------------------------------ the kernel
// PUSH: iterations it < p.push_iters use the push-form Decide (the column
// pass pushes / counts, decide_push touches no edges); all others -- and
// every iteration of a !PUSH kernel -- the pull form of Alg. 1 as written.
// The switch needs no conversion: the push state (oflag, cnt) is only
// written and read by push iterations and cnt is cleared by decide_push.
template <int G, bool STATS, bool PUSH>
__global__ void __launch_bounds__(kMB, kMinBlocksPerSM) mis2_persistent(MisParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
    const int t = threadIdx.x;
    const int64_t B = gridDim.x;
    const Rows rows = make_rows(p.n, B, blockIdx.x, kMB / G, p.cyclic != 0);
    stamp(p, 2 * p.max_iters);  // timeline: kernel entry

    if (t == 0) {
        sm.nhuge = 0;
        sm.gen0 = 0;
        sm.pending = 0;
        s_nin = 0;
        {
            uint64_t pol;
            if (p.gather_keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
            s_keep_pol = pol;
        }
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        constexpr int kRowGroups = kMB / sparse_group<G>();
        mbar_init(&sm.mbarS[0], kRowGroups);
        mbar_init(&sm.mbarS[1], kRowGroups);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sm.pol = l2_policy(p, rows);
    }
    uint32_t ph = 0u;  // mbarrier phase bits: 0,1 dense buffers; 2,3 sparse buffers

    // worklists <- 0..|V|; Refresh Row of iteration 0.
    // A masked call (phase 2 of Alg. 3) also lists its active rows, so its
    // first passes can be sparse (the active rows are a small fraction).
    int act_block = 0;
    {
        const uint64_t fi0 = p.prio.iter_term(0);
        int act_cnt = 0;
        int64_t maxdeg = 0;
        if (t == 0) sm.cnt = 0;
        __syncthreads();
        for (int64_t base = 0; base < rows.count; base += kMB) {
            const bool in = base + t < rows.count;
            const int64_t v = in ? rows.row_at(base + t) : 0;
            const bool act = in && (p.labels ? (p.labels[v] < 0) : true);
            if (in) {
                set_T(p, v, act ? p.prio.word(0, fi0, gid_of(p, v)) : kOUT);
                // M: the first column pass of an unmasked call takes every
                // row without reading M (`fresh`); a masked one marks the
                // inactive rows (0 = inactive sentinel, reading Q15)
                if (p.labels) p.M[v] = act ? kPending : 0u;
                p.oflag[v] = 0;
                p.cnt[v] = 0u;
                p.in_set[v] = 0;
                if (p.K && !p.keys_mode) maxdeg = max(maxdeg, p.rowptr[v + 1] - p.rowptr[v]);
            }
            act_cnt += act;
            if (p.labels) {  // worklist_1 = worklist_2 = the active rows
                const unsigned ball = __ballot_sync(kFull, act);
                if (ball) {
                    const int lane = t & 31, leader = __ffs(ball) - 1;
                    int pos = 0;
                    if (lane == leader) pos = atomicAdd(&sm.cnt, __popc(ball));
                    pos = __shfl_sync(kFull, pos, leader);
                    if (act) {
                        const int64_t at = rows.seg + pos + __popc(ball & lanemask_lt());
                        p.L1[0][at] = (int32_t)v;
                        p.L2[0][at] = (int32_t)v;
                    }
                }
            }
        }
        const long long s = block_sum_int(sm, act_cnt);
        act_block = (int)s;
        if (p.K && !p.keys_mode) {
            const uint64_t bm = ~block_min_u64(sm, ~(uint64_t)maxdeg);  // block max
            if (t == 0 && bm) atomicMax(&p.ctrl[8], (unsigned long long)bm);
        }
    }
    const int64_t range = rows.count;
    // this block's worklist segment sizes (a masked call starts from its lists)
    int cnt1 = p.labels ? act_block : (int)range, cnt2 = cnt1;
    __shared__ SumBarrier sb;
    if (t == 0) {
        sb.last[0] = sb.last[1] = 0ull;
        sb.k = 0u;
    }
    __shared__ unsigned long long s_sum;
    unsigned long long* sumc = &p.ctrl[16];
    // Every phase's prologue (PhaseState: its first tile's bulk copy, its
    // first rows' bounds and own status words) is issued between this
    // block's barrier arrival and its wait, so it lands while the other
    // blocks finish the previous phase.
    auto col_begin = [&](int i, int c2, const int32_t* l2) {
        if ((i == 0 && !p.labels) || (int64_t)c2 * kDenseDen >= range * kDenseNum)
            dense_begin<G, 0>(sm, p, rows, i == 0 && !p.labels);
        else sparse_begin<G>(sm, p, rows.seg, l2, c2);
    };
    unsigned long long bold = grid_arrive_sum(sumc, sb, (unsigned long long)act_block);
    if (MIS2_HOIST) col_begin(0, cnt2, p.L2[0]);  // own rows: written above by this block
    const unsigned long long n_active = grid_wait_sum(sumc, sb, bold, &s_sum);
    if (!MIS2_HOIST) col_begin(0, cnt2, p.L2[0]);
    stamp(p, 0);
    // 32-bit column keys for skewed degree distributions: random neighbour
    // ids gather from all of T, which does not stay in L2 (C4); on meshes the
    // extra key arithmetic costs more than the halved bytes save
    if (t == 0) {
        int use = 0;
        if (p.K) use = p.keys_mode ? 1 : (double)ld_acquire_u64(&p.ctrl[8]) > 16.0 * (double)p.nnz / (double)p.n;
        s_use_keys = use;
        s_gq_on = !STATS && p.gq != nullptr && n_active * 64ull > (unsigned long long)p.n;
    }
    __syncthreads();

    int it = 0;
    int status = MIS2_OK;
    const bool skip_loop = n_active == 0;
    while (!skip_loop) {  // while worklist_1 != {}
        const int cur = it & 1;
        // ---- Refresh Column over worklist_2; its prologue was issued
        const bool push = PUSH && it < p.push_iters;
        const bool dense2 = (it == 0 && !p.labels) || (int64_t)cnt2 * kDenseDen >= range * kDenseNum;
        const bool fresh = it == 0 && !p.labels;
        if (push) {
            cnt2 = dense2 ? dense_run<G, STATS, 0, PUSH>(sm, p, it, rows, p.L2[cur ^ 1], ph, 0, fresh)
                          : sparse_run<G, STATS, 0, PUSH>(sm, p, it, rows.seg, p.L2[cur], cnt2, p.L2[cur ^ 1], ph, 0);
        } else {
            cnt2 = dense2 ? dense_run<G, STATS, 0, false>(sm, p, it, rows, p.L2[cur ^ 1], ph, 0, fresh)
                          : sparse_run<G, STATS, 0, false>(sm, p, it, rows.seg, p.L2[cur], cnt2, p.L2[cur ^ 1], ph, 0);
        }
        if (t == 0) sm.pending = 0;
        // prologue of Decide (pull form: its rows' colinds and own T_v)
        const bool dense1 = (it == 0 && !p.labels) || (int64_t)cnt1 * kDenseDen >= range * kDenseNum;
        auto dec_begin = [&]() {
            if (push) return;
            if (dense1) dense_begin<G, 1>(sm, p, rows);
            else sparse_begin<G>(sm, p, rows.seg, p.L1[cur], cnt1);
        };
        bold = grid_arrive_sum(sumc, sb, 0ull);
        if (MIS2_HOIST) dec_begin();
        grid_wait_sum(sumc, sb, bold, &s_sum);
        if (!MIS2_HOIST) dec_begin();
        stamp(p, 1 + 2 * it);
        // ---- Decide over worklist_1 + fused refresh of iteration it+1
        const uint64_t fi_next = p.prio.iter_term(it + 1);
        if (push) cnt1 = decide_push<STATS>(sm, p, it, rows, p.L1[cur], cnt1, dense1, p.L1[cur ^ 1], fi_next);
        else if (dense1) cnt1 = dense_run<G, STATS, 1>(sm, p, it, rows, p.L1[cur ^ 1], ph, fi_next);
        else cnt1 = sparse_run<G, STATS, 1>(sm, p, it, rows.seg, p.L1[cur], cnt1, p.L1[cur ^ 1], ph, fi_next);
        if (t == 0) sm.pending = 0;
        // the loop condition rides on the barrier; the next Refresh Column's
        // prologue is issued even if the loop ends (drained below)
        // the IN decisions of this Decide go to the count beside the barrier
        __shared__ int s_nin_rep;
        if (it == 0 && t == 0) s_nin_rep = 0;
        bold = grid_arrive_sum(sumc, sb, (unsigned long long)cnt1, &p.ctrl[5],
                               t == 0 ? (unsigned long long)(s_nin - s_nin_rep) : 0ull);
        if (t == 0) s_nin_rep = s_nin;
        if (MIS2_HOIST) col_begin(it + 1, cnt2, p.L2[cur ^ 1]);
        const unsigned long long remaining = grid_wait_sum(sumc, sb, bold, &s_sum);
        // the queue's two extra barriers pay only while many rows remain
        if (t == 0) s_gq_on = !STATS && p.gq != nullptr && remaining * 64ull > (unsigned long long)p.n;
        stamp(p, 2 + 2 * it);
        it++;
        if (remaining == 0) break;
        if (it >= p.max_iters) {  // reading Q12
            status = MIS2_ENOTCONVERGED;
            break;
        }
        if (!MIS2_HOIST) col_begin(it, cnt2, p.L2[cur ^ 1]);  // it already advanced
    }
    __syncthreads();
    drain_pending(sm, ph);

    // return {v : T_v = IN}: the mask was written at the decisions
    // (set_IN) and every Decide's IN count was added beside its barrier, so
    // after the last barrier the count is complete: block 0 publishes
    if (blockIdx.x == 0 && t == 0) {
        *p.d_count = (int64_t)ld_acquire_u64(&p.ctrl[5]);
        *p.d_iters = it;
        *p.d_status = status;
        if (p.timeline) {  // timeline: kernel end (of block 0)
            unsigned long long ns;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
            p.timeline[2 * p.max_iters + 1] = (long long)ns;
        }
    }
    l2_release(p, rows);
}

// ------------------------------------------------------------ partitioned kernel
// Alg. 1 over a 1-D row partition as ONE persistent kernel
// per GPU: every phase of the single-GPU kernel runs on the partition's own
// rows, the halo values are pushed by the kernel itself -- after Refresh
// Column the M words, after Decide the T words of the owned rows other
// partitions hold as ghosts are stored straight into those partitions' ghost
// slots (peer memory over NVLink, or another buffer of this GPU for the
// local transport) -- and partitions meet at a barrier whose mailboxes carry
// the per-partition counts, so the loop condition |worklist_1| = 0 is
// evaluated on the device: no host round trip per iteration.  P:117 (each
// phase reads only the previous phase's arrays) makes any partition
// bit-identical to one GPU: global ids in the hash, the global n in b.
//
// One launch holds one or several local partitions (the local transport
// runs all P of them in one cooperative grid, so a partition barrier never
// waits for a partition that is not resident); partition i's blocks are
// [blk0, blk0 + nblk).
constexpr int kMaxParts = 64;
struct PartK {
    MisParams mp;                     // n = owned rows; T / M over [owned | ghosts]; contiguous Rows
    int blk0, nblk;                   // this partition's blocks in the grid
    int gpart;                        // global partition id
    int64_t nsend;                    // halo entries: owned row send_src[i] -> partition send_peer[i], slot send_dst[i]
    const int64_t* send_csp;          // entries of owned rows [8c, 8c + 8): [send_csp[c], send_csp[c + 1]) (sorted by row)
    const int32_t* send_src;
    const int32_t* send_peer;
    const int64_t* send_dst;          // index into the peer's T / M arrays (its ghost region)
    unsigned int* bar;                // sub-grid barrier counter of this partition
    unsigned long long* acc;          // [2] per-epoch sum of the partition's block contributions
    unsigned long long* box;          // [2][P] mailbox: box[e & 1][q] = e << 32 | value of partition q
    unsigned long long* rel;          // leader -> blocks: e << 32 | sum over partitions
};
struct PeerTab {
    int P;                            // partitions in total (all ranks)
    int sys;                          // peers on other GPUs: system-scope fences / mailbox accesses
    uint64_t* T[kMaxParts];           // partition q's T (peer / local address)
    uint32_t* M[kMaxParts];
    unsigned long long* box[kMaxParts];
};

// sense-flip barrier over the nblk blocks of one partition (lb = block index in it)
__device__ __forceinline__ void part_barrier(unsigned int* bar, int lb, int nblk) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int nb = (lb == 0) ? (0x80000000u - (unsigned)(nblk - 1)) : 1u;
        unsigned int old, cur;
        asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
        for (;;) {
            asm volatile("ld.relaxed.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
            if ((old ^ cur) & 0x80000000u) break;
            __nanosleep(32);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

// Partition barrier number e (1, 2, ...): every block adds `value` for its
// partition, the partition's leader (block 0 of it) posts the partition sum
// in every partition's mailbox (system-scope release: the halo stores of all
// its blocks come first) and sums all partitions' posts of epoch e; returns
// that global sum to every block.  Mailboxes are double buffered by epoch
// parity: a partition can post e + 2 only after every partition has posted
// e + 1, i.e. after every leader has read the posts of e.
// A leader that waits more than kPeerWaitNs for a peer partition's post (a
// GPU of the job gone or hung) sets *tflag, treats the missing posts as 0 --
// so the loop ends -- and the call returns MIS2_EINTERNAL instead of hanging.
constexpr unsigned long long kPeerWaitNs = 10000000000ull;  // 10 s
static __device__ unsigned long long part_sync(const PartK& pk, const PeerTab& peers, int lb, unsigned int e,
                                        unsigned long long value, unsigned long long* tflag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (value) atomicAdd(&pk.acc[e & 1], value);
        // this block's halo stores before the post
        if (peers.P > 1 && peers.sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    part_barrier(pk.bar, lb, pk.nblk);
    __shared__ unsigned long long s_sum;
    if (peers.P == 1) {  // one partition: the sum is complete after the barrier
        if (threadIdx.x == 0) {
            s_sum = *(volatile unsigned long long*)&pk.acc[e & 1];
            if (lb == 0) pk.acc[(e + 1) & 1] = 0ull;  // last read at epoch e - 1
        }
        __syncthreads();
        return s_sum;
    }
    if (threadIdx.x == 0) {
        if (lb == 0) {
            const unsigned long long mine = *(volatile unsigned long long*)&pk.acc[e & 1];
            pk.acc[(e + 1) & 1] = 0ull;  // last read at epoch e - 1
            const unsigned long long post = ((unsigned long long)e << 32) | (mine & 0xffffffffull);
            for (int q = 0; q < peers.P; q++) {
                unsigned long long* dst = peers.box[q] + (e & 1) * peers.P + pk.gpart;
                if (peers.sys) asm volatile("st.release.sys.u64 [%0], %1;" ::"l"(dst), "l"(post) : "memory");
                else asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(dst), "l"(post) : "memory");
            }
            unsigned long long sum = 0;
            unsigned long long t0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            bool dead = *(volatile unsigned long long*)tflag != 0ull;
            for (int q = 0; q < peers.P; q++) {
                unsigned long long v;
                const unsigned long long* src = pk.box + (e & 1) * peers.P + q;
                for (;;) {
                    if (peers.sys) asm volatile("ld.acquire.sys.u64 %0,[%1];" : "=l"(v) : "l"(src) : "memory");
                    else asm volatile("ld.acquire.gpu.u64 %0,[%1];" : "=l"(v) : "l"(src) : "memory");
                    if ((unsigned int)(v >> 32) == e) break;
                    unsigned long long now;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                    if (dead || now - t0 > kPeerWaitNs) {
                        dead = true;
                        *(volatile unsigned long long*)tflag = 1ull;
                        v = 0ull;
                        break;
                    }
                    __nanosleep(64);
                }
                sum += v & 0xffffffffull;
            }
            if (dead) sum = 0ull;
            asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(pk.rel), "l"(((unsigned long long)e << 32) | sum)
                         : "memory");
            s_sum = sum;
        } else {
            unsigned long long v;
            for (;;) {
                asm volatile("ld.relaxed.gpu.u64 %0,[%1];" : "=l"(v) : "l"(pk.rel) : "memory");
                if ((unsigned int)(v >> 32) == e) break;
                __nanosleep(32);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            s_sum = v & 0xffffffffull;
        }
    }
    __syncthreads();
    return s_sum;
}

// halo entries of the rows this block owns, pushed right after the block
// computed them (its own __syncthreads ends the phase): peer[X][dst] = X[src].
// No partition-wide barrier before the pushes -- the values are this block's.
// The entries of run k are [send_csp[lo_k / 8], send_csp[ceil(hi_k / 8)]);
// every thread takes a contiguous group of runs, the groups' entry counts
// are scanned in shared memory (the staging buffers are idle between
// phases) and the entries are then pushed by all threads at once.
template <typename W>
__device__ __forceinline__ void push_halo(TileSmem& sm, const PartK& pk, const Rows& rows, const W* src_arr,
                                          W* const* peer_arr) {
    if (pk.nsend == 0) return;
    __syncthreads();
    const int t = threadIdx.x;
    const int64_t per = (rows.nruns + kMB - 1) / kMB;  // runs of this thread: [t * per, t * per + per)
    int64_t* pre = reinterpret_cast<int64_t*>(sm.buf[0]);  // [kMB + 1] exclusive prefix of the groups' counts
    if (t == 0) sm.gen0 = 1;
    int64_t cnt = 0;
    for (int64_t k = t * per; k < rows.nruns && k < (t + 1) * per; k++)
        cnt += pk.send_csp[(rows.run_hi(k) + 7) >> 3] - pk.send_csp[rows.run_lo(k) >> 3];
    // block exclusive scan of cnt
    int64_t x = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, x, off);
        if ((t & 31) >= off) x += y;
    }
    if ((t & 31) == 31) sm.red64[t >> 5] = (uint64_t)x;
    __syncthreads();
    int64_t wbase = 0;
    for (int w = 0; w < (t >> 5); w++) wbase += (int64_t)sm.red64[w];
    pre[t] = wbase + x - cnt;
    if (t == kMB - 1) pre[kMB] = wbase + x;
    __syncthreads();
    const int64_t total = pre[kMB];
    for (int64_t j = t; j < total; j += kMB) {
        int lo = 0, hi = kMB;  // the group holding entry j: pre[g] <= j < pre[g + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= j) lo = mid;
            else hi = mid;
        }
        // walk the group's runs to the one holding entry j
        int64_t r = j - pre[lo];
        int64_t k = (int64_t)lo * per;
        for (;; k++) {
            const int64_t a = pk.send_csp[rows.run_lo(k) >> 3], b = pk.send_csp[(rows.run_hi(k) + 7) >> 3];
            if (r < b - a) {
                const int64_t i = a + r;
                peer_arr[pk.send_peer[i]][pk.send_dst[i]] = src_arr[pk.send_src[i]];
                break;
            }
            r -= b - a;
        }
    }
    __syncthreads();
}

template <int G>
__global__ void __launch_bounds__(kMB, kMinBlocksPerSM) mis2_dist_persistent(const PartK* __restrict__ parts,
                                                                            int nlocal, PeerTab peers,
                                                                            unsigned int epoch0, int max_iters,
                                                                            unsigned long long* out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
    const int t = threadIdx.x;
    int pid = 0;
    while (pid + 1 < nlocal && (int)blockIdx.x >= parts[pid + 1].blk0) pid++;
    const PartK& pk = parts[pid];
    const MisParams& p = pk.mp;  // read through the (restrict) parameter block: no local copy
    const int lb = (int)blockIdx.x - pk.blk0;
    // cyclic chunks of the partition's own rows (ghost indices follow them
    // and are never owned)
    const Rows rows = make_rows(p.n, pk.nblk, lb, kMB / G, true);
    unsigned int e = epoch0;
    if (t == 0) {
        sm.nhuge = 0;
        sm.gen0 = 0;
        sm.pending = 0;
        {
            uint64_t pol;
            if (p.gather_keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
            s_keep_pol = pol;
        }
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        mbar_init(&sm.mbarS[0], kMB / sparse_group<G>());
        mbar_init(&sm.mbarS[1], kMB / sparse_group<G>());
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sm.pol = l2_policy(p, rows);
        s_use_keys = 0;
    }
    uint32_t ph = 0u;
    // worklists <- the active owned rows; Refresh Row of iteration 0
    int act_block = 0;
    {
        const uint64_t fi0 = p.prio.iter_term(0);
        if (t == 0) sm.cnt = 0;
        __syncthreads();
        for (int64_t base = 0; base < rows.count; base += kMB) {
            const bool in = base + t < rows.count;
            const int64_t v = in ? rows.row_at(base + t) : 0;
            const bool act = in && (p.labels ? (p.labels[v] < 0) : true);
            if (in) {
                p.T[v] = act ? p.prio.word(0, fi0, p.gbase + v) : kOUT;
                p.M[v] = act ? kPending : 0u;  // 0 = inactive sentinel (reading Q15)
            }
            const unsigned ball = __ballot_sync(kFull, act);
            if (ball) {
                const int lane = t & 31, leader = __ffs(ball) - 1;
                int pos = 0;
                if (lane == leader) pos = atomicAdd(&sm.cnt, __popc(ball));
                pos = __shfl_sync(kFull, pos, leader);
                if (act) {
                    const int64_t at = rows.seg + pos + __popc(ball & lanemask_lt());
                    p.L1[0][at] = (int32_t)v;
                    p.L2[0][at] = (int32_t)v;
                }
            }
        }
        __syncthreads();
        act_block = sm.cnt;
        __syncthreads();
    }
    // ghost T / M of iteration 0 (inactive ghosts: T = OUT, M = 0)
    push_halo<uint64_t>(sm, pk, rows, p.T, peers.T);
    push_halo<uint32_t>(sm, pk, rows, p.M, peers.M);
    const unsigned long long n_active = part_sync(pk, peers, lb, ++e, (unsigned long long)act_block, out + 3);

    int it = 0, status = MIS2_OK;
    const int64_t range = rows.count;
    int cnt1 = act_block, cnt2 = act_block;
    while (n_active > 0) {  // while worklist_1 != {}
        const int cur = it & 1;
        // ---- Refresh Column over worklist_2; ghost M pushed to the peers
        const bool dense2 = (int64_t)cnt2 * kDenseDen >= range * kDenseNum;
        cnt2 = dense2 ? dense_phase<G, false, 0>(sm, p, it, rows, p.L2[cur ^ 1], ph, 0)
                      : sparse_phase<G, false, 0>(sm, p, it, rows.seg, p.L2[cur], cnt2, p.L2[cur ^ 1], ph, 0);
        push_halo<uint32_t>(sm, pk, rows, p.M, peers.M);
        part_sync(pk, peers, lb, ++e, 0ull, out + 3);
        // ---- Decide over worklist_1 + fused refresh; ghost T pushed
        const uint64_t fi_next = p.prio.iter_term(it + 1);
        const bool dense1 = (int64_t)cnt1 * kDenseDen >= range * kDenseNum;
        cnt1 = dense1 ? dense_phase<G, false, 1>(sm, p, it, rows, p.L1[cur ^ 1], ph, fi_next)
                      : sparse_phase<G, false, 1>(sm, p, it, rows.seg, p.L1[cur], cnt1, p.L1[cur ^ 1], ph, fi_next);
        push_halo<uint64_t>(sm, pk, rows, p.T, peers.T);
        const unsigned long long remaining = part_sync(pk, peers, lb, ++e, (unsigned long long)cnt1, out + 3);
        it++;
        if (remaining == 0) break;
        if (it >= max_iters) {  // reading Q12
            status = MIS2_ENOTCONVERGED;
            break;
        }
    }
    // return {v : T_v = IN}; the global count through one more barrier
    l2_release(p, rows);
    int cnt = 0;
    for (int64_t i = t; i < rows.count; i += kMB) {
        const int64_t v = rows.row_at(i);
        const uint8_t in = (p.T[v] == kIN);
        p.in_set[v] = in;
        cnt += in;
    }
    const long long bc = block_sum_int(sm, cnt);
    const unsigned long long total = part_sync(pk, peers, lb, ++e, (unsigned long long)bc, out + 3);
    if (blockIdx.x == 0 && t == 0) {
        out[0] = total;
        if (*(volatile unsigned long long*)(out + 3)) status = MIS2_EINTERNAL;  // a peer never arrived
        out[1] = (unsigned long long)(unsigned)it | ((unsigned long long)(unsigned)status << 32);
        out[2] = e;  // the last epoch used
    }
}

}  // namespace mis2k
