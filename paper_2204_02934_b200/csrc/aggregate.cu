// aggregate.cu -- Alg. 3 "MIS-2 based Aggregation" (§III-B) on
// the device.  Both MIS-2 calls run the persistent kernel of mis2_core.cu;
// the phase bookkeeping is a handful of row-parallel kernels (G lanes per
// CSR row, as in the MIS-2 passes) plus two exclusive scans that number the
// aggregates in ascending root order (reading Q18).
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace mis2k {

enum AggErr : int { kErrTwoRoots = 1, kErrPhase2Conflict = 2, kErrNoCandidate = 4 };

// warp-uniform loop over rows, G lanes per row
#define ROWS_BEGIN(G, n)                                                                   \
    constexpr int RPW = 32 / (G);                                                          \
    const int lane = threadIdx.x & 31, grp = lane / (G), sub = lane % (G);                 \
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);                         \
    const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);    \
    for (int64_t base = gwarp * RPW; base < (n); base += nwarps * RPW) {                   \
        const int64_t v = base + grp;                                                      \
        const bool valid = v < (n);

#define ROWS_END }

constexpr int kBatch = 8;  // gathers in flight per lane (row_batched)

// Phase 1: roots = MIS-2; every root and its neighbours get the
// root's id (pull form: each vertex looks for its unique root neighbour).
template <int G>
__global__ void k_phase1(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                         const uint8_t* __restrict__ in1, const int32_t* __restrict__ rid,
                         int32_t* __restrict__ labels, int32_t* __restrict__ roots, int* err) {
    ROWS_BEGIN(G, n)
    int found = -1;
    int bad = 0;
    const bool root = valid && in1[v];
    if (valid && !root)
        row_batched<G, kBatch>(rowptr[v], rowptr[v + 1], sub, colinds, [&](int32_t w) { return in1[w]; },
                               [&](int32_t w, uint8_t x) {
                                   if (w != v && x) {
                                       const int r = rid[w];
                                       if (found >= 0 && found != r) bad = 1;
                                       found = r;
                                   }
                               });
    // combine: all lanes that found a root must agree (roots are >= 3 apart)
    int mx = found, mn = found < 0 ? 0x7fffffff : found;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        mx = max(mx, __shfl_xor_sync(kFull, mx, off));
        mn = min(mn, __shfl_xor_sync(kFull, mn, off));
    }
    bad = group_or<G>(bad);
    if (valid && sub == 0) {
        if (root) {
            labels[v] = rid[v];
            if (roots) roots[rid[v]] = (int32_t)v;
        } else {
            labels[v] = mx;  // -1 when no root neighbour (UNAGG)
            if (bad || (mx >= 0 && mn != mx)) atomicOr(err, kErrTwoRoots);
        }
    }
    ROWS_END
}

// Phase 2 accept rule (reading Q16): an M2 root is accepted iff it has
// >= 2 neighbours w != v that are unaggregated after phase 1.
template <int G>
__global__ void k_phase2_accept(int64_t n, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ colinds, const uint8_t* __restrict__ in2,
                                const int32_t* __restrict__ labels, uint8_t* __restrict__ acc) {
    ROWS_BEGIN(G, n)
    const bool r = valid && in2[v];
    int cnt = 0;
    if (r)
        row_batched<G, kBatch>(rowptr[v], rowptr[v + 1], sub, colinds, [&](int32_t w) { return labels[w]; },
                               [&](int32_t w, int32_t x) { cnt += (w != v && x < 0); });
    cnt = group_sum<G>(cnt);
    if (valid && sub == 0) acc[v] = (r && cnt >= 2) ? 1 : 0;
    ROWS_END
}

// Phase 2 labels (reading Q17): accepted root v gets id n1 + aid[v];
// its unaggregated neighbours join it (pull form).
template <int G>
__global__ void k_phase2_label(int64_t n, const int64_t* __restrict__ rowptr,
                               const int32_t* __restrict__ colinds, const uint8_t* __restrict__ acc,
                               const int32_t* __restrict__ aid, const int32_t* __restrict__ d_n1,
                               int32_t* __restrict__ labels, int32_t* __restrict__ roots, int* err) {
    const int32_t n1 = *d_n1;
    ROWS_BEGIN(G, n)
    const bool un = valid && labels[v] < 0;
    const bool root = un && acc[v];
    int found = -1, bad = 0;
    if (un && !root)
        row_batched<G, kBatch>(rowptr[v], rowptr[v + 1], sub, colinds, [&](int32_t w) { return acc[w]; },
                               [&](int32_t w, uint8_t x) {
                                   if (w != v && x) {
                                       if (found >= 0 && found != aid[w]) bad = 1;
                                       found = aid[w];
                                   }
                               });
    int mx = found, mn = found < 0 ? 0x7fffffff : found;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        mx = max(mx, __shfl_xor_sync(kFull, mx, off));
        mn = min(mn, __shfl_xor_sync(kFull, mn, off));
    }
    bad = group_or<G>(bad);
    if (un && sub == 0) {
        if (root) {
            labels[v] = n1 + aid[v];
            if (roots) roots[n1 + aid[v]] = (int32_t)v;
        } else if (mx >= 0) {
            labels[v] = n1 + mx;
            if (bad || mn != mx) atomicOr(err, kErrPhase2Conflict);
        }
    }
    ROWS_END
}

// tent <- labels; aggsize(a) <- |{v : tent_v = a}|
__global__ void k_tent_size(int64_t n, const int32_t* __restrict__ labels, int32_t* __restrict__ tent,
                            int32_t* __restrict__ size, unsigned long long* leftovers) {
    int cnt = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = labels[v];
        tent[v] = a;
        if (a >= 0) atomicAdd(&size[a], 1);
        else cnt++;
    }
    cnt = group_sum<32>(cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(leftovers, (unsigned long long)cnt);
}

// candidate order for phase 3: larger coupling, then smaller aggsize, then
// smaller aggregate id (reading Q19)
__device__ __forceinline__ bool better(int c1, int s1, int a1, int c2, int s2, int a2) {
    if (a2 < 0) return a1 >= 0;
    if (a1 < 0) return false;
    if (c1 != c2) return c1 > c2;
    if (s1 != s2) return s1 < s2;
    return a1 < a2;
}

template <int G>
__device__ __forceinline__ void group_best(int& c, int& s, int& a) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        const int c2 = __shfl_xor_sync(kFull, c, off), s2 = __shfl_xor_sync(kFull, s, off),
                  a2 = __shfl_xor_sync(kFull, a, off);
        if (better(c2, s2, a2, c, s, a)) { c = c2; s = s2; a = a2; }
    }
}

constexpr int kHeavyDeg = 512;
#ifndef MIS2_P3LIST
#define MIS2_P3LIST 8
#endif
// distinct candidate aggregates kept per lane in phase 3 (C5 aggregation
// 18.4 / 20.4 / 26.1 ms with 8 / 12 / 16: register pressure beyond 8)
constexpr int kP3List = MIS2_P3LIST;

// Phase 3 for leftover rows of degree <= kHeavyDeg: each lane
// takes candidate entries and counts their coupling over the whole row.
template <int G>
__global__ void k_phase3(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                         const int32_t* __restrict__ tent, const int32_t* __restrict__ size,
                         int32_t* __restrict__ labels, int32_t* __restrict__ heavy, int* heavy_cnt, int* err) {
    ROWS_BEGIN(G, n)
    const bool left = valid && tent[v] < 0;
    int64_t s = 0, e = 0;
    if (left) { s = rowptr[v]; e = rowptr[v + 1]; }
    const bool is_heavy = left && (e - s) > kHeavyDeg;
    int bc = 0, bs = 0, ba = -1;
    bool done = false;
    {
        // one pass: each lane keeps the distinct candidate aggregates of its
        // entries (stride G) and their couplings in registers (a leftover sees
        // few aggregates); the group then adds up the lanes' counts by
        // shuffles.  A lane with more than 8 -> the group takes the quadratic
        // pass below.
        int32_t lab[kP3List];
        int cnt[kP3List];
        int nl = 0;
        bool overflow = false;
#pragma unroll
        for (int q = 0; q < kP3List; q++) {
            lab[q] = -1;
            cnt[q] = 0;
        }
        if (left && !is_heavy) {
            for (int64_t j0 = s + sub; j0 < e; j0 += 8 * G) {
                int32_t aa[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int64_t j = j0 + (int64_t)u * G;
                    aa[u] = -1;
                    if (j < e) {
                        const int32_t w = colinds[j];
                        aa[u] = (w != v) ? tent[w] : -1;
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int32_t a = aa[u];
                    if (a < 0) continue;
                    bool found = false;
#pragma unroll
                    for (int q = 0; q < kP3List; q++)
                        if (lab[q] == a) {
                            cnt[q]++;
                            found = true;
                        }
                    if (!found) {
                        if (nl < kP3List) {
#pragma unroll
                            for (int q = 0; q < kP3List; q++)
                                if (q == nl) {
                                    lab[q] = a;
                                    cnt[q] = 1;
                                }
                            nl++;
                        } else {
                            overflow = true;
                        }
                    }
                }
            }
        }
        int tot[kP3List];
#pragma unroll
        for (int q = 0; q < kP3List; q++) tot[q] = cnt[q];
#pragma unroll 1
        for (int r = 1; r < G; r++) {
            overflow |= __shfl_xor_sync(kFull, (int)overflow, r) != 0;
#pragma unroll
            for (int q2 = 0; q2 < kP3List; q2++) {
                const int32_t l2 = __shfl_xor_sync(kFull, lab[q2], r);
                const int c2 = __shfl_xor_sync(kFull, cnt[q2], r);
#pragma unroll
                for (int q = 0; q < kP3List; q++)
                    if (l2 >= 0 && lab[q] == l2) tot[q] += c2;
            }
        }
        if (left && !is_heavy && !overflow) {
#pragma unroll
            for (int q = 0; q < kP3List; q++)
                if (q < nl) {
                    const int sz = size[lab[q]];
                    if (better(tot[q], sz, lab[q], bc, bs, ba)) { bc = tot[q]; bs = sz; ba = lab[q]; }
                }
            done = true;
        }
    }
    if (left && !is_heavy && !done) {
        for (int64_t j = s + sub; j < e; j += G) {
            const int32_t u = colinds[j];
            const int32_t a = (u != v) ? tent[u] : -1;
            if (a < 0) continue;
            int c = 0;
            for (int64_t k = s; k < e; k++) {
                const int32_t x = colinds[k];
                c += (x != v && tent[x] == a);
            }
            const int sz = size[a];
            if (better(c, sz, a, bc, bs, ba)) { bc = c; bs = sz; ba = a; }
        }
    }
    group_best<G>(bc, bs, ba);
    if (left && sub == 0) {
        if (is_heavy) {
            heavy[atomicAdd(heavy_cnt, 1)] = (int32_t)v;
        } else if (ba < 0) {
            atomicOr(err, kErrNoCandidate);  // impossible by maximality of M1 (Q20)
        } else {
            labels[v] = ba;
        }
    }
    ROWS_END
}

// Phase 3 for heavy leftover rows: one block per row, coupling counted in a
// shared-memory hash table; labels are split into hash passes so any number
// of distinct candidates fits.
constexpr int kHashSlots = 4096;
__global__ void k_phase3_heavy(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                               const int32_t* __restrict__ tent, const int32_t* __restrict__ size,
                               int32_t* __restrict__ labels, const int32_t* __restrict__ heavy,
                               const int* heavy_cnt, int* err) {
    __shared__ int32_t keys[kHashSlots];
    __shared__ int32_t cnts[kHashSlots];
    __shared__ int s_c[32], s_s[32], s_a[32];
    const int nh = *heavy_cnt;
    for (int h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t v = heavy[h];
        const int64_t s = rowptr[v], e = rowptr[v + 1];
        const int64_t d = e - s;
        const int passes = (int)((d + kHashSlots / 2 - 1) / (kHashSlots / 2));
        int bc = 0, bs = 0, ba = -1;
        for (int pass = 0; pass < passes; pass++) {
            for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) { keys[i] = -1; cnts[i] = 0; }
            __syncthreads();
            for (int64_t j = s + threadIdx.x; j < e; j += blockDim.x) {
                const int32_t u = colinds[j];
                if (u == v) continue;
                const int32_t a = tent[u];
                if (a < 0) continue;
                const uint32_t hsh = (uint32_t)a * 2654435761u;
                if ((int)(hsh % (uint32_t)passes) != pass) continue;
                uint32_t slot = (hsh >> 7) & (kHashSlots - 1);
                for (;;) {
                    const int32_t prev = atomicCAS(&keys[slot], -1, a);
                    if (prev == -1 || prev == a) { atomicAdd(&cnts[slot], 1); break; }
                    slot = (slot + 1) & (kHashSlots - 1);
                }
            }
            __syncthreads();
            for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) {
                const int32_t a = keys[i];
                if (a >= 0) {
                    const int c = cnts[i], sz = size[a];
                    if (better(c, sz, a, bc, bs, ba)) { bc = c; bs = sz; ba = a; }
                }
            }
            __syncthreads();
        }
        group_best<32>(bc, bs, ba);
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) { s_c[warp] = bc; s_s[warp] = bs; s_a[warp] = ba; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                if (better(s_c[w], s_s[w], s_a[w], bc, bs, ba)) { bc = s_c[w]; bs = s_s[w]; ba = s_a[w]; }
            if (ba < 0) atomicOr(err, kErrNoCandidate);
            else labels[v] = ba;
        }
        __syncthreads();
    }
}

// Alg. 2 join: a vertex left unaggregated by phase 1 joins the
// aggregate of its smallest-id aggregated neighbour ("any neighbor", made
// deterministic -- reading Q28).
template <int G>
__global__ void k_basic_join(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colinds,
                             const int32_t* __restrict__ tent, int32_t* __restrict__ labels, int* err) {
    ROWS_BEGIN(G, n)
    const bool left = valid && tent[v] < 0;
    int best = 0x7fffffff;
    if (left)
        for (int64_t j = rowptr[v] + sub; j < rowptr[v + 1]; j += G) {
            const int32_t u = colinds[j];
            if (u != v && tent[u] >= 0 && u < best) best = u;
        }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(kFull, best, off));
    if (left && sub == 0) {
        if (best == 0x7fffffff) atomicOr(err, kErrNoCandidate);  // impossible by maximality
        else labels[v] = tent[best];
    }
    ROWS_END
}

__global__ void k_finish(const int32_t* d_n1, const int32_t* d_n2, int64_t* out_na) {
    *out_na = (int64_t)*d_n1 + (int64_t)*d_n2;
}

}  // namespace mis2k

namespace mis2h {
using namespace mis2k;

struct AggWs {
    Mis2Ws mis;
    uint8_t *in1, *in2, *acc;
    int32_t *rid, *aid, *tent, *size, *heavy;
    void* scan_tmp;
    long long* scal;  // device scalars
};

static void carve_agg(Carve& c, int64_t n, int64_t nnz, int max_warps, AggWs* w) {
    carve_mis2(c, n, nnz, max_warps, &w->mis);
    w->in1 = c.take<uint8_t>((size_t)n + 1);
    w->in2 = c.take<uint8_t>((size_t)n + 1);
    w->acc = c.take<uint8_t>((size_t)n + 1);
    w->rid = c.take<int32_t>((size_t)n + 1);
    w->aid = c.take<int32_t>((size_t)n + 1);
    w->tent = c.take<int32_t>((size_t)n + 1);
    w->size = c.take<int32_t>((size_t)n + 1);
    w->heavy = c.take<int32_t>((size_t)n + 1);
    w->scan_tmp = c.take<char>(scan_ws_bytes(n));
    w->scal = c.take<long long>(32);
}

// device scalar slots in AggWs::scal
enum { kCount1 = 0, kCount2 = 1, kNa = 2, kLeft = 3, kIters1 = 8, kIters2 = 9, kStatus1 = 10,
       kStatus2 = 11, kN1 = 12, kN2 = 13, kErr = 14, kHeavyCnt = 15 };

template <int G>
static void launch_rows(int64_t n, int sms, cudaStream_t s, int which, const mis2_graph& g, AggWs& w,
                        int32_t* labels, int32_t* roots) {
    int32_t* s32 = (int32_t*)w.scal;
    const int64_t rows_per_block = (int64_t)(kBlock / 32) * (32 / G);
    int64_t blocks = (n + rows_per_block - 1) / rows_per_block;
    const int64_t cap = (int64_t)sms * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    switch (which) {
        case 1:
            k_phase1<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.in1, w.rid, labels, roots,
                                                          &s32[2 * kErr]);
            break;
        case 2:
            k_phase2_accept<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.in2, labels, w.acc);
            break;
        case 3:
            k_phase2_label<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.acc, w.aid,
                                                                &s32[2 * kN1], labels, roots, &s32[2 * kErr]);
            break;
        case 4:
            k_phase3<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.tent, w.size, labels, w.heavy,
                                                          &s32[2 * kHeavyCnt], &s32[2 * kErr]);
            break;
        case 5:
            k_basic_join<G><<<(unsigned)blocks, kBlock, 0, s>>>(n, g.rowptr, g.colinds, w.tent, labels, &s32[2 * kErr]);
            break;
    }
    count_launch();
}

static void rows(int G, int64_t n, int sms, cudaStream_t s, int which, const mis2_graph& g, AggWs& w,
                 int32_t* labels, int32_t* roots) {
    switch (G) {
        case 1: launch_rows<1>(n, sms, s, which, g, w, labels, roots); break;
        case 2: launch_rows<2>(n, sms, s, which, g, w, labels, roots); break;
        case 4: launch_rows<4>(n, sms, s, which, g, w, labels, roots); break;
        case 8: launch_rows<8>(n, sms, s, which, g, w, labels, roots); break;
        case 16: launch_rows<16>(n, sms, s, which, g, w, labels, roots); break;
        default: launch_rows<32>(n, sms, s, which, g, w, labels, roots); break;
    }
}

// ---- raw-array launchers of the row kernels, for the partitioned driver
// (dist.cu): rows are a partition's owned rows, colinds are local indices
// and every array read through colinds holds the ghosts after the owned rows.
static int64_t row_blocks(int G, int64_t n, int sms) {
    const int64_t rows_per_block = (int64_t)(kBlock / 32) * (32 / G);
    int64_t blocks = (n + rows_per_block - 1) / rows_per_block;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    return blocks < 1 ? 1 : blocks;
}
#define AGG_DISPATCH(G, CALL)                  \
    switch (G) {                               \
        case 1: { constexpr int GG = 1; CALL; } break;  \
        case 2: { constexpr int GG = 2; CALL; } break;  \
        case 4: { constexpr int GG = 4; CALL; } break;  \
        case 8: { constexpr int GG = 8; CALL; } break;  \
        case 16: { constexpr int GG = 16; CALL; } break; \
        default: { constexpr int GG = 32; CALL; } break; \
    }
void agg_phase1(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* in1,
                const int32_t* rid, int32_t* labels, int* err, int sms, cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase1<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, in1, rid, labels, nullptr, err)));
    count_launch();
}
void agg_accept(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* in2,
                const int32_t* labels, uint8_t* acc, int sms, cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase2_accept<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, in2, labels, acc)));
    count_launch();
}
void agg_phase2_label(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const uint8_t* acc,
                      const int32_t* aid, const int32_t* d_n1, int32_t* labels, int* err, int sms, cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase2_label<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, acc, aid, d_n1, labels, nullptr, err)));
    count_launch();
}
void agg_tent_size(int64_t n, const int32_t* labels, int32_t* tent, int32_t* size, unsigned long long* left, int sms,
                   cudaStream_t s) {
    int64_t blocks = (n + kBlock - 1) / kBlock;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    if (blocks < 1) blocks = 1;
    k_tent_size<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, tent, size, left);
    count_launch();
}
void agg_phase3(int G, int64_t n, const int64_t* rowptr, const int32_t* colinds, const int32_t* tent,
                const int32_t* size, int32_t* labels, int32_t* heavy, int* heavy_cnt, int* err, int sms,
                cudaStream_t s) {
    const unsigned b = (unsigned)row_blocks(G, n, sms);
    AGG_DISPATCH(G, (k_phase3<GG><<<b, kBlock, 0, s>>>(n, rowptr, colinds, tent, size, labels, heavy, heavy_cnt, err)));
    count_launch();
    k_phase3_heavy<<<sms * 4, kBlock, 0, s>>>(rowptr, colinds, tent, size, labels, heavy, heavy_cnt, err);
    count_launch();
}
#undef AGG_DISPATCH

int run_aggregate(const mis2_graph& g, const mis2_opts& o, int32_t* labels, int64_t* num_aggs, int32_t* roots,
                  int64_t* stats, void* ws, size_t ws_bytes, cudaStream_t s, size_t* bytes_needed) {
    DeviceInfo di;
    MIS2_TRY(device_info(&di));
    Carve c(ws, ws_bytes);
    AggWs w;
    carve_agg(c, g.n, g.nnz, max_coop_warps(di), &w);
    if (bytes_needed) { *bytes_needed = c.off; return MIS2_OK; }
    if (!c.ok()) { set_error("workspace too small: need %zu bytes", c.off); return MIS2_ENOMEM; }
    const int64_t n = g.n;
    const int G = choose_group(g.n, g.nnz, o.group);
    int32_t* s32 = (int32_t*)w.scal;
    MIS2_CUDA_TRY(cudaMemsetAsync(w.scal, 0, 32 * sizeof(long long), s));

    // per-iteration worklist statistics of both MIS-2 calls (MIS2_FLAG_ITER_STATS)
    const bool iter_stats = stats && (o.flags & MIS2_FLAG_ITER_STATS) && !(o.flags & MIS2_FLAG_TIMELINE);
    const int64_t mi = max_iters_for(n, o.max_iters);
    int64_t* ist1 = iter_stats ? stats + 8 : nullptr;
    int64_t* ist2 = iter_stats ? stats + 8 + 6 * mi : nullptr;
    if (iter_stats) memset(stats + 8, 0, sizeof(int64_t) * 12 * (size_t)mi);

    // ---- phase 1: M1 = MIS2(G)
    MIS2_TRY(run_mis2(g, o, nullptr, w.in1, (int64_t*)&w.scal[kCount1], &s32[2 * kIters1],
                      &s32[2 * kStatus1], ist1, w.mis, s));
    MIS2_TRY(scan_flags(w.in1, n, w.rid, &s32[2 * kN1], w.scan_tmp, s));
    rows(G, n, di.sms, s, 1, g, w, labels, roots);

    const bool basic = (o.flags & MIS2_FLAG_BASIC) != 0;
    if (basic) {
        // ---- Alg. 2: every leftover joins an adjacent phase-1 aggregate
        MIS2_CUDA_TRY(cudaMemsetAsync(w.size, 0, sizeof(int32_t) * ((size_t)n + 1), s));
        int64_t blocks = (n + kBlock - 1) / kBlock;
        if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
        if (blocks < 1) blocks = 1;
        k_tent_size<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, w.tent, w.size,
                                                        (unsigned long long*)&w.scal[kLeft]);
        count_launch();
        rows(G, n, di.sms, s, 5, g, w, labels, roots);
        k_finish<<<1, 1, 0, s>>>(&s32[2 * kN1], &s32[2 * kN2], (int64_t*)&w.scal[kNa]);
        count_launch();
    } else {

    // ---- phase 2: M2 = MIS2(G \ aggregated) on the same ids / seed (Q15)
    MIS2_TRY(run_mis2(g, o, labels, w.in2, (int64_t*)&w.scal[kCount2], &s32[2 * kIters2],
                      &s32[2 * kStatus2], ist2, w.mis, s));
    rows(G, n, di.sms, s, 2, g, w, labels, roots);
    MIS2_TRY(scan_flags(w.acc, n, w.aid, &s32[2 * kN2], w.scan_tmp, s));
    rows(G, n, di.sms, s, 3, g, w, labels, roots);

    // ---- phase 3: frozen tentative labels, max coupling / min size / min id
    MIS2_CUDA_TRY(cudaMemsetAsync(w.size, 0, sizeof(int32_t) * ((size_t)n + 1), s));
    {
        int64_t blocks = (n + kBlock - 1) / kBlock;
        if (blocks > (int64_t)di.sms * 16) blocks = (int64_t)di.sms * 16;
        if (blocks < 1) blocks = 1;
        k_tent_size<<<(unsigned)blocks, kBlock, 0, s>>>(n, labels, w.tent, w.size,
                                                        (unsigned long long*)&w.scal[kLeft]);
        count_launch();
    }
    rows(G, n, di.sms, s, 4, g, w, labels, roots);
    k_phase3_heavy<<<di.sms * 4, kBlock, 0, s>>>(g.rowptr, g.colinds, w.tent, w.size, labels, w.heavy,
                                                &s32[2 * kHeavyCnt], &s32[2 * kErr]);
    count_launch();
    k_finish<<<1, 1, 0, s>>>(&s32[2 * kN1], &s32[2 * kN2], (int64_t*)&w.scal[kNa]);
    count_launch();
    }  // Alg. 3
    MIS2_CUDA_TRY(cudaGetLastError());

    long long h[32];
    MIS2_CUDA_TRY(cudaMemcpyAsync(h, w.scal, sizeof(h), cudaMemcpyDeviceToHost, s));
    MIS2_CUDA_TRY(cudaStreamSynchronize(s));
    const int32_t* h32 = (const int32_t*)h;
    if (h32[2 * kStatus1] != MIS2_OK || h32[2 * kStatus2] != MIS2_OK) {
        set_error("MIS-2 did not converge within max_iters");
        return MIS2_ENOTCONVERGED;
    }
    if (h32[2 * kErr] != 0) {
        set_error("aggregation invariant failed (flags 0x%x): input graph not symmetric?", h32[2 * kErr]);
        return MIS2_EINTERNAL;
    }
    *num_aggs = h[kNa];
    if (stats) {
        stats[0] = h[kCount1];
        stats[1] = h32[2 * kIters1];
        stats[2] = h[kCount2];
        stats[3] = h32[2 * kIters2];
        stats[4] = h32[2 * kN2];
        stats[5] = h[kLeft];
        stats[6] = h32[2 * kN1];
        stats[7] = h[kNa];
    }
    return MIS2_OK;
}

}  // namespace mis2h
